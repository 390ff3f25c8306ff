// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into or called by the
// product path (paper_1704_01144_b200/). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.
//
// A CPU restatement of the reference's LTS finite-volume iteration
// (arxiv/paper_1704_01144, proj/core), generalised from scalar 2D to
// {scalar 2D advection/Burgers, compressible Euler 3D}:
//   * kernels            proj/core/src/kernels.cpp:13-271
//   * levels and plan    proj/core/src/levels.cpp:10-155
//   * driver             proj/core/src/reference.cpp:27-199
//   * adjacency/closure  proj/core/src/mesh.cpp:241-284
//   * state bookkeeping  proj/core/src/state.cpp:14-75
//   * physics            proj/core/include/tafv/physics.hpp:14-47
// Every expression keeps the reference's association order, the build uses
// -ffp-contract=off (proj/core/CMakeLists.txt:26), min/max keep std::min /
// std::max operand semantics, and per-cell sums run over the CSR slots in
// ascending face id. The scalar-2D instantiation is pinned BITWISE against
// the real reference library (oracle/_ref) and the golden fixtures under
// tests/golden; the Euler-3D instantiation differs only in the physics
// functions, which no reference test pins ("parity
// unpinned" for the Euler physics; the LTS machinery around it is pinned).
//
// Threading: every kernel is a pure per-item loop (kernels.hpp:12-21), so the
// item list is split into contiguous chunks over a small thread pool, the
// same shape as the reference's LaneGang (runtime.cpp:16-79). Results are
// bitwise independent of the thread count. A second driver (TaskDriver, below)
// runs the same kernels as per-CE tasks with declared data accesses on a
// sequential-task-flow runtime, the shape of the reference's TaskEngine
// (taskgen.cpp:348-661), as a timed CPU baseline; bitwise the same state.
// ============================================================================

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <exception>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

namespace oracle {

// --- error convention (common.hpp:9-25) -------------------------------------
inline void require(bool cond, const char* what) {
  if (!cond) throw std::invalid_argument(what);
}
#define ORC_ASSERT(cond, what) \
  do {                         \
    if (!(cond)) throw std::logic_error(what); \
  } while (0)

// std::min / std::max operand semantics (NaN behaviour matters).
inline double smin(double a, double b) { return (b < a) ? b : a; }
inline double smax(double a, double b) { return (a < b) ? b : a; }

// --- thread pool (LaneGang shape) --------------------------------------------
class Pool {
 public:
  explicit Pool(int n) : n_(std::max(1, n)) {
    for (int t = 1; t < n_; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return n_; }
  // Run body(begin, end) over [0, n) in n_ contiguous chunks.
  void run(int64_t n, const std::function<void(int64_t, int64_t)>& body) {
    if (n_ == 1 || n < 4096) {
      body(0, n);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      body_ = &body;
      total_ = n;
      pending_ = n_ - 1;
      err_ = nullptr;
      ++gen_;
    }
    cv_.notify_all();
    chunk(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    body_ = nullptr;
    if (err_) std::rethrow_exception(err_);
  }

 private:
  void chunk(int t) {
    const int64_t b = total_ * t / n_, e = total_ * (t + 1) / n_;
    try {
      (*body_)(b, e);
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu_);
      if (!err_) err_ = std::current_exception();
    }
  }
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      chunk(t);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  int n_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  uint64_t gen_ = 0;
  bool stop_ = false;
  const std::function<void(int64_t, int64_t)>* body_ = nullptr;
  int64_t total_ = 0;
  int pending_ = 0;
  std::exception_ptr err_;
};

// --- mesh (mesh.hpp:26-65 generalised to Vec3) --------------------------------
struct Mesh {
  int dim = 2;
  int nc = 0, nf = 0;
  std::vector<double> vol, cen, chl;   // cen: nc x 3
  std::vector<int> fl, fr, fp;         // left, right, periodic partner
  std::vector<double> fn, fa, fc;      // fn, fc: nf x 3
  std::vector<int> adj_off, adj_face, adj_nb;
  std::vector<double> adj_sign;

  int resolved_right(int f) const {  // kernels.cpp:15-20
    if (fr[f] >= 0) return fr[f];
    if (fp[f] >= 0) return fl[fp[f]];
    return -1;
  }
};

// mesh.cpp:241-271: faces visited in ascending id, so each cell's slots are
// sorted by face id; this fixes every per-cell summation order.
void build_adjacency(Mesh& m) {
  std::vector<int> count(m.nc, 0);
  for (int f = 0; f < m.nf; ++f) {
    require(m.fl[f] >= 0 && m.fl[f] < m.nc, "mesh: face left cell out of range");
    require(m.fr[f] < m.nc, "mesh: face right cell out of range");
    ++count[m.fl[f]];
    if (m.fr[f] >= 0) ++count[m.fr[f]];
  }
  m.adj_off.assign(m.nc + 1, 0);
  for (int c = 0; c < m.nc; ++c) m.adj_off[c + 1] = m.adj_off[c] + count[c];
  const int total = m.adj_off.back();
  m.adj_face.resize(total);
  m.adj_nb.resize(total);
  m.adj_sign.resize(total);
  std::vector<int> cursor(m.adj_off.begin(), m.adj_off.end() - 1);
  for (int f = 0; f < m.nf; ++f) {
    int nb = m.fr[f];
    if (nb < 0 && m.fp[f] >= 0) nb = m.fl[m.fp[f]];
    const int sl = cursor[m.fl[f]]++;
    m.adj_face[sl] = f;
    m.adj_nb[sl] = nb;
    m.adj_sign[sl] = 1.0;
    if (m.fr[f] >= 0) {
      const int sr = cursor[m.fr[f]]++;
      m.adj_face[sr] = f;
      m.adj_nb[sr] = m.fl[f];
      m.adj_sign[sr] = -1.0;
    }
  }
}

// mesh.cpp:273-284 (plus the z component in 3D). `mask` (optional) limits
// the check to cells with a complete face set (a shard's ring-2 cells are not).
void check_closure(const Mesh& m, const uint8_t* mask = nullptr) {
  for (int c = 0; c < m.nc; ++c) {
    if (mask && !mask[c]) continue;
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
      const int f = m.adj_face[t];
      sx += m.adj_sign[t] * m.fn[3 * f] * m.fa[f];
      sy += m.adj_sign[t] * m.fn[3 * f + 1] * m.fa[f];
      sz += m.adj_sign[t] * m.fn[3 * f + 2] * m.fa[f];
    }
    if (std::abs(sx) > 1e-12 || std::abs(sy) > 1e-12 || std::abs(sz) > 1e-12)
      throw std::logic_error("mesh: geometric closure violated for a cell");
  }
}

// --- physics (physics.hpp:14-47; Euler per SURVEY.md Appendix B) ------------
// Face-state admissibility (Euler only; SURVEY.md Appendix B.7 decision, see
// DESIGN.md): a reconstructed face state with non-positive density or
// pressure falls back to the first-order cell value on that side. Scalar
// models accept every state, leaving the reference arithmetic untouched.
struct Advection2D {
  static constexpr int NV = 1, DIM = 2;
  static bool admissible(const double*) { return true; }
  double ax, ay;
  void flux_n(const double* w, const double* n, double* f) const {
    f[0] = ax * w[0] * n[0] + ay * w[0] * n[1];  // flux(w).x*n.x + flux(w).y*n.y
  }
  double speed(const double*) const { return std::sqrt(ax * ax + ay * ay); }  // norm(a)
  double speed_n(const double* w, const double*) const { return speed(w); }
};

struct Burgers2D {
  static constexpr int NV = 1, DIM = 2;
  static bool admissible(const double*) { return true; }
  double ax, ay;  // unit direction (parse_flux_model normalises)
  void flux_n(const double* w, const double* n, double* f) const {
    const double q = 0.5 * w[0] * w[0];
    f[0] = ax * q * n[0] + ay * q * n[1];
  }
  double speed(const double* w) const { return std::abs(w[0]); }
  double speed_n(const double* w, const double*) const { return speed(w); }
};

// Compressible Euler, ideal gas. w = (rho, rho u, rho v, rho w, E).
struct Euler3D {
  static constexpr int NV = 5, DIM = 3;
  double gamma, gm1;
  void prim(const double* w, double& ux, double& uy, double& uz, double& p) const {
    const double rho = w[0];
    ux = w[1] / rho;
    uy = w[2] / rho;
    uz = w[3] / rho;
    const double ke = 0.5 * ((w[1] * ux + w[2] * uy) + w[3] * uz);
    p = gm1 * (w[4] - ke);
  }
  void flux_n(const double* w, const double* n, double* f) const {
    double ux, uy, uz, p;
    prim(w, ux, uy, uz, p);
    const double un = (ux * n[0] + uy * n[1]) + uz * n[2];
    f[0] = w[0] * un;
    f[1] = w[1] * un + p * n[0];
    f[2] = w[2] * un + p * n[1];
    f[3] = w[3] * un + p * n[2];
    f[4] = (w[4] + p) * un;
  }
  double sound(const double* w, double p) const { return std::sqrt((gamma * p) / w[0]); }
  bool admissible(const double* w) const {
    if (!(w[0] > 0.0)) return false;
    double ux, uy, uz, p;
    prim(w, ux, uy, uz, p);
    return p > 0.0;
  }
  double speed(const double* w) const {
    double ux, uy, uz, p;
    prim(w, ux, uy, uz, p);
    return std::sqrt((ux * ux + uy * uy) + uz * uz) + sound(w, p);
  }
  double speed_n(const double* w, const double* n) const {
    double ux, uy, uz, p;
    prim(w, ux, uy, uz, p);
    const double un = (ux * n[0] + uy * n[1]) + uz * n[2];
    return std::abs(un) + sound(w, p);
  }
};

inline double minmod(double x, double y) {  // physics.hpp:32-36
  if (x > 0.0 && y > 0.0) return smin(x, y);
  if (x < 0.0 && y < 0.0) return smax(x, y);
  return 0.0;
}

// physics.hpp:42-47, per component: 0.5*(fl+fr) - 0.5*s*(wR-wL).
template <class P>
void rusanov(const P& ph, const double* wL, const double* wR, const double* n, double* out) {
  double fl[P::NV], fr[P::NV];
  ph.flux_n(wL, n, fl);
  ph.flux_n(wR, n, fr);
  const double s = smax(ph.speed_n(wL, n), ph.speed_n(wR, n));
  for (int k = 0; k < P::NV; ++k) out[k] = 0.5 * (fl[k] + fr[k]) - 0.5 * s * (wR[k] - wL[k]);
}

// --- state (state.hpp:17-50) ------------------------------------------------
enum Phase { kCorrector = 0, kPredictor = 1 };
inline int stage_stamp(int front, int phase) { return 2 * front + phase; }  // kernels.hpp:23-27

struct State {
  int nv = 1;
  std::vector<double> w, W, W_pred, w_pred, w_eval, grad, residual, dt_max;
  std::vector<int> raw_level, committed_front, staged_front;
  std::vector<double> face_wL, face_wR, phi_pred, int_substep, int_window;
  std::vector<int> face_staged, face_front;
  double t0 = 0.0;
  int iteration = 0;

  void init(const Mesh& m, int nv_) {  // state.cpp:14-38
    nv = nv_;
    const size_t nc = m.nc, nf = m.nf;
    for (auto* v : {&w, &W, &W_pred, &w_pred, &w_eval, &residual}) v->assign(nc * nv, 0.0);
    grad.assign(nc * nv * 3, 0.0);
    dt_max.assign(nc, 0.0);
    raw_level.assign(nc, 0);
    committed_front.assign(nc, 0);
    staged_front.assign(nc, 0);
    for (auto* v : {&face_wL, &face_wR, &phi_pred, &int_substep, &int_window}) v->assign(nf * nv, 0.0);
    face_staged.assign(nf, -1);
    face_front.assign(nf, -1);
    t0 = 0.0;
    iteration = 0;
  }
};

void sync_extensive(const Mesh& m, State& st) {  // state.cpp:61-68
  for (int c = 0; c < m.nc; ++c) {
    for (int k = 0; k < st.nv; ++k) {
      st.W[c * st.nv + k] = st.w[c * st.nv + k] * m.vol[c];
      st.w_eval[c * st.nv + k] = st.w[c * st.nv + k];
    }
    st.committed_front[c] = 0;
    st.staged_front[c] = 0;
  }
}

void reset_fronts(State& st) {  // state.cpp:70-75
  std::fill(st.committed_front.begin(), st.committed_front.end(), 0);
  std::fill(st.staged_front.begin(), st.staged_front.end(), -1);
  std::fill(st.face_staged.begin(), st.face_staged.end(), -1);
  std::fill(st.face_front.begin(), st.face_front.end(), -1);
}

// --- levels (levels.cpp) ----------------------------------------------------
int subiteration_level(int s, int theta) {  // levels.cpp:10-16
  require(theta >= 0, "subiteration_level: theta must be >= 0");
  require(s >= 1 && s <= (1 << theta), "subiteration_level: s out of [1, 2^theta]");
  for (int tmp = theta; tmp > 0; --tmp)
    if ((s - 1) % (1 << tmp) == 0) return tmp;
  return 0;
}

int classify_raw(double dt_max, double dt_min, int theta_max) {  // levels.cpp:18-25
  require(dt_min > 0.0, "classify: dt_min must be positive");
  require(theta_max >= 0, "classify: theta_max must be >= 0");
  const double ratio = dt_max / dt_min;
  const int raw = ratio >= 1.0 ? std::ilogb(ratio) : 0;
  return std::clamp(raw, 0, theta_max);
}

bool smooth_sweep(const Mesh& m, const std::vector<int>& in, std::vector<int>& out) {  // :33-46
  out.resize(in.size());
  bool changed = false;
  for (int c = 0; c < m.nc; ++c) {
    int bound = in[c];
    for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
      const int nb = m.adj_nb[t];
      if (nb >= 0) bound = std::min(bound, in[nb] + 1);
    }
    out[c] = bound;
    changed = changed || bound != in[c];
  }
  return changed;
}

int smooth_to_fixpoint(const Mesh& m, std::vector<int>& tau) {  // :48-51 (returns sweeps)
  std::vector<int> next;
  int sweeps = 1;
  while (smooth_sweep(m, tau, next)) {
    tau.swap(next);
    ++sweeps;
  }
  return sweeps;
}

struct LevelMap {  // levels.hpp:12-22
  std::vector<int> tau;
  int theta = 0;
  double dt = 0.0;
  std::vector<std::vector<int>> cells_of_level;
  int64_t level_cost(int l) const {
    return (int64_t{1} << (theta - l)) * static_cast<int64_t>(cells_of_level[l].size());
  }
  double cost_ratio() const {
    int64_t total = 0;
    for (int l = 0; l <= theta; ++l) total += level_cost(l);
    if (total == 0) return 1.0;
    const int64_t plain = (int64_t{1} << theta) * static_cast<int64_t>(tau.size());
    return static_cast<double>(plain) / static_cast<double>(total);
  }
};

LevelMap make_level_map(std::vector<int> tau, double dt) {  // levels.cpp:53-66
  require(dt > 0.0, "level map: dt must be positive");
  LevelMap map;
  map.tau = std::move(tau);
  map.dt = dt;
  map.theta = 0;
  for (int t : map.tau) map.theta = std::max(map.theta, t);
  map.cells_of_level.assign(map.theta + 1, {});
  for (size_t c = 0; c < map.tau.size(); ++c) {
    require(map.tau[c] >= 0, "level map: negative level");
    map.cells_of_level[map.tau[c]].push_back(static_cast<int>(c));
  }
  return map;
}

std::vector<double> cost_shares_from_cell_shares(const std::vector<double>& cs) {  // :99-111
  require(!cs.empty(), "cost model: empty share vector");
  const int theta = static_cast<int>(cs.size()) - 1;
  std::vector<double> cost(cs.size());
  double total = 0.0;
  for (int l = 0; l <= theta; ++l) {
    cost[l] = static_cast<double>(int64_t{1} << (theta - l)) * cs[l];
    total += cost[l];
  }
  for (double& v : cost) v /= total;
  return cost;
}

double cost_ratio_from_cell_shares(const std::vector<double>& cs) {  // :113-121
  require(!cs.empty(), "cost model: empty share vector");
  const int theta = static_cast<int>(cs.size()) - 1;
  double whole = 0.0, total = 0.0;
  for (int l = 0; l <= theta; ++l) {
    whole += cs[l];
    total += static_cast<double>(int64_t{1} << (theta - l)) * cs[l];
  }
  return static_cast<double>(int64_t{1} << theta) * whole / total;
}

struct IterationPlan {  // levels.hpp:46-61
  LevelMap levels;
  std::vector<int> face_cadence;
  std::vector<std::vector<int>> faces_of_cadence;
  std::vector<std::vector<int>> fringe;
  int theta() const { return levels.theta; }
  int subiterations() const { return 1 << levels.theta; }
};

IterationPlan build_iteration_plan(const Mesh& m, LevelMap levels) {  // levels.cpp:123-155
  IterationPlan plan;
  plan.levels = std::move(levels);
  const std::vector<int>& tau = plan.levels.tau;
  require(tau.size() == static_cast<size_t>(m.nc), "plan: level/mesh mismatch");
  plan.face_cadence.resize(m.nf);
  plan.faces_of_cadence.assign(plan.levels.theta + 1, {});
  for (int f = 0; f < m.nf; ++f) {
    int nb = m.fr[f];
    if (nb < 0 && m.fp[f] >= 0) nb = m.fl[m.fp[f]];
    const int cadence = nb >= 0 ? std::min(tau[m.fl[f]], tau[nb]) : tau[m.fl[f]];
    plan.face_cadence[f] = cadence;
    plan.faces_of_cadence[cadence].push_back(f);
  }
  plan.fringe.assign(std::max(plan.levels.theta, 0), {});
  for (int c = 0; c < m.nc; ++c) {
    if (tau[c] == 0) continue;
    const int l = tau[c] - 1;
    if (l >= plan.levels.theta) continue;
    for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
      const int nb = m.adj_nb[t];
      if (nb >= 0 && tau[nb] == l) {
        plan.fringe[l].push_back(c);
        break;
      }
    }
  }
  return plan;
}

// --- kernels (kernels.cpp:31-271), templated over the physics ----------------
using Items = std::vector<int>;

struct Record {  // mirrors tafv_record (include/tafv_gpu.h)
  int32_t iteration;
  int32_t theta;
  double t_start, dt, advance, cost_ratio;
  double total_extensive[8];
  int64_t level_cells[16];
  int32_t n_levels;
  int32_t nv;
  double boundary_flux[8];  // ledger (new): outflow through transmissive faces this iteration
};

template <class P>
struct Kernels {
  static constexpr int NV = P::NV;
  static constexpr int DIM = P::DIM;
  const Mesh& m;
  State& st;
  const P& ph;
  Pool& pool;

  template <class F>
  void each(const int* items, int64_t n, F&& f) {
    pool.run(n, [&](int64_t b, int64_t e) {
      for (int64_t i = b; i < e; ++i) f(items[i]);
    });
  }

  // kernels.cpp:25-27, extended with a z term appended left to right.
  static double extrapolate(double w, const double* g, const double* from, const double* to) {
    double v = (w + g[0] * (to[0] - from[0])) + g[1] * (to[1] - from[1]);
    if constexpr (DIM == 3) v = v + g[2] * (to[2] - from[2]);
    return v;
  }

  void stage_committed(const int* it, int64_t n, int front) {  // :31-39
    const int stamp = stage_stamp(front, kPredictor);
    each(it, n, [&](int c) {
      ORC_ASSERT(st.committed_front[c] == front,
                 "predictor staging requires a window starting at this front");
      for (int k = 0; k < NV; ++k) st.w_eval[c * NV + k] = st.w[c * NV + k];
      st.staged_front[c] = stamp;
    });
  }

  void stage_predicted(const std::vector<int>& tau, const int* it, int64_t n, int front) {  // :41-49
    const int stamp = stage_stamp(front, kCorrector);
    each(it, n, [&](int c) {
      ORC_ASSERT(st.committed_front[c] + (1 << tau[c]) == front,
                 "corrector staging requires a window ending at this front");
      for (int k = 0; k < NV; ++k) st.w_eval[c * NV + k] = st.w_pred[c * NV + k];
      st.staged_front[c] = stamp;
    });
  }

  void stage_interpolated(const std::vector<int>& tau, const int* it, int64_t n, int front,
                          int phase) {  // :51-63
    const int stamp = stage_stamp(front, phase);
    each(it, n, [&](int c) {
      const int window = 1 << tau[c];
      const int offset = front - st.committed_front[c];
      ORC_ASSERT(offset > 0 && offset < window,
                 "repositioning requires a window strictly straddling this front");
      const double theta_f = static_cast<double>(offset) / static_cast<double>(window);
      for (int k = 0; k < NV; ++k) {
        const double w = st.w[c * NV + k];
        st.w_eval[c * NV + k] = w + theta_f * (st.w_pred[c * NV + k] - w);
      }
      st.staged_front[c] = stamp;
    });
  }

  void green_gauss_gradient(const int* it, int64_t n, int front, int phase) {  // :65-89
    const int stamp = stage_stamp(front, phase);
    each(it, n, [&](int c) {
      ORC_ASSERT(st.staged_front[c] == stamp, "gradient requires the cell staged at this front");
      double g[NV][3] = {};
      for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
        const int nb = m.adj_nb[t];
        if (nb >= 0)
          ORC_ASSERT(st.staged_front[nb] == stamp,
                     "gradient requires every neighbor staged at this front");
        const int f = m.adj_face[t];
        const double scale = m.adj_sign[t] * m.fa[f];
        const double* nrm = &m.fn[3 * f];
        for (int k = 0; k < NV; ++k) {
          const double w_face = nb >= 0 ? 0.5 * (st.w_eval[c * NV + k] + st.w_eval[nb * NV + k])
                                        : st.w_eval[c * NV + k];
          for (int d = 0; d < DIM; ++d) g[k][d] += w_face * nrm[d] * scale;
        }
      }
      const double inv_v = 1.0 / m.vol[c];
      for (int k = 0; k < NV; ++k)
        for (int d = 0; d < 3; ++d) st.grad[(c * NV + k) * 3 + d] = d < DIM ? g[k][d] * inv_v : 0.0;
    });
  }

  void limit_gradients(const int* it, int64_t n, int front, int phase) {  // :91-121
    const int stamp = stage_stamp(front, phase);
    each(it, n, [&](int c) {
      ORC_ASSERT(st.staged_front[c] == stamp, "limiter requires the cell staged at this front");
      double w_min[NV], w_max[NV];
      for (int k = 0; k < NV; ++k) {
        w_min[k] = std::numeric_limits<double>::infinity();
        w_max[k] = -std::numeric_limits<double>::infinity();
      }
      bool any = false;
      for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
        const int nb = m.adj_nb[t];
        if (nb < 0) continue;
        ORC_ASSERT(st.staged_front[nb] == stamp,
                   "limiter requires every neighbor staged at this front");
        for (int k = 0; k < NV; ++k) {
          w_min[k] = smin(w_min[k], st.w_eval[nb * NV + k]);
          w_max[k] = smax(w_max[k], st.w_eval[nb * NV + k]);
        }
        any = true;
      }
      if (!any) return;
      const double* cc = &m.cen[3 * c];
      for (int k = 0; k < NV; ++k) {
        double* g = &st.grad[(c * NV + k) * 3];
        const double wc = st.w_eval[c * NV + k];
        double alpha = 1.0;
        for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
          const double* fc = &m.fc[3 * m.adj_face[t]];
          double delta = g[0] * (fc[0] - cc[0]) + g[1] * (fc[1] - cc[1]);
          if constexpr (DIM == 3) delta = delta + g[2] * (fc[2] - cc[2]);
          if (delta == 0.0) continue;
          const double headroom = delta > 0.0 ? w_max[k] - wc : w_min[k] - wc;
          alpha = smin(alpha, minmod(delta, headroom) / delta);
        }
        for (int d = 0; d < DIM; ++d) g[d] *= alpha;
      }
    });
  }

  void reset_windows(const int* it, int64_t n, int front) {  // :123-130
    each(it, n, [&](int f) {
      const int nb = m.resolved_right(f);
      bool shared_start = st.committed_front[m.fl[f]] == front;
      if (nb >= 0) shared_start = shared_start && st.committed_front[nb] == front;
      if (shared_start)
        for (int k = 0; k < NV; ++k) st.int_window[f * NV + k] = 0.0;
    });
  }

  // One side of a face: limited extrapolation (kernels.cpp:25-27), with the
  // Euler admissibility fallback to the staged cell value.
  void side_state(int cell, const double* to, double* out) const {
    for (int k = 0; k < NV; ++k)
      out[k] = extrapolate(st.w_eval[cell * NV + k], &st.grad[(cell * NV + k) * 3], &m.cen[3 * cell], to);
    if (!ph.admissible(out))
      for (int k = 0; k < NV; ++k) out[k] = st.w_eval[cell * NV + k];
  }

  void reconstruct_faces(const int* it, int64_t n, int front, int phase) {  // :132-159
    const int stamp = stage_stamp(front, phase);
    each(it, n, [&](int f) {
      const int left = m.fl[f];
      ORC_ASSERT(st.staged_front[left] == stamp,
                 "face evaluation requires the left cell staged at this front");
      side_state(left, &m.fc[3 * f], &st.face_wL[f * NV]);
      if (m.fr[f] >= 0) {
        const int right = m.fr[f];
        ORC_ASSERT(st.staged_front[right] == stamp,
                   "face evaluation requires the right cell staged at this front");
        side_state(right, &m.fc[3 * f], &st.face_wR[f * NV]);
      } else if (m.fp[f] >= 0) {
        const int p = m.fp[f];
        const int right = m.fl[p];
        ORC_ASSERT(st.staged_front[right] == stamp,
                   "face evaluation requires the periodic cell staged at this front");
        side_state(right, &m.fc[3 * p], &st.face_wR[f * NV]);
      } else {
        for (int k = 0; k < NV; ++k) st.face_wR[f * NV + k] = st.face_wL[f * NV + k];
      }
      st.face_staged[f] = stamp;
    });
  }

  void riemann_predict(const int* it, int64_t n, int front) {  // :161-171
    const int stamp = stage_stamp(front, kPredictor);
    each(it, n, [&](int f) {
      ORC_ASSERT(st.face_staged[f] == stamp,
                 "predictor flux requires face states reconstructed at this front");
      double r[NV];
      rusanov(ph, &st.face_wL[f * NV], &st.face_wR[f * NV], &m.fn[3 * f], r);
      for (int k = 0; k < NV; ++k) st.phi_pred[f * NV + k] = r[k] * m.fa[f];
      st.face_front[f] = stamp;
    });
  }

  void riemann_correct(const std::vector<int>& cad, double dt, const int* it, int64_t n,
                       int front) {  // :173-186
    const int stamp = stage_stamp(front, kCorrector);
    each(it, n, [&](int f) {
      ORC_ASSERT(st.face_staged[f] == stamp,
                 "corrector flux requires face states reconstructed at this front");
      double r[NV];
      rusanov(ph, &st.face_wL[f * NV], &st.face_wR[f * NV], &m.fn[3 * f], r);
      const double dt_sub = dt * static_cast<double>(1 << cad[f]);
      for (int k = 0; k < NV; ++k) {
        const double phi_corr = r[k] * m.fa[f];
        st.int_substep[f * NV + k] = 0.5 * dt_sub * (st.phi_pred[f * NV + k] + phi_corr);
        st.int_window[f * NV + k] += st.int_substep[f * NV + k];
      }
      st.face_front[f] = stamp;
    });
  }

  void flux_sum_predict(const int* it, int64_t n, int front) {  // :188-200
    const int stamp = stage_stamp(front, kPredictor);
    each(it, n, [&](int c) {
      double sum[NV] = {};
      for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
        const int f = m.adj_face[t];
        ORC_ASSERT(st.face_front[f] == stamp,
                   "predictor residual requires every face flux evaluated at this front");
        for (int k = 0; k < NV; ++k) sum[k] += m.adj_sign[t] * st.phi_pred[f * NV + k];
      }
      for (int k = 0; k < NV; ++k) st.residual[c * NV + k] = -sum[k];
    });
  }

  void flux_sum_correct(const std::vector<int>& tau, const std::vector<int>& cad, const int* it,
                        int64_t n, int front) {  // :202-216
    const int stamp = stage_stamp(front, kCorrector);
    each(it, n, [&](int c) {
      double sum[NV] = {};
      for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
        const int f = m.adj_face[t];
        ORC_ASSERT(st.face_front[f] == stamp,
                   "correction requires every face integral evaluated at this front");
        const double* phi = tau[c] > cad[f] ? &st.int_window[f * NV] : &st.int_substep[f * NV];
        for (int k = 0; k < NV; ++k) sum[k] += m.adj_sign[t] * phi[k];
      }
      for (int k = 0; k < NV; ++k) st.residual[c * NV + k] = -sum[k];
    });
  }

  void extensive_predict(const std::vector<int>& tau, double dt, const int* it, int64_t n) {
    each(it, n, [&](int c) {  // :218-223
      const double dt_window = dt * static_cast<double>(1 << tau[c]);
      for (int k = 0; k < NV; ++k)
        st.W_pred[c * NV + k] = st.W[c * NV + k] + dt_window * st.residual[c * NV + k];
    });
  }

  void intensive_predict(const int* it, int64_t n) {  // :225-227
    each(it, n, [&](int c) {
      for (int k = 0; k < NV; ++k) st.w_pred[c * NV + k] = st.W_pred[c * NV + k] / m.vol[c];
    });
  }

  void extensive_correct(const int* it, int64_t n) {  // :229-231
    each(it, n, [&](int c) {
      for (int k = 0; k < NV; ++k) st.W[c * NV + k] += st.residual[c * NV + k];
    });
  }

  void intensive_correct(const std::vector<int>& tau, const int* it, int64_t n, int front) {
    each(it, n, [&](int c) {  // :233-241
      ORC_ASSERT(st.committed_front[c] + (1 << tau[c]) == front,
                 "a correction must close exactly one window");
      for (int k = 0; k < NV; ++k) st.w[c * NV + k] = st.W[c * NV + k] / m.vol[c];
      st.committed_front[c] = front;
    });
  }

  void finalize_cells(const int* it, int64_t n) {  // :243-245
    each(it, n, [&](int c) {
      for (int k = 0; k < NV; ++k) st.w[c * NV + k] = st.W[c * NV + k] / m.vol[c];
    });
  }

  void compute_dt_max(double cfl, double dt_cap, const int* it, int64_t n) {  // :247-254
    each(it, n, [&](int c) {
      const double speed = ph.speed(&st.w[c * NV]);
      st.dt_max[c] = speed > 0.0 ? smin(dt_cap, cfl * m.chl[c] / speed) : dt_cap;
    });
  }

  void classify_cells(double dt_min, int theta_max, const int* it, int64_t n) {  // :256-258
    each(it, n, [&](int c) { st.raw_level[c] = classify_raw(st.dt_max[c], dt_min, theta_max); });
  }

  double min_dt(const int* it, int64_t n) {  // :260-264 (sequential: order-free min)
    double lowest = std::numeric_limits<double>::infinity();
    for (int64_t i = 0; i < n; ++i) lowest = smin(lowest, st.dt_max[it[i]]);
    return lowest;
  }

  bool finite_state(const int* it, int64_t n) {  // :266-271
    for (int64_t i = 0; i < n; ++i) {
      const int c = it[i];
      for (int k = 0; k < NV; ++k)
        if (!std::isfinite(st.w[c * NV + k]) || !std::isfinite(st.W[c * NV + k])) return false;
    }
    return true;
  }
};

// --- the sequential driver (reference.cpp) -----------------------------------
struct Options {
  int theta_max = 3;
  double cfl = 0.9;
  double dt_cap = 1.0;
};

std::vector<int> iota_items(int n) {
  std::vector<int> v(n);
  std::iota(v.begin(), v.end(), 0);
  return v;
}

template <class P>
struct Driver {
  const Mesh& m;
  State& st;
  const P& ph;
  Pool& pool;
  Kernels<P> k{m, st, ph, pool};

  struct ActiveSets {  // reference.cpp:21-39
    std::vector<Items> cells, faces;
  };

  ActiveSets build_active_sets(const IterationPlan& plan) {
    ActiveSets sets;
    const int theta = plan.theta();
    sets.cells.resize(theta + 1);
    sets.faces.resize(theta + 1);
    for (int l = 0; l <= theta; ++l) {
      for (int c = 0; c < m.nc; ++c)
        if (plan.levels.tau[c] <= l) sets.cells[l].push_back(c);
      for (int f = 0; f < m.nf; ++f)
        if (plan.face_cadence[f] <= l) sets.faces[l].push_back(f);
    }
    return sets;
  }

  void corrector_phase(const IterationPlan& plan, double dt, const Items& cells,
                       const Items& faces, const Items& fringe, int front) {  // :41-54
    const auto& tau = plan.levels.tau;
    const int nc = static_cast<int>(cells.size()), nf = static_cast<int>(faces.size());
    k.stage_predicted(tau, cells.data(), nc, front);
    k.stage_interpolated(tau, fringe.data(), fringe.size(), front, kCorrector);
    k.green_gauss_gradient(cells.data(), nc, front, kCorrector);
    k.limit_gradients(cells.data(), nc, front, kCorrector);
    k.reconstruct_faces(faces.data(), nf, front, kCorrector);
    k.riemann_correct(plan.face_cadence, dt, faces.data(), nf, front);
    ledger(faces.data(), nf);
    k.flux_sum_correct(tau, plan.face_cadence, cells.data(), nc, front);
    k.extensive_correct(cells.data(), nc);
    k.intensive_correct(tau, cells.data(), nc, front);
  }

  void predictor_phase(const IterationPlan& plan, double dt, const Items& cells,
                       const Items& faces, const Items& fringe, int front) {  // :56-70
    const auto& tau = plan.levels.tau;
    const int nc = static_cast<int>(cells.size()), nf = static_cast<int>(faces.size());
    k.stage_committed(cells.data(), nc, front);
    k.stage_interpolated(tau, fringe.data(), fringe.size(), front, kPredictor);
    k.green_gauss_gradient(cells.data(), nc, front, kPredictor);
    k.limit_gradients(cells.data(), nc, front, kPredictor);
    k.reset_windows(faces.data(), nf, front);
    k.reconstruct_faces(faces.data(), nf, front, kPredictor);
    k.riemann_predict(faces.data(), nf, front);
    k.flux_sum_predict(cells.data(), nc, front);
    k.extensive_predict(tau, dt, cells.data(), nc);
    k.intensive_predict(cells.data(), nc);
  }

  // Conservation ledger (new; the reference keeps none): a transmissive
  // face's slot adds +int_substep to its left cell's residual sum
  // (flux_sum_correct, kernels.cpp:204-216: tau_c == cadence_f on a boundary
  // face, so the substep integral is the one read), i.e. takes it out of the
  // domain. Summed over the active boundary faces of every corrector, in
  // ascending face id, compensated (TwoSum).
  double bflux[8] = {}, bcomp[8] = {};
  void ledger(const int* faces, int64_t nf) {
    for (int64_t i = 0; i < nf; ++i) {
      const int f = faces[i];
      if (m.resolved_right(f) >= 0) continue;
      for (int k = 0; k < P::NV; ++k) {
        const double b = st.int_substep[f * P::NV + k];
        const double s = bflux[k] + b, bb = s - bflux[k];
        bcomp[k] += (bflux[k] - (s - bb)) + (b - bb);
        bflux[k] = s;
      }
    }
  }

  void totals(double* out) const {  // state.cpp:40-44 (ascending id, per component)
    for (int j = 0; j < P::NV; ++j) {
      double total = 0.0;
      for (int c = 0; c < m.nc; ++c) total += st.W[c * P::NV + j];
      out[j] = total;
    }
  }

  Record make_record(const IterationPlan& plan, double t_start) const {  // :74-87
    Record r;
    std::memset(&r, 0, sizeof r);
    r.iteration = st.iteration;
    r.t_start = t_start;
    r.dt = plan.levels.dt;
    r.theta = plan.theta();
    r.advance = plan.levels.dt * static_cast<double>(plan.subiterations());
    totals(r.total_extensive);
    for (int k = 0; k < P::NV; ++k) r.boundary_flux[k] = bflux[k] + bcomp[k];
    r.cost_ratio = plan.levels.cost_ratio();
    r.n_levels = static_cast<int32_t>(plan.levels.cells_of_level.size());
    for (int l = 0; l < r.n_levels && l < 16; ++l)
      r.level_cells[l] = static_cast<int64_t>(plan.levels.cells_of_level[l].size());
    r.nv = P::NV;
    return r;
  }

  IterationPlan plan_iteration(const Options& opt) {  // :89-98
    const Items cells = iota_items(m.nc);
    k.compute_dt_max(opt.cfl, opt.dt_cap, cells.data(), m.nc);
    const double dt_min = k.min_dt(cells.data(), m.nc);
    require(std::isfinite(dt_min) && dt_min > 0.0, "integrate: stable step collapsed");
    k.classify_cells(dt_min, opt.theta_max, cells.data(), m.nc);
    std::vector<int> tau = st.raw_level;
    smooth_to_fixpoint(m, tau);
    return build_iteration_plan(m, make_level_map(std::move(tau), dt_min));
  }

  Record run_iteration(const IterationPlan& plan) {  // :100-129
    const int theta = plan.theta();
    const double dt = plan.levels.dt;
    const Items all_cells = iota_items(m.nc);
    const Items all_faces = iota_items(m.nf);
    const ActiveSets sets = build_active_sets(plan);
    const double t_start = st.t0;
    const Items none;
    reset_fronts(st);
    for (int k = 0; k < 8; ++k) bflux[k] = bcomp[k] = 0.0;
    const int subiterations = plan.subiterations();
    for (int s = 1; s <= subiterations; ++s) {
      const int level = subiteration_level(s, theta);
      const int front = s - 1;
      const Items& fringe = level < theta ? plan.fringe[level] : none;
      if (s > 1) corrector_phase(plan, dt, sets.cells[level], sets.faces[level], fringe, front);
      predictor_phase(plan, dt, sets.cells[level], sets.faces[level], fringe, front);
    }
    corrector_phase(plan, dt, all_cells, all_faces, none, subiterations);
    if (!k.finite_state(all_cells.data(), m.nc))
      throw std::runtime_error("integrate: solution diverged to a non-finite state");
    k.finalize_cells(all_cells.data(), m.nc);
    st.t0 = t_start + dt * static_cast<double>(subiterations);
    st.iteration += 1;
    return make_record(plan, t_start);
  }

  std::vector<Record> plain_heun(const Options& opt, int iterations) {  // :144-199
    require(iterations >= 0, "integrate: negative iteration count");
    const Items cells = iota_items(m.nc), faces = iota_items(m.nf);
    const std::vector<int> tau(m.nc, 0), cad(m.nf, 0);
    const int nc = m.nc, nf = m.nf;
    std::vector<Record> out;
    for (int i = 0; i < iterations; ++i) {
      k.compute_dt_max(opt.cfl, opt.dt_cap, cells.data(), nc);
      const double dt = k.min_dt(cells.data(), nc);
      require(std::isfinite(dt) && dt > 0.0, "integrate: stable step collapsed");
      reset_fronts(st);
      k.stage_committed(cells.data(), nc, 0);
      k.green_gauss_gradient(cells.data(), nc, 0, kPredictor);
      k.limit_gradients(cells.data(), nc, 0, kPredictor);
      k.reset_windows(faces.data(), nf, 0);
      k.reconstruct_faces(faces.data(), nf, 0, kPredictor);
      k.riemann_predict(faces.data(), nf, 0);
      k.flux_sum_predict(cells.data(), nc, 0);
      k.extensive_predict(tau, dt, cells.data(), nc);
      k.intensive_predict(cells.data(), nc);
      k.stage_predicted(tau, cells.data(), nc, 1);
      k.green_gauss_gradient(cells.data(), nc, 1, kCorrector);
      k.limit_gradients(cells.data(), nc, 1, kCorrector);
      k.reconstruct_faces(faces.data(), nf, 1, kCorrector);
      for (int q = 0; q < 8; ++q) bflux[q] = bcomp[q] = 0.0;
      k.riemann_correct(cad, dt, faces.data(), nf, 1);
      ledger(faces.data(), nf);
      k.flux_sum_correct(tau, cad, cells.data(), nc, 1);
      k.extensive_correct(cells.data(), nc);
      k.intensive_correct(tau, cells.data(), nc, 1);
      if (!k.finite_state(cells.data(), nc))
        throw std::runtime_error("integrate: solution diverged to a non-finite state");
      k.finalize_cells(cells.data(), nc);
      Record r;
      std::memset(&r, 0, sizeof r);
      r.iteration = ++st.iteration;
      r.t_start = st.t0;
      r.dt = dt;
      r.theta = 0;
      r.advance = dt;
      totals(r.total_extensive);
      for (int q = 0; q < P::NV; ++q) r.boundary_flux[q] = bflux[q] + bcomp[q];
      r.cost_ratio = 1.0;
      r.n_levels = 1;
      r.level_cells[0] = m.nc;
      r.nv = P::NV;
      st.t0 += dt;
      out.push_back(r);
    }
    return out;
  }
};

// --- the task-shaped driver (the reference's STF engine shape) ----------------
// CPU baseline only: the same Euler / scalar kernels
// driven the way TaskEngine::run_iteration drives the reference's
// (taskgen.cpp:348-523, 525-661): the mesh is cut into computational elements
// (CEs; ce.cpp:19-64 -- here equal chunks of the id or a Morton order), each CE's cells are split
// into inner cells (every neighbour in the CE) and border cells, its faces into
// intra-CE faces and inter-CE pair groups, all binned by level; every phase is
// emitted as the reference's four passes of per-CE tasks -- (0) stage border
// cells, (1) stage inner, gradient + limiter inner, then border, (2) window
// reset / reconstruction / Riemann on intra faces and on pair groups, (3) flux
// sums and updates, inner then border -- whose data accesses on four kinds of
// handles (inner[ce], border[ce], faces[ce], pair[a,b]) are declared read or
// write, and a sequential-task-flow runtime (runtime.cpp's model: a task waits
// for the last writer of what it reads, and for every reader since the last
// writer of what it writes) runs them on worker threads with NO barrier between
// kernels, phases or subiterations. Every kernel call is the barrier driver's,
// on a CE's item list, so the state is bitwise the sequential driver's; only
// the ledger's compensated sum takes its terms in (phase, CE) order.
struct TaskGraph {
  struct Task {
    std::function<void()> fn;
    std::vector<int> succ;
    int ndeps = 0;
  };
  struct Handle {
    int last_writer = -1;
    std::vector<int> readers;
  };
  std::vector<Task> tasks;
  std::vector<Handle> handles;

  explicit TaskGraph(int nhandles) : handles(nhandles) {}

  void add(std::function<void()> fn, const std::vector<int>& reads, const std::vector<int>& writes) {
    const int id = static_cast<int>(tasks.size());
    std::vector<int> deps;
    for (int h : reads) {
      if (handles[h].last_writer >= 0) deps.push_back(handles[h].last_writer);
      handles[h].readers.push_back(id);
    }
    for (int h : writes) {
      Handle& hd = handles[h];
      if (hd.last_writer >= 0) deps.push_back(hd.last_writer);
      for (int r : hd.readers)
        if (r != id) deps.push_back(r);
      hd.last_writer = id;
      hd.readers.clear();
    }
    std::sort(deps.begin(), deps.end());
    deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
    tasks.emplace_back();
    tasks.back().fn = std::move(fn);
    tasks.back().ndeps = static_cast<int>(deps.size());
    for (int d : deps) tasks[d].succ.push_back(id);
  }

  void run(int threads) {
    const int n = static_cast<int>(tasks.size());
    std::vector<int> left(n);
    std::deque<int> ready;
    for (int i = 0; i < n; ++i) {
      left[i] = tasks[i].ndeps;
      if (left[i] == 0) ready.push_back(i);
    }
    std::mutex mu;
    std::condition_variable cv;
    int done = 0;
    std::exception_ptr err;
    auto worker = [&] {
      std::unique_lock<std::mutex> lk(mu);
      for (;;) {
        cv.wait(lk, [&] { return !ready.empty() || done == n || err; });
        if (done == n || err) return;
        const int t = ready.front();
        ready.pop_front();
        lk.unlock();
        std::exception_ptr e;
        try {
          tasks[t].fn();
        } catch (...) {
          e = std::current_exception();
        }
        lk.lock();
        if (e && !err) err = e;
        ++done;
        int woke = 0;
        for (int sidx : tasks[t].succ)
          if (--left[sidx] == 0) {
            ready.push_back(sidx);
            ++woke;
          }
        if (done == n || err) cv.notify_all();
        else if (woke > 1) cv.notify_all();
        else if (woke == 1) cv.notify_one();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < std::max(1, threads); ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
  }
};

// The CE decomposition of a mesh (static: ce.cpp:19-90's role): compact
// equal-size CEs; a cell is a border cell when a neighbour lies in another CE; a face
// belongs to its CE (both sides inside, or a boundary face) or to the pair of
// CEs it joins.
struct CeDecomp {
  int n_ce = 1, chunk = 1;
  std::vector<int> ce_id;  // cell -> CE
  std::vector<uint8_t> is_border;
  std::vector<std::vector<int>> inner_raw, border_raw, intra_raw, pair_raw;
  std::vector<std::pair<int, int>> pairs;
  std::vector<std::vector<int>> ce_pairs, ce_nbrs;
};
inline std::shared_ptr<CeDecomp> build_decomp(const Mesh& m, int nce_signed, Pool& pool) {
  auto dc = std::make_shared<CeDecomp>();
  const int nce = std::abs(nce_signed);
  const int n_ce = dc->n_ce = std::max(1, std::min(nce, m.nc));
  const int chunk = dc->chunk = (m.nc + n_ce - 1) / n_ce;
  dc->ce_id.resize(m.nc);
  if (nce_signed > 0) {
    // equal chunks of the id order: on a lattice-ordered mesh these are sheets
    // across the graded direction, so every CE holds its share of every level
    // (the level-cost balance DistDriver::repartition aims at, exchange.cpp:598-603)
    for (int c = 0; c < m.nc; ++c) dc->ce_id[c] = c / chunk;
  } else {
    // compact CEs (the role of partition.cpp's region growing): equal chunks of
    // the cells in Morton order of their centroids
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = m.cen[a];
    for (int c = 0; c < m.nc; ++c)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], m.cen[3 * static_cast<size_t>(c) + a]);
        hi[a] = std::max(hi[a], m.cen[3 * static_cast<size_t>(c) + a]);
      }
    // one scale for every axis, so that the curve's cells are cubes in space
    double ext = 0.0;
    for (int a = 0; a < 3; ++a) ext = std::max(ext, hi[a] - lo[a]);
    const double scale = ext > 0.0 ? 1048575.0 / ext : 0.0;
    auto spread = [](uint64_t v) {
      v &= 0x1fffffull;
      v = (v | v << 32) & 0x1f00000000ffffull;
      v = (v | v << 16) & 0x1f0000ff0000ffull;
      v = (v | v << 8) & 0x100f00f00f00f00full;
      v = (v | v << 4) & 0x10c30c30c30c30c3ull;
      v = (v | v << 2) & 0x1249249249249249ull;
      return v;
    };
    std::vector<std::pair<uint64_t, int>> key(m.nc);
    pool.run(m.nc, [&](int64_t b, int64_t e) {
      for (int64_t c = b; c < e; ++c) {
        uint64_t k = 0;
        for (int a = 0; a < 3; ++a)
          k |= spread(static_cast<uint64_t>((m.cen[3 * c + a] - lo[a]) * scale)) << a;
        key[c] = {k, static_cast<int>(c)};
      }
    });
    std::sort(key.begin(), key.end());
    for (int i = 0; i < m.nc; ++i) dc->ce_id[key[i].second] = i / chunk;
  }
  auto ce_of = [&](int c) { return dc->ce_id[c]; };
  dc->is_border.assign(m.nc, 0);
  pool.run(m.nc, [&](int64_t b, int64_t e) {
    for (int64_t c = b; c < e; ++c)
      for (int t = m.adj_off[c]; t < m.adj_off[c + 1]; ++t) {
        const int nb = m.adj_nb[t];
        if (nb >= 0 && ce_of(nb) != ce_of(static_cast<int>(c))) dc->is_border[c] = 1;
      }
  });
  dc->inner_raw.resize(n_ce);
  dc->border_raw.resize(n_ce);
  dc->intra_raw.resize(n_ce);
  for (int c = 0; c < m.nc; ++c) (dc->is_border[c] ? dc->border_raw : dc->inner_raw)[ce_of(c)].push_back(c);
  std::map<std::pair<int, int>, int> pair_index;
  for (int f = 0; f < m.nf; ++f) {
    const int a = ce_of(m.fl[f]);
    const int r = m.resolved_right(f);
    const int b = r >= 0 ? ce_of(r) : a;
    if (a == b) {
      dc->intra_raw[a].push_back(f);
    } else {
      const std::pair<int, int> key{std::min(a, b), std::max(a, b)};
      auto it = pair_index.find(key);
      if (it == pair_index.end()) {
        it = pair_index.emplace(key, static_cast<int>(dc->pairs.size())).first;
        dc->pairs.push_back(key);
        dc->pair_raw.emplace_back();
      }
      dc->pair_raw[it->second].push_back(f);
    }
  }
  dc->ce_pairs.resize(n_ce);
  dc->ce_nbrs.resize(n_ce);
  for (int q = 0; q < static_cast<int>(dc->pairs.size()); ++q) {
    dc->ce_pairs[dc->pairs[q].first].push_back(q);
    dc->ce_pairs[dc->pairs[q].second].push_back(q);
    dc->ce_nbrs[dc->pairs[q].first].push_back(dc->pairs[q].second);
    dc->ce_nbrs[dc->pairs[q].second].push_back(dc->pairs[q].first);
  }
  return dc;
}

template <class P>
struct TaskDriver {
  Driver<P>& d;
  const CeDecomp& decomp;
  Pool serial{1};
  Kernels<P> ks{d.m, d.st, d.ph, serial};

  // Items of one iteration (taskgen.cpp build_iteration_items): per CE the
  // cells sorted by level (prefix = "tau <= l"), inner and border apart; intra
  // faces and pair groups sorted by cadence; the fringe lists split likewise.
  struct Sorted {
    std::vector<int> items;
    std::vector<int> upto;  // upto[l] = |{items : level <= l}|
    const int* data() const { return items.data(); }
    int64_t count(int level) const { return upto.empty() ? 0 : upto[std::min<size_t>(level, upto.size() - 1)]; }
  };
  static Sorted sort_by_level(const std::vector<int>& items, const std::vector<int>& level_of, int theta) {
    Sorted s;
    s.upto.assign(theta + 1, 0);
    for (int x : items) ++s.upto[level_of[x]];
    std::vector<int> at(theta + 1, 0);
    for (int l = 1; l <= theta; ++l) at[l] = at[l - 1] + s.upto[l - 1];
    s.items.resize(items.size());
    std::vector<int> cur = at;
    for (int x : items) s.items[cur[level_of[x]]++] = x;
    for (int l = 0; l <= theta; ++l) s.upto[l] = cur[l];
    return s;
  }

  Record run_iteration(const IterationPlan& plan, int threads) {
    const Mesh& m = d.m;
    State& st = d.st;
    const int theta = plan.theta();
    const double dt = plan.levels.dt;
    const std::vector<int>& tau = plan.levels.tau;
    const std::vector<int>& cad = plan.face_cadence;
    const CeDecomp& dc = decomp;
    const int n_ce = dc.n_ce;
    auto ce_of = [&](int c) { return dc.ce_id[c]; };
    const std::vector<uint8_t>& is_border = dc.is_border;
    const auto& inner_raw = dc.inner_raw;
    const auto& border_raw = dc.border_raw;
    const auto& intra_raw = dc.intra_raw;
    const auto& pair_raw = dc.pair_raw;
    const auto& pairs = dc.pairs;
    const auto& ce_pairs = dc.ce_pairs;
    const auto& ce_nbrs = dc.ce_nbrs;
    const int n_pair = static_cast<int>(pairs.size());
    std::vector<Sorted> inner(n_ce), border(n_ce), intra(n_ce), pfaces(n_pair);
    d.pool.run(n_ce, [&](int64_t b, int64_t e) {
      for (int64_t q = b; q < e; ++q) {
        inner[q] = sort_by_level(inner_raw[q], tau, theta);
        border[q] = sort_by_level(border_raw[q], tau, theta);
        intra[q] = sort_by_level(intra_raw[q], cad, theta);
      }
    });
    d.pool.run(n_pair, [&](int64_t b, int64_t e) {
      for (int64_t q = b; q < e; ++q) pfaces[q] = sort_by_level(pair_raw[q], cad, theta);
    });
    // fringe[level] split by CE and class
    std::vector<std::vector<std::vector<int>>> fr_in(theta), fr_bd(theta);
    for (int l = 0; l < theta; ++l) {
      fr_in[l].resize(n_ce);
      fr_bd[l].resize(n_ce);
      for (int c : plan.fringe[l]) (is_border[c] ? fr_bd[l] : fr_in[l])[ce_of(c)].push_back(c);
    }

    // --- handles and the ledger's partial sums
    auto h_inner = [&](int q) { return q; };
    auto h_border = [&](int q) { return n_ce + q; };
    auto h_faces = [&](int q) { return 2 * n_ce + q; };
    auto h_pair = [&](int q) { return 3 * n_ce + q; };
    TaskGraph g(3 * n_ce + n_pair);
    const int subiterations = plan.subiterations();
    const int n_corr = subiterations;  // correctors: subiterations - 1 inside the sweep + the trailing one
    std::vector<double> led(static_cast<size_t>(n_corr) * n_ce * 2 * P::NV, 0.0);

    const double t_start = st.t0;
    reset_fronts(st);
    int corr_index = 0;
    const std::vector<int> none;  // outlives the tasks that hold a reference to it
    auto emit_phase = [&](bool corr, int level, int front, int ci) {
      const int phase = corr ? kCorrector : kPredictor;
      // pass 0: border cells staged first (taskgen.cpp:360-383)
      for (int q = 0; q < n_ce; ++q) {
        const int64_t nb = border[q].count(level);
        const std::vector<int>& fb = level < theta ? fr_bd[level][q] : none;
        if (nb == 0 && fb.empty()) continue;
        g.add([this, &tau, &border, &fb, q, nb, front, corr, phase] {
          if (corr) ks.stage_predicted(tau, border[q].data(), nb, front);
          else ks.stage_committed(border[q].data(), nb, front);
          ks.stage_interpolated(tau, fb.data(), fb.size(), front, phase);
        }, {}, {h_border(q)});
      }
      // pass 1: inner staging, gradients and limiter inner, then border (:385-421)
      for (int q = 0; q < n_ce; ++q) {
        const int64_t ni = inner[q].count(level), nb = border[q].count(level);
        const std::vector<int>& fi = level < theta ? fr_in[level][q] : none;
        if (ni > 0 || !fi.empty())
          g.add([this, &tau, &inner, &fi, q, ni, front, corr, phase] {
            if (corr) ks.stage_predicted(tau, inner[q].data(), ni, front);
            else ks.stage_committed(inner[q].data(), ni, front);
            ks.stage_interpolated(tau, fi.data(), fi.size(), front, phase);
          }, {}, {h_inner(q)});
        if (ni > 0)
          g.add([this, &inner, q, ni, front, phase] {
            ks.green_gauss_gradient(inner[q].data(), ni, front, phase);
            ks.limit_gradients(inner[q].data(), ni, front, phase);
          }, {h_border(q)}, {h_inner(q)});
        if (nb > 0) {
          std::vector<int> reads{h_inner(q)};
          for (int o : ce_nbrs[q]) reads.push_back(h_border(o));
          g.add([this, &border, q, nb, front, phase] {
            ks.green_gauss_gradient(border[q].data(), nb, front, phase);
            ks.limit_gradients(border[q].data(), nb, front, phase);
          }, reads, {h_border(q)});
        }
      }
      // pass 2: faces -- intra-CE, then the pair groups, emitted once (:423-474)
      for (int q = 0; q < n_ce; ++q) {
        const int64_t nf = intra[q].count(level);
        if (nf == 0) continue;
        double* part = corr ? &led[(static_cast<size_t>(ci) * n_ce + q) * 2 * P::NV] : nullptr;
        g.add([this, &cad, &intra, q, nf, front, corr, phase, dt, part] {
          const int* f = intra[q].data();
          if (!corr) ks.reset_windows(f, nf, front);
          ks.reconstruct_faces(f, nf, front, phase);
          if (corr) {
            ks.riemann_correct(cad, dt, f, nf, front);
            for (int64_t i = 0; i < nf; ++i) {  // the ledger's terms of this CE and phase
              if (d.m.resolved_right(f[i]) >= 0) continue;
              for (int k = 0; k < P::NV; ++k) {
                const double b = d.st.int_substep[f[i] * P::NV + k];
                const double sum = part[k] + b, bb = sum - part[k];
                part[P::NV + k] += (part[k] - (sum - bb)) + (b - bb);
                part[k] = sum;
              }
            }
          } else {
            ks.riemann_predict(f, nf, front);
          }
        }, {h_inner(q), h_border(q)}, {h_faces(q)});
      }
      for (int q = 0; q < n_pair; ++q) {
        const int64_t nf = pfaces[q].count(level);
        if (nf == 0) continue;
        g.add([this, &cad, &pfaces, q, nf, front, corr, phase, dt] {
          const int* f = pfaces[q].data();
          if (!corr) ks.reset_windows(f, nf, front);
          ks.reconstruct_faces(f, nf, front, phase);
          if (corr) ks.riemann_correct(cad, dt, f, nf, front);
          else ks.riemann_predict(f, nf, front);
        }, {h_border(pairs[q].first), h_border(pairs[q].second)}, {h_pair(q)});
      }
      // pass 3: flux sums and updates, inner then border (:476-513)
      for (int q = 0; q < n_ce; ++q) {
        const int64_t ni = inner[q].count(level), nb = border[q].count(level);
        auto update = [this, &tau, &cad, front, corr, dt](const int* c, int64_t n) {
          if (corr) {
            ks.flux_sum_correct(tau, cad, c, n, front);
            ks.extensive_correct(c, n);
            ks.intensive_correct(tau, c, n, front);
          } else {
            ks.flux_sum_predict(c, n, front);
            ks.extensive_predict(tau, dt, c, n);
            ks.intensive_predict(c, n);
          }
        };
        if (ni > 0)
          g.add([&inner, q, ni, update] { update(inner[q].data(), ni); }, {h_faces(q)}, {h_inner(q)});
        if (nb > 0) {
          std::vector<int> reads{h_faces(q)};
          for (int pq : ce_pairs[q]) reads.push_back(h_pair(pq));
          g.add([&border, q, nb, update] { update(border[q].data(), nb); }, reads, {h_border(q)});
        }
      }
    };
    // the phase order of run_iteration (reference.cpp:100-129)
    for (int s = 1; s <= subiterations; ++s) {
      const int level = subiteration_level(s, theta);
      const int front = s - 1;
      if (s > 1) emit_phase(true, level, front, corr_index++);
      emit_phase(false, level, front, -1);
    }
    emit_phase(true, theta, subiterations, corr_index++);
    n_tasks = static_cast<int64_t>(g.tasks.size());
    g.run(threads);

    // ledger: the partials in (phase, CE) order, compensated
    for (int k = 0; k < 8; ++k) d.bflux[k] = d.bcomp[k] = 0.0;
    for (size_t i = 0; i < led.size() / (2 * P::NV); ++i)
      for (int k = 0; k < P::NV; ++k)
        for (int part = 0; part < 2; ++part) {
          const double b = led[i * 2 * P::NV + part * P::NV + k];
          const double sum = d.bflux[k] + b, bb = sum - d.bflux[k];
          d.bcomp[k] += (d.bflux[k] - (sum - bb)) + (b - bb);
          d.bflux[k] = sum;
        }
    const Items all_cells = iota_items(m.nc);
    if (!d.k.finite_state(all_cells.data(), m.nc))
      throw std::runtime_error("integrate: solution diverged to a non-finite state");
    d.k.finalize_cells(all_cells.data(), m.nc);
    st.t0 = t_start + dt * static_cast<double>(subiterations);
    st.iteration += 1;
    return d.make_record(plan, t_start);
  }
  int64_t n_tasks = 0;
};

// --- type-erased solver -------------------------------------------------------
enum Model { kAdvection = 0, kBurgers = 1, kEuler = 2 };

struct Solver {
  const Mesh* m;
  int model;
  int nv;
  Advection2D adv{};
  Burgers2D bur{};
  Euler3D eul{};
  State st;
  Options opt;
  IterationPlan plan;
  bool has_plan = false;
  std::unique_ptr<Pool> pool = std::make_unique<Pool>(1);
  std::shared_ptr<CeDecomp> decomp;  // task driver: the CE decomposition of the last n_ce
  int decomp_nce = 0;
};

template <class F>
auto with_physics(Solver& s, F&& f) {
  switch (s.model) {
    case kAdvection: {
      Driver<Advection2D> d{*s.m, s.st, s.adv, *s.pool};
      return f(d);
    }
    case kBurgers: {
      Driver<Burgers2D> d{*s.m, s.st, s.bur, *s.pool};
      return f(d);
    }
    default: {
      Driver<Euler3D> d{*s.m, s.st, s.eul, *s.pool};
      return f(d);
    }
  }
}

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

double* darr(State& st, const std::string& n) {
  if (n == "w") return st.w.data();
  if (n == "W") return st.W.data();
  if (n == "W_pred") return st.W_pred.data();
  if (n == "w_pred") return st.w_pred.data();
  if (n == "w_eval") return st.w_eval.data();
  if (n == "grad") return st.grad.data();
  if (n == "residual") return st.residual.data();
  if (n == "dt_max") return st.dt_max.data();
  if (n == "face_wL") return st.face_wL.data();
  if (n == "face_wR") return st.face_wR.data();
  if (n == "phi_pred") return st.phi_pred.data();
  if (n == "int_substep") return st.int_substep.data();
  if (n == "int_window") return st.int_window.data();
  return nullptr;
}

size_t dsize(const State& st, const Mesh& m, const std::string& n) {
  if (n == "dt_max") return m.nc;
  if (n == "grad") return size_t(m.nc) * st.nv * 3;
  if (n.rfind("face_", 0) == 0 || n == "phi_pred" || n == "int_substep" || n == "int_window")
    return size_t(m.nf) * st.nv;
  return size_t(m.nc) * st.nv;
}

std::vector<int>* iarr(State& st, const std::string& n) {
  if (n == "raw_level") return &st.raw_level;
  if (n == "committed_front") return &st.committed_front;
  if (n == "staged_front") return &st.staged_front;
  if (n == "face_staged") return &st.face_staged;
  if (n == "face_front") return &st.face_front;
  return nullptr;
}

}  // namespace oracle

using namespace oracle;

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// Mesh from reference-layout arrays (Face/Cell of mesh.hpp:26-39, Vec3).
// Builds the ascending-face-id CSR adjacency and checks closure.
int orc_mesh_create_masked(int dim, int nc, int nf, const double* vol, const double* cen,
                           const double* chl, const int* fl, const int* fr, const int* fp,
                           const double* fn, const double* fa, const double* fc,
                           const uint8_t* closure_mask, void** out);

int orc_mesh_create(int dim, int nc, int nf, const double* vol, const double* cen,
                    const double* chl, const int* fl, const int* fr, const int* fp,
                    const double* fn, const double* fa, const double* fc, void** out) {
  return orc_mesh_create_masked(dim, nc, nf, vol, cen, chl, fl, fr, fp, fn, fa, fc, nullptr, out);
}

int orc_mesh_create_masked(int dim, int nc, int nf, const double* vol, const double* cen,
                           const double* chl, const int* fl, const int* fr, const int* fp,
                           const double* fn, const double* fa, const double* fc,
                           const uint8_t* closure_mask, void** out) {
  return guard([&] {
    require(nc >= 0 && nf >= 0, "mesh: negative counts");
    auto m = std::make_unique<Mesh>();
    m->dim = dim;
    m->nc = nc;
    m->nf = nf;
    m->vol.assign(vol, vol + nc);
    m->cen.assign(cen, cen + 3 * size_t(nc));
    m->chl.assign(chl, chl + nc);
    m->fl.assign(fl, fl + nf);
    m->fr.assign(fr, fr + nf);
    m->fp.assign(fp, fp + nf);
    m->fn.assign(fn, fn + 3 * size_t(nf));
    m->fa.assign(fa, fa + nf);
    m->fc.assign(fc, fc + 3 * size_t(nf));
    build_adjacency(*m);
    check_closure(*m, closure_mask);
    *out = m.release();
  });
}

void orc_mesh_free(void* m) { delete static_cast<Mesh*>(m); }

int orc_mesh_nadj(void* mp) { return static_cast<Mesh*>(mp)->adj_off.back(); }

void orc_mesh_adjacency(void* mp, int* off, int* face, int* nb, double* sign) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  std::copy(m.adj_off.begin(), m.adj_off.end(), off);
  std::copy(m.adj_face.begin(), m.adj_face.end(), face);
  std::copy(m.adj_nb.begin(), m.adj_nb.end(), nb);
  std::copy(m.adj_sign.begin(), m.adj_sign.end(), sign);
}

// model: "advection" | "burgers" | "euler". a = advection vector / Burgers
// direction (normalised, physics.cpp:7-21); gamma for Euler.
int orc_solver_create(void* mesh, const char* model, double ax, double ay, double gamma,
                      void** out) {
  return guard([&] {
    auto s = std::make_unique<Solver>();
    s->m = static_cast<Mesh*>(mesh);
    const std::string name = model;
    if (name == "advection") {
      s->model = kAdvection;
      s->nv = 1;
      s->adv = {ax, ay};
    } else if (name == "burgers") {
      const double len = std::sqrt(ax * ax + ay * ay);
      require(len > 0.0, "physics: burgers direction must be nonzero");
      s->model = kBurgers;
      s->nv = 1;
      s->bur = {ax / len, ay / len};
    } else if (name == "euler") {
      require(gamma > 1.0, "physics: gamma must exceed 1");
      s->model = kEuler;
      s->nv = 5;
      s->eul.gamma = gamma;
      s->eul.gm1 = gamma - 1.0;
    } else {
      require(false, "physics: unknown model");
    }
    s->st.init(*s->m, s->nv);
    *out = s.release();
  });
}

void orc_solver_free(void* s) { delete static_cast<Solver*>(s); }

void orc_set_threads(void* sp, int n) {
  auto* s = static_cast<Solver*>(sp);
  s->pool = std::make_unique<Pool>(n);
}

void orc_set_options(void* sp, int theta_max, double cfl, double dt_cap) {
  auto* s = static_cast<Solver*>(sp);
  s->opt = {theta_max, cfl, dt_cap};
}

// st.init + w <- values + sync_extensive (state.cpp:61-68).
int orc_init_values(void* sp, const double* w) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    s->st.init(*s->m, s->nv);
    std::copy(w, w + size_t(s->m->nc) * s->nv, s->st.w.begin());
    sync_extensive(*s->m, s->st);
  });
}

int orc_get(void* sp, const char* name, void* out) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    if (double* d = darr(s->st, name)) {
      std::memcpy(out, d, dsize(s->st, *s->m, name) * sizeof(double));
    } else if (auto* i = iarr(s->st, name)) {
      std::memcpy(out, i->data(), i->size() * sizeof(int));
    } else {
      throw std::invalid_argument(std::string("orc_get: unknown array ") + name);
    }
  });
}

int orc_set(void* sp, const char* name, const void* in) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    if (double* d = darr(s->st, name)) {
      std::memcpy(d, in, dsize(s->st, *s->m, name) * sizeof(double));
    } else if (auto* i = iarr(s->st, name)) {
      std::memcpy(i->data(), in, i->size() * sizeof(int));
    } else {
      throw std::invalid_argument(std::string("orc_set: unknown array ") + name);
    }
  });
}

void orc_time(void* sp, double* t0, int* iteration) {
  auto* s = static_cast<Solver*>(sp);
  *t0 = s->st.t0;
  *iteration = s->st.iteration;
}

void orc_set_time(void* sp, double t0, int iteration) {
  auto* s = static_cast<Solver*>(sp);
  s->st.t0 = t0;
  s->st.iteration = iteration;
}

int orc_plan_iteration(void* sp) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    s->plan = with_physics(*s, [&](auto& d) { return d.plan_iteration(s->opt); });
    s->has_plan = true;
  });
}

int orc_inject_plan(void* sp, const int* tau, double dt) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    std::vector<int> t(tau, tau + s->m->nc);
    s->plan = build_iteration_plan(*s->m, make_level_map(std::move(t), dt));
    s->has_plan = true;
  });
}

void orc_plan_info(void* sp, int* theta, double* dt, double* cost_ratio, int64_t* cells_per_level,
                   int64_t* faces_per_cadence, int64_t* fringe_per_level) {
  auto* s = static_cast<Solver*>(sp);
  const IterationPlan& p = s->plan;
  *theta = p.theta();
  *dt = p.levels.dt;
  *cost_ratio = p.levels.cost_ratio();
  for (int l = 0; l <= p.theta(); ++l) {
    cells_per_level[l] = int64_t(p.levels.cells_of_level[l].size());
    faces_per_cadence[l] = int64_t(p.faces_of_cadence[l].size());
  }
  for (int l = 0; l < p.theta(); ++l) fringe_per_level[l] = int64_t(p.fringe[l].size());
}

void orc_plan_lists(void* sp, int* tau, int* cadence, int* cells_flat, int* faces_flat,
                    int* fringe_flat) {
  auto* s = static_cast<Solver*>(sp);
  const IterationPlan& p = s->plan;
  std::copy(p.levels.tau.begin(), p.levels.tau.end(), tau);
  std::copy(p.face_cadence.begin(), p.face_cadence.end(), cadence);
  for (const auto& v : p.levels.cells_of_level) cells_flat = std::copy(v.begin(), v.end(), cells_flat);
  for (const auto& v : p.faces_of_cadence) faces_flat = std::copy(v.begin(), v.end(), faces_flat);
  for (const auto& v : p.fringe) fringe_flat = std::copy(v.begin(), v.end(), fringe_flat);
}

int orc_run_iteration(void* sp, Record* rec) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    require(s->has_plan, "run_iteration: no plan");
    *rec = with_physics(*s, [&](auto& d) { return d.run_iteration(s->plan); });
  });
}

int orc_integrate(void* sp, int n, Record* recs) {  // reference.cpp:131-142
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    require(n >= 0, "integrate: negative iteration count");
    for (int i = 0; i < n; ++i) {
      s->plan = with_physics(*s, [&](auto& d) { return d.plan_iteration(s->opt); });
      s->has_plan = true;
      recs[i] = with_physics(*s, [&](auto& d) { return d.run_iteration(s->plan); });
    }
  });
}

// reference_integrate with run_iteration through the task-shaped driver
// (TaskEngine::integrate, taskgen.cpp:663-672): n_ce computational elements,
// the solver's thread count as workers. tasks_out: tasks of the last iteration.
int orc_integrate_tasks(void* sp, int n, int n_ce, int threads, Record* recs, int64_t* tasks_out) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    require(n >= 0, "integrate: negative iteration count");
    require(n_ce != 0 && threads >= 1, "integrate_tasks: n_ce must be non-zero and threads positive");
    if (!s->decomp || s->decomp_nce != n_ce) {
      s->decomp = build_decomp(*s->m, n_ce, *s->pool);
      s->decomp_nce = n_ce;
    }
    for (int i = 0; i < n; ++i) {
      s->plan = with_physics(*s, [&](auto& d) { return d.plan_iteration(s->opt); });
      s->has_plan = true;
      recs[i] = with_physics(*s, [&](auto& d) {
        using PH = std::remove_cv_t<std::remove_reference_t<decltype(d.ph)>>;
        TaskDriver<PH> td{d, *s->decomp};
        Record r = td.run_iteration(s->plan, threads);
        if (tasks_out) *tasks_out = td.n_tasks;
        return r;
      });
    }
  });
}

int orc_plain_heun(void* sp, int n, Record* recs) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    const auto r = with_physics(*s, [&](auto& d) { return d.plain_heun(s->opt, n); });
    std::copy(r.begin(), r.end(), recs);
  });
}

int orc_kernel(void* sp, const char* name, const int* items, int n, int front, int phase,
               const int* tau_in, const int* cadence_in, double dt, double cfl, double dt_cap,
               int theta_max, double* scalar_out) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    const Mesh& m = *s->m;
    std::vector<int> tau, cad;
    if (tau_in) tau.assign(tau_in, tau_in + m.nc);
    if (cadence_in) cad.assign(cadence_in, cadence_in + m.nf);
    const std::string k = name;
    with_physics(*s, [&](auto& d) {
      auto& K = d.k;
      if (k == "stage_committed") K.stage_committed(items, n, front);
      else if (k == "stage_predicted") K.stage_predicted(tau, items, n, front);
      else if (k == "stage_interpolated") K.stage_interpolated(tau, items, n, front, phase);
      else if (k == "green_gauss_gradient") K.green_gauss_gradient(items, n, front, phase);
      else if (k == "limit_gradients") K.limit_gradients(items, n, front, phase);
      else if (k == "reset_windows") K.reset_windows(items, n, front);
      else if (k == "reconstruct_faces") K.reconstruct_faces(items, n, front, phase);
      else if (k == "riemann_predict") K.riemann_predict(items, n, front);
      else if (k == "riemann_correct") K.riemann_correct(cad, dt, items, n, front);
      else if (k == "flux_sum_predict") K.flux_sum_predict(items, n, front);
      else if (k == "flux_sum_correct") K.flux_sum_correct(tau, cad, items, n, front);
      else if (k == "extensive_predict") K.extensive_predict(tau, dt, items, n);
      else if (k == "intensive_predict") K.intensive_predict(items, n);
      else if (k == "extensive_correct") K.extensive_correct(items, n);
      else if (k == "intensive_correct") K.intensive_correct(tau, items, n, front);
      else if (k == "finalize_cells") K.finalize_cells(items, n);
      else if (k == "compute_dt_max") K.compute_dt_max(cfl, dt_cap, items, n);
      else if (k == "classify_cells") K.classify_cells(dt, theta_max, items, n);
      else if (k == "min_dt") *scalar_out = K.min_dt(items, n);
      else if (k == "finite_state") *scalar_out = K.finite_state(items, n) ? 1.0 : 0.0;
      else if (k == "reset_fronts") reset_fronts(s->st);
      else throw std::invalid_argument("orc_kernel: unknown kernel " + k);
      return 0;
    });
  });
}

double orc_minmod(double x, double y) { return minmod(x, y); }

// Flux through one face for a single state pair (nv values each).
int orc_rusanov(void* sp, const double* wl, const double* wr, const double* n, double* out) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    switch (s->model) {
      case kAdvection: rusanov(s->adv, wl, wr, n, out); break;
      case kBurgers: rusanov(s->bur, wl, wr, n, out); break;
      default: rusanov(s->eul, wl, wr, n, out); break;
    }
  });
}

int orc_subiteration_level(int s, int theta, int* out) {
  return guard([&] { *out = subiteration_level(s, theta); });
}

int orc_classify_raw(double dt_max, double dt_min, int theta_max, int* out) {
  return guard([&] { *out = classify_raw(dt_max, dt_min, theta_max); });
}

int orc_smooth_to_fixpoint(void* mp, int* tau) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  std::vector<int> t(tau, tau + m.nc);
  const int sweeps = smooth_to_fixpoint(m, t);
  std::copy(t.begin(), t.end(), tau);
  return sweeps;
}

int orc_cost_shares(const double* cell_shares, int n, double* cost_out, double* ratio_out) {
  return guard([&] {
    std::vector<double> v(cell_shares, cell_shares + n);
    const auto c = cost_shares_from_cell_shares(v);
    std::copy(c.begin(), c.end(), cost_out);
    *ratio_out = cost_ratio_from_cell_shares(v);
  });
}

}  // extern "C"
