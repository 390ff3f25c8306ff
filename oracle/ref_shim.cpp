// TEST INFRASTRUCTURE ONLY — not part of the product.
//
// C-ABI shim over the UNMODIFIED reference library (arxiv/paper_1704_01144,
// `proj/core`), compiled from its sources where they lie under
// /root/reference by oracle/Makefile into oracle/_ref/libtafv_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load it, and only as the checker. It exposes the reference's own entry
// points (proj/core/include/tafv/reference.hpp:35-58, kernels.hpp:31-111,
// levels.hpp:24-63, mesh.hpp:67, state.hpp:52-79) to ctypes so the oracle
// restatement and the golden fixtures can be pinned against the real thing.
// The reference is scalar 2D only (physics.hpp:11-28, mesh.cpp:303).

#include <cstdint>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tafv/ce.hpp"
#include "tafv/kernels.hpp"
#include "tafv/partition.hpp"
#include "tafv/runtime.hpp"
#include "tafv/taskgen.hpp"
#include "tafv/levels.hpp"
#include "tafv/mesh.hpp"
#include "tafv/physics.hpp"
#include "tafv/reference.hpp"
#include "tafv/state.hpp"

using namespace tafv;

namespace {

thread_local std::string g_err;

// Status codes shared with the product C-ABI (include/tafv_gpu.h).
enum { kOk = 0, kInvalid = 1, kLogic = 2, kRuntime = 3 };

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalid;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return kLogic;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return kRuntime;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kRuntime;
  }
}

struct Record {  // layout mirrors tafv_record in include/tafv_gpu.h
  int32_t iteration;
  int32_t theta;
  double t_start, dt, advance, cost_ratio;
  double total_extensive[8];
  int64_t level_cells[16];
  int32_t n_levels;
  int32_t nv;
  double boundary_flux[8];  // not kept by the reference: zero
};

void fill(Record* out, const IterationRecord& r) {
  std::memset(out, 0, sizeof *out);
  out->iteration = r.iteration;
  out->theta = r.theta;
  out->t_start = r.t_start;
  out->dt = r.dt;
  out->advance = r.advance;
  out->cost_ratio = r.cost_ratio;
  out->total_extensive[0] = r.total_extensive;
  out->n_levels = static_cast<int32_t>(r.level_cells.size());
  for (size_t l = 0; l < r.level_cells.size() && l < 16; ++l) out->level_cells[l] = r.level_cells[l];
  out->nv = 1;
}

struct Solver {
  const Mesh* mesh;
  SolverState st;
  SolverOptions opt;
  IterationPlan plan;
  bool has_plan = false;
};

std::vector<double>* darr(SolverState& st, const std::string& n) {
  if (n == "w") return &st.w;
  if (n == "W") return &st.W;
  if (n == "W_pred") return &st.W_pred;
  if (n == "w_pred") return &st.w_pred;
  if (n == "w_eval") return &st.w_eval;
  if (n == "gx") return &st.gx;
  if (n == "gy") return &st.gy;
  if (n == "residual") return &st.residual;
  if (n == "dt_max") return &st.dt_max;
  if (n == "face_wL") return &st.face_wL;
  if (n == "face_wR") return &st.face_wR;
  if (n == "phi_pred") return &st.phi_pred;
  if (n == "int_substep") return &st.int_substep;
  if (n == "int_window") return &st.int_window;
  return nullptr;
}

std::vector<int>* iarr(SolverState& st, const std::string& n) {
  if (n == "raw_level") return &st.raw_level;
  if (n == "committed_front") return &st.committed_front;
  if (n == "staged_front") return &st.staged_front;
  if (n == "face_staged") return &st.face_staged;
  if (n == "face_front") return &st.face_front;
  return nullptr;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- mesh --------------------------------------------------------------------

int ref_mesh_generate(int dim, int nx, int ny, const double* domain /*lo.x lo.y hi.x hi.y*/,
                      int periodic_x, int periodic_y, int n_regions,
                      const double* region_boxes /*4 per region*/, const int* region_scales,
                      void** out) {
  return guard([&] {
    MeshSpec spec;
    spec.dim = dim;
    spec.nx = nx;
    spec.ny = ny;
    spec.domain = {{domain[0], domain[1]}, {domain[2], domain[3]}};
    spec.periodic_x = periodic_x != 0;
    spec.periodic_y = periodic_y != 0;
    for (int r = 0; r < n_regions; ++r) {
      RefinementRegion reg;
      reg.bbox = {{region_boxes[4 * r], region_boxes[4 * r + 1]},
                  {region_boxes[4 * r + 2], region_boxes[4 * r + 3]}};
      reg.scale = region_scales[r];
      spec.regions.push_back(reg);
    }
    *out = new Mesh(generate_mesh(spec));
  });
}

void ref_mesh_free(void* m) { delete static_cast<Mesh*>(m); }

void ref_mesh_counts(void* mp, int* nc, int* nf, int* nadj) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  *nc = m.cell_count();
  *nf = m.face_count();
  *nadj = static_cast<int>(m.adj_face.size());
}

uint64_t ref_mesh_hash(void* mp) { return static_cast<Mesh*>(mp)->hash(); }

// Mesh::save (mesh.cpp:345-382) to a file.
int ref_mesh_save(void* mp, const char* path) {
  return guard([&] {
    std::ofstream os(path, std::ios::binary);
    static_cast<Mesh*>(mp)->save(os);
    if (!os) throw std::runtime_error("ref_mesh_save: write failed");
  });
}

// cell: nc x 4 (cx, cy, volume, char_length); face_i: nf x 3 (left, right,
// partner); face_d: nf x 5 (nx, ny, area, fcx, fcy).
void ref_mesh_export(void* mp, double* cell, int* face_i, double* face_d, int* adj_off,
                     int* adj_face, int* adj_nb, double* adj_sign) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  for (int c = 0; c < m.cell_count(); ++c) {
    cell[4 * c] = m.cells[c].centroid.x;
    cell[4 * c + 1] = m.cells[c].centroid.y;
    cell[4 * c + 2] = m.cells[c].volume;
    cell[4 * c + 3] = m.cells[c].char_length;
  }
  for (int f = 0; f < m.face_count(); ++f) {
    const Face& fa = m.faces[f];
    face_i[3 * f] = fa.left;
    face_i[3 * f + 1] = fa.right;
    face_i[3 * f + 2] = fa.periodic_partner;
    face_d[5 * f] = fa.normal.x;
    face_d[5 * f + 1] = fa.normal.y;
    face_d[5 * f + 2] = fa.area;
    face_d[5 * f + 3] = fa.centroid.x;
    face_d[5 * f + 4] = fa.centroid.y;
  }
  std::copy(m.adj_offset.begin(), m.adj_offset.end(), adj_off);
  std::copy(m.adj_face.begin(), m.adj_face.end(), adj_face);
  std::copy(m.adj_neighbor.begin(), m.adj_neighbor.end(), adj_nb);
  std::copy(m.adj_sign.begin(), m.adj_sign.end(), adj_sign);
}

// --- solver ------------------------------------------------------------------

int ref_solver_create(void* mesh, const char* model, double ax, double ay, void** out) {
  return guard([&] {
    auto* s = new Solver;
    s->mesh = static_cast<Mesh*>(mesh);
    s->opt.model = parse_flux_model(model, {ax, ay});
    s->st.init(*s->mesh);
    *out = s;
  });
}

void ref_solver_free(void* s) { delete static_cast<Solver*>(s); }

void ref_set_options(void* sp, int theta_max, double cfl, double dt_cap) {
  auto* s = static_cast<Solver*>(sp);
  s->opt.theta_max = theta_max;
  s->opt.cfl = cfl;
  s->opt.dt_cap = dt_cap;
}

int ref_init_gaussian(void* sp, double base, double amp, double cx, double cy, double sigma) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    GaussianProfile p;
    p.base = base;
    p.amplitude = amp;
    p.center = {cx, cy};
    p.sigma = sigma;
    init_gaussian(*s->mesh, s->st, p);
  });
}

int ref_init_uniform(void* sp, double v) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    init_uniform(*s->mesh, s->st, v);
  });
}

// st.init + w <- given + sync_extensive (the tests' "st.w = {...}; sync_extensive").
int ref_init_values(void* sp, const double* w) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    s->st.init(*s->mesh);
    std::copy(w, w + s->mesh->cell_count(), s->st.w.begin());
    sync_extensive(*s->mesh, s->st);
  });
}

int ref_get(void* sp, const char* name, void* out) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    if (auto* d = darr(s->st, name)) {
      std::memcpy(out, d->data(), d->size() * sizeof(double));
    } else if (auto* i = iarr(s->st, name)) {
      std::memcpy(out, i->data(), i->size() * sizeof(int));
    } else {
      throw std::invalid_argument(std::string("ref_get: unknown array ") + name);
    }
  });
}

int ref_set(void* sp, const char* name, const void* in) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    if (auto* d = darr(s->st, name)) {
      std::memcpy(d->data(), in, d->size() * sizeof(double));
    } else if (auto* i = iarr(s->st, name)) {
      std::memcpy(i->data(), in, i->size() * sizeof(int));
    } else {
      throw std::invalid_argument(std::string("ref_set: unknown array ") + name);
    }
  });
}

void ref_time(void* sp, double* t0, int* iteration) {
  auto* s = static_cast<Solver*>(sp);
  *t0 = s->st.t0;
  *iteration = s->st.iteration;
}

// save_snapshot (state.cpp:77-91) to a file.
int ref_snapshot_save(void* sp, const char* path) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    std::ofstream os(path);
    save_snapshot(os, *s->mesh, s->st);
  });
}

// compare_snapshots(Snapshot::load(a), Snapshot::load(b)) (state.cpp:93-132).
int ref_snapshot_compare(const char* a, const char* b, double* worst) {
  return guard([&] {
    std::ifstream ia(a), ib(b);
    *worst = compare_snapshots(Snapshot::load(ia), Snapshot::load(ib));
  });
}

double ref_total_extensive(void* sp) { return static_cast<Solver*>(sp)->st.total_extensive(); }

// --- plan --------------------------------------------------------------------

int ref_plan_iteration(void* sp) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    s->plan = plan_iteration(*s->mesh, s->st, s->opt);
    s->has_plan = true;
  });
}

int ref_inject_plan(void* sp, const int* tau, double dt) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    std::vector<int> t(tau, tau + s->mesh->cell_count());
    s->plan = build_iteration_plan(*s->mesh, make_level_map(std::move(t), dt));
    s->has_plan = true;
  });
}

// info: theta, dt, cost_ratio, counts per level / cadence / fringe (<=16 each).
void ref_plan_info(void* sp, int* theta, double* dt, double* cost_ratio, int64_t* cells_per_level,
                   int64_t* faces_per_cadence, int64_t* fringe_per_level) {
  auto* s = static_cast<Solver*>(sp);
  const IterationPlan& p = s->plan;
  *theta = p.theta();
  *dt = p.levels.dt;
  *cost_ratio = p.levels.cost_ratio();
  for (int l = 0; l <= p.theta(); ++l) {
    cells_per_level[l] = static_cast<int64_t>(p.levels.cells_of_level[l].size());
    faces_per_cadence[l] = static_cast<int64_t>(p.faces_of_cadence[l].size());
  }
  for (int l = 0; l < p.theta(); ++l) fringe_per_level[l] = static_cast<int64_t>(p.fringe[l].size());
}

// Flattened lists in level order (ascending ids within each level).
void ref_plan_lists(void* sp, int* tau, int* cadence, int* cells_flat, int* faces_flat,
                    int* fringe_flat) {
  auto* s = static_cast<Solver*>(sp);
  const IterationPlan& p = s->plan;
  std::copy(p.levels.tau.begin(), p.levels.tau.end(), tau);
  std::copy(p.face_cadence.begin(), p.face_cadence.end(), cadence);
  for (const auto& v : p.levels.cells_of_level) cells_flat = std::copy(v.begin(), v.end(), cells_flat);
  for (const auto& v : p.faces_of_cadence) faces_flat = std::copy(v.begin(), v.end(), faces_flat);
  for (const auto& v : p.fringe) fringe_flat = std::copy(v.begin(), v.end(), fringe_flat);
}

int ref_run_iteration(void* sp, Record* rec) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    if (!s->has_plan) throw std::invalid_argument("ref_run_iteration: no plan");
    fill(rec, run_iteration(*s->mesh, s->st, s->opt, s->plan));
  });
}

int ref_integrate(void* sp, int n, Record* recs) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    const auto r = reference_integrate(*s->mesh, s->st, s->opt, n);
    for (size_t i = 0; i < r.size(); ++i) fill(&recs[i], r[i]);
  });
}

// The reference's own task-parallel CPU path (TaskEngine::integrate,
// taskgen.cpp:663-675) over `workers` single-lane workers and `ces`
// computation elements, prio scheduler, packing on (the survey's baseline
// shape).
int ref_taskengine_integrate(void* sp, int n, int workers, int ces, Record* recs) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    RuntimeOptions ro;
    ro.worker_lanes.assign(workers, 1);
    ro.scheduler = "prio";
    ro.probe_period_ms = 0.0;
    ro.record_trace = false;
    Runtime rt(ro);
    const Partition part =
        make_partition(*s->mesh, 1, ces, std::vector<int64_t>(s->mesh->cell_count(), 1));
    const CESet set = build_ces(*s->mesh, part);
    TaskgenOptions topt;
    topt.packing = true;
    TaskEngine engine(*s->mesh, set, rt, topt);
    const auto r = engine.integrate(s->st, s->opt, n);
    for (size_t i = 0; i < r.size(); ++i) fill(&recs[i], r[i]);
  });
}

int ref_plain_heun(void* sp, int n, Record* recs) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    const auto r = plain_heun_integrate(*s->mesh, s->st, s->opt, n);
    for (size_t i = 0; i < r.size(); ++i) fill(&recs[i], r[i]);
  });
}

// --- kernels over explicit item lists (kernels.hpp:31-111) ---------------------

int ref_kernel(void* sp, const char* name, const int* items, int n, int front, int phase,
               const int* tau_in, const int* cadence_in, double dt, double cfl, double dt_cap,
               int theta_max, double* scalar_out) {
  return guard([&] {
    auto* s = static_cast<Solver*>(sp);
    const Mesh& m = *s->mesh;
    SolverState& st = s->st;
    const kernels::Items it(items, static_cast<size_t>(n));
    const Phase ph = phase == 0 ? Phase::corrector : Phase::predictor;
    std::vector<int> tau, cad;
    if (tau_in) tau.assign(tau_in, tau_in + m.cell_count());
    if (cadence_in) cad.assign(cadence_in, cadence_in + m.face_count());
    const std::string k = name;
    if (k == "stage_committed") kernels::stage_committed(st, it, front);
    else if (k == "stage_predicted") kernels::stage_predicted(st, tau, it, front);
    else if (k == "stage_interpolated") kernels::stage_interpolated(st, tau, it, front, ph);
    else if (k == "green_gauss_gradient") kernels::green_gauss_gradient(m, st, it, front, ph);
    else if (k == "limit_gradients") kernels::limit_gradients(m, st, it, front, ph);
    else if (k == "reset_windows") kernels::reset_windows(m, st, it, front);
    else if (k == "reconstruct_faces") kernels::reconstruct_faces(m, st, it, front, ph);
    else if (k == "riemann_predict") kernels::riemann_predict(m, s->opt.model, st, it, front);
    else if (k == "riemann_correct") kernels::riemann_correct(m, s->opt.model, st, cad, dt, it, front);
    else if (k == "flux_sum_predict") kernels::flux_sum_predict(m, st, it, front);
    else if (k == "flux_sum_correct") kernels::flux_sum_correct(m, st, tau, cad, it, front);
    else if (k == "extensive_predict") kernels::extensive_predict(st, tau, dt, it);
    else if (k == "intensive_predict") kernels::intensive_predict(m, st, it);
    else if (k == "extensive_correct") kernels::extensive_correct(st, it);
    else if (k == "intensive_correct") kernels::intensive_correct(m, st, tau, it, front);
    else if (k == "finalize_cells") kernels::finalize_cells(m, st, it);
    else if (k == "compute_dt_max") kernels::compute_dt_max(m, s->opt.model, st, cfl, dt_cap, it);
    else if (k == "classify_cells") kernels::classify_cells(st, dt, theta_max, it);
    else if (k == "min_dt") *scalar_out = kernels::min_dt(st, it);
    else if (k == "finite_state") *scalar_out = kernels::finite_state(st, it) ? 1.0 : 0.0;
    else if (k == "reset_fronts") reset_fronts(st);
    else throw std::invalid_argument("ref_kernel: unknown kernel " + k);
  });
}

// --- pure functions ----------------------------------------------------------

double ref_minmod(double x, double y) { return minmod(x, y); }

int ref_rusanov(const char* model, double ax, double ay, double wl, double wr, double nx, double ny,
                double* out) {
  return guard([&] { *out = rusanov(parse_flux_model(model, {ax, ay}), wl, wr, {nx, ny}); });
}

int ref_subiteration_level(int s, int theta, int* out) {
  return guard([&] { *out = subiteration_level(s, theta); });
}

int ref_classify_raw(double dt_max, double dt_min, int theta_max, int* out) {
  return guard([&] { *out = classify_raw(dt_max, dt_min, theta_max); });
}

void ref_smooth_to_fixpoint(void* mp, int* tau) {
  const Mesh& m = *static_cast<Mesh*>(mp);
  std::vector<int> t(tau, tau + m.cell_count());
  smooth_to_fixpoint(m, t);
  std::copy(t.begin(), t.end(), tau);
}

int ref_cost_shares(const double* cell_shares, int n, double* cost_out, double* ratio_out) {
  return guard([&] {
    std::vector<double> v(cell_shares, cell_shares + n);
    const auto c = cost_shares_from_cell_shares(v);
    std::copy(c.begin(), c.end(), cost_out);
    *ratio_out = cost_ratio_from_cell_shares(v);
  });
}

}  // extern "C"
