// Host runtime of the B200 LTS finite-volume hot path: implements the C ABI
// of include/tafv_gpu.h (the drop-in boundary for plan_iteration /
// run_iteration / reference_integrate, proj/core/include/tafv/reference.hpp).
//
// Data layout in HBM:
//   * cells renumbered once at upload by a 63-bit Morton key of the centroid
//     (locality for the neighbour gathers); faces grouped by their left cell;
//     the per-cell CSR slots keep the reference order (ascending ORIGINAL
//     face id, mesh.cpp:241-271) so every sum associates exactly as the
//     reference's;
//   * FP64 AoS rows per cell/face ([N][nv] state, [N][nv][3] gradients,
//     [F][nv] face fluxes) so a gathered neighbour is one contiguous run;
//   * per-iteration plan: int8 levels/cadences and level-sorted index lists
//     whose prefixes are the active sets of every subiteration level.
// One plan read-back per iteration (theta, counts, dt: the host needs theta
// to size the 2^theta sweep), stored by a kernel into mapped pinned memory
// (store_plan); everything else stays on the device.
//
// Streams: the library stream `st` carries the plan and sweep graphs; a
// shard's halo exchange runs on a high-priority comm stream `cst` under the
// next phase's K1/K2 over the deep cells / interior faces (halo_rows /
// halo_join); run_batch adds copy streams per lane and a twin handle (a
// second state over the same mesh arrays) so two inputs advance
// concurrently.

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <cstdint>
#include <chrono>
#include <cstring>
#include <array>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "comm.h"
#include "kernels.cuh"
#include "meshprep.cuh"
#include "shard.h"
#include "tafv_gpu.h"

using namespace tafv;

namespace {

thread_local std::string g_create_error;

// NVTX ranges mirroring the reference's TraceRecord kinds (runtime.hpp:110-118):
// one per plan, sweep and (direct launches) phase; free without a tool.
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

struct Error {
  int code;
  std::string what;
};

void check_cuda(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw Error{TAFV_ECUDA, std::string(where) + ": " + cudaGetErrorString(e)};
}
#define CK(x) check_cuda((x), #x)
#ifndef TAFV_K1_BRICK_MAX_RAGGED
#define TAFV_K1_BRICK_MAX_RAGGED 0.25  // auto mode: largest share of bricks that may not fit the stage
#endif
#ifndef TAFV_K1_BRICK_AUTO
#define TAFV_K1_BRICK_AUTO (4 << 20)  // auto threshold (owned cells) of the brick K1
#endif

void require(bool cond, const char* what) {
  if (!cond) throw Error{TAFV_EINVAL, what};
}

template <class T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

inline uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

int subiteration_level(int s, int theta) {  // levels.cpp:10-16
  for (int tmp = theta; tmp > 0; --tmp)
    if ((s - 1) % (1 << tmp) == 0) return tmp;
  return 0;
}

}  // namespace

struct tafv_gpu {
  int device = 0;
  cudaStream_t st = nullptr;
  std::string err;
  int model = TAFV_EULER, nv = 5, dim = 3;
  PhysParams pp{};
  tafv_physics phys{};  // as created (in-place rebuilds)
  bool levels_made = false;  // a plan has been made (device tau = the last plan's levels)
  // DistDriver's repartition_every (exchange.hpp:140-143): tafv_gpu_iterate
  // repartitions shards by level cost every `rep_every` iterations
  const tafv_mesh_view* rep_mesh = nullptr;
  int rep_every = 0, rep_axis = 0;
  double rep_ms = 0.0;  // wall time of the last repartition
  int N = 0, F = 0, M = 0;
  bool periodic = false;
  int sms = 148;
  std::vector<int> cperm, fperm;  // internal -> original
  std::vector<double> vol_host;

  // device mesh
  double *vol = nullptr, *ivol = nullptr, *cen = nullptr, *chl = nullptr, *fcen = nullptr;
  bool deg6 = false;  // every cell has exactly 6 CSR slots (hex meshes): fast path
  // Launch shapes: grid-stride kernels with a fixed, occupancy-sized grid
  // (graph mode) so the captured sweep of a theta never changes.
  bool use_graph = true;
  // theta (x2 + kernel_timing) -> instantiated sweep graph. With kernel
  // timing on, event-record nodes bracket every hot kernel INSIDE the graph,
  // so the instrumented replay runs exactly like the timed one.
  struct GraphRec {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
    std::vector<int> kinds;
    std::vector<std::array<long long, 3>> items;
    std::vector<cudaEvent_t> evs;  // 2 per timed kernel
  };
  std::map<int, GraphRec> graphs;
  GraphRec* cap = nullptr;            // record being captured
  GraphRec* pending_graph = nullptr;  // replayed graph whose events await collection
  cudaGraphExec_t plan_graph = nullptr;   // plan_iteration for plan_opt
  bool plan_graph_on = true;
  tafv_options plan_opt{};
  int64_t plan_graph_launches = 0;
  bool capturing = false;
  int grid_k1 = 0, grid_k2 = 0, grid_k3 = 0;
  int plan_nkeys = 0;
  // single-domain plans fuse the ilogb classification into the first Jacobi
  // sweep, so raw levels live only in registers; get_array("raw_level")
  // recomputes them (k_classify, the same function) while this is set
  bool raw_lazy = false;
  int* adj_off = nullptr;
  int* adj_face = nullptr;  // [M] face id, ~f on the face's right side
  int* adj_nb = nullptr;    // [M] neighbour cell or -1
  int2* lr = nullptr;
  int* rcf = nullptr;
  double4* geo = nullptr;
  double4* sgeo = nullptr;  // hex fast path per-slot geometry (see MeshDev)
  double4* sdx = nullptr;
  double4* fdx = nullptr;  // see MeshDev::fdx
  bool slot_geo = true;
  bool slot_n = true, slot_dx = true;  // A/B: per-slot normals / limiter offsets individually
  // identity-phase K1 in Morton bricks (k_grad_limit<.., true>): -1 auto
  // (meshes of >= 4M cells, where it measured -2 % K1; +3-4 % on 0.26M / 1M)
  int k1_tile = -1;
  bool use_k1_tile() const { return deg6 && (k1_tile > 0 || (k1_tile < 0 && n_own >= (4 << 20))); }
  // identity-phase K1 with the brick's streams bulk-copied into shared memory
  // (k_grad_limit_brick; per-face geometry windows): -1 auto, 0 off, 1 on
  int k1_brick = -1;
  // the bricks' static structures (BrickDev; mesh data, shared with the twin),
  // built on first use, and the cells left to k_grad_limit (ragged bricks, tail)
  unsigned short* brick_idx = nullptr;
  int* brick_halo = nullptr;
  double *brick_geo = nullptr, *brick_fcen = nullptr;
  int4* brick_info = nullptr;
  long long brick_entries = 0;
  int *brick_rest = nullptr, *brick_nrest = nullptr;  // list and its count (device)
  int brick_rest_host = 0, brick_ragged = 0, nbricks = 0;
  bool brick_declined = false;  // auto mode found too many ragged bricks on this mesh
  BrickDev brick_dev() const { return BrickDev{brick_idx, brick_info, brick_halo, brick_geo, brick_fcen}; }
  int grid_k1b = 0;
  bool use_k1_brick() const {
    return deg6 && brick_idx && (k1_brick > 0 || (k1_brick < 0 && n_own >= (TAFV_K1_BRICK_AUTO)));
  }
  bool face_dx = true;
  int dl_stream = 1;  // run_batch downloads on the copy stream (0: on the library stream, A/B)
  // run_batch lanes: a twin handle sharing this one's (read-only) mesh arrays
  // with its own state, plan, graphs and streams, so two independent inputs
  // advance concurrently and each fills the other's idle SMs (small level
  // phases, kernel tails). Owned; rebuilt after any set_flag.
  tafv_gpu* twin = nullptr;
  bool owns_mesh = true;
  int batch_lanes = 2;
  int *d_cperm = nullptr, *d_fperm = nullptr;
  int* d_cinv = nullptr;  // original -> internal cell (iterate_host's chunked copies; lazily built)
  std::vector<cudaEvent_t> ev_gather;  // iterate_host: per-chunk "gathered for download" events
  // device state
  double *w = nullptr, *W = nullptr, *wp = nullptr, *grad = nullptr;
  size_t gs = 0;  // gradient row stride in doubles (padded, see GradRow)
  size_t fs = 0;  // face-integral row stride in doubles (padded, see FaceRow)
  double *phi = nullptr, *isub = nullptr, *iwin = nullptr;
  uint8_t* ialias = nullptr;  // [F] see StateDev::ialias
  // conservation ledger (k_ledger): transmissive faces touching owned cells
  int NB = 0;
  int* bface = nullptr;       // [NB] internal face ids (mesh, shared with the twin)
  double* bsum = nullptr;     // [NB][nv] running outflow since the last trailing corrector
  DD* lpart = nullptr;        // [nv][nblk_led] per-block partials of the outflow (k_ledger_reduce)
  int nblk_led = 1;
  cudaStream_t lst = nullptr; // side stream of the ledger kernels
  cudaEvent_t ev_led_fork = nullptr, ev_led = nullptr;
  bool led_pending = false;
  bool iwin_alias = true;
  int8_t *tau = nullptr, *cad = nullptr, *raw = nullptr, *tmpa = nullptr, *tmpb = nullptr;
  int skip_top_lists = 1;         // flag "skip_top_lists": do not write the top level's list entries
  bool lists_skip_top = false;    // the last plan's lists lack their top-level segment
  uint8_t* sweep_tile = nullptr;  // [sweep][cell tile] marks of the Jacobi sweeps (k_level_sweep)
  int sweep_marks = 1;            // flag "sweep_marks": skip the tiles no level change can reach
  uint8_t* fflag = nullptr;
  double *dtmax = nullptr, *blockmin = nullptr;
  unsigned* dt_ticket = nullptr;  // last-block ticket of k_dt_max
  int nblk_dt = 0;
  int *cell_counts = nullptr, *face_counts = nullptr;
  int ntile_c = 0, ntile_f = 0;
  int *clist = nullptr, *flist = nullptr;
  DD* partials = nullptr;
  int nblk_last = 0;
  PlanDev* dplan = nullptr;
  PlanDev* hplan = nullptr;  // pinned
  double* stage_buf = nullptr;
  size_t stage_len = 0;
  // run_batch: copy streams and double-buffered input / output staging
  cudaStream_t cin = nullptr, cout = nullptr;
  double* bin[2] = {nullptr, nullptr};
  double* bout[2] = {nullptr, nullptr};
  cudaEvent_t ev_in[2] = {}, ev_in_free[2] = {}, ev_out[2] = {}, ev_out_free[2] = {};
  std::vector<cudaEvent_t> ev_chunk;  // iterate_host: per-chunk "download landed" events
  // one-graph iteration (build_iter_graph) and its per-iteration plan copies
  cudaGraphExec_t iter_graph = nullptr;
  cudaGraphConditionalHandle iter_cond{};
  tafv_options iter_opt{};
  PlanDev* batch_plans = nullptr;  // pinned: the copies stay asynchronous
  size_t batch_cap = 0;
  cudaEvent_t ev[6] = {};  // [0,1] sweep, [2,3] plan, [4,5] whole call

  // host copy of the plan
  bool has_plan = false;
  int theta = 0;
  double dt = 0.0;
  long long ccount[kMaxLevels] = {}, fcount[kMaxLevels] = {}, frcount[kMaxLevels] = {};
  double t0 = 0.0;
  int iteration = 0;
  bool state_set = false;

  // per-kernel device timing (flag "kernel_timing"): event pairs around each
  // hot launch, summed per kind after the call's host sync.
  enum { kK1 = 0, kK2P, kK2C, kK3P, kK3C, kPlan, kNumKinds };
  bool ktime = false;
  bool klog = getenv("TAFV_KLOG") != nullptr;  // per-launch times on stderr (kernel_timing runs)
  std::vector<cudaEvent_t> evpool;
  std::vector<int> evkind;
  double kms[kNumKinds] = {};
  int64_t kcnt[kNumKinds] = {};
  int64_t kitems[kNumKinds][3] = {};  // active cells, active faces, fringe cells per kind

  // multi-GPU shard. Internal cells [0, n_deep) are owned
  // cells with no halo neighbour, [n_deep, n_own) owned cells next to the
  // halo, [n_own, n_k1) ring 1, [n_k1, N) ring 2; faces [0, F_own) touch an
  // owned cell. Single domain: n_deep = n_own = n_k1 = N, F_own = F, no comm.
  int rank = 0, nranks = 1, n_deep = 0, n_own = 0, n_k1 = 0, F_own = 0, N_global = 0;
  tafv_comm* comm = nullptr;
  std::vector<int> shard_cells;  // local original id -> global cell id
  struct Peer {
    int rank, nsend, nrecv, soff, roff;
  };
  std::vector<Peer> peers;
  int *d_send_idx = nullptr, *d_recv_idx = nullptr;
  int send_total = 0, recv_total = 0;
  double *sendbuf = nullptr, *recvbuf = nullptr;
  // shards: faces [0, F_int) are interior (both sides deep owned, or a
  // boundary face of a deep cell), [F_int, F_own) the border ones; each
  // group has its own cadence-sorted K2 list (prefixes nfi / nfb_prefix)
  int F_int = 0;
  // level-sorted exchange lists: each peer segment of the
  // send / recv lists sorted by the cells' levels in every plan, so a phase
  // at level l moves only the rows of cells with tau <= l (the rows it
  // updated); xs / xr = the plan's per-peer prefix counts, host copies
  bool xfilter = false;
  int8_t *xkey_s = nullptr, *xkey_r = nullptr;
  int *xpos_s = nullptr, *xpos_r = nullptr, *xsorted_s = nullptr, *xsorted_r = nullptr;
  int* xcounts = nullptr;  // per-segment tile counts, [2 * peers][kMaxLevels * max tiles]
  int xtile_stride = 0;
  int xs[kMaxPeers][kMaxLevels] = {}, xr[kMaxPeers][kMaxLevels] = {};
  int* filist = nullptr;
  int* fblist = nullptr;
  int* fi_counts = nullptr;
  int* fb_counts = nullptr;
  int ntile_fi = 0, ntile_fb = 0;
  int* klist = nullptr;       // K1 list of the deep cells; == clist when single domain
  int* kblist = nullptr;      // K1 list of the border cells (owned next to the halo + ring 1)
  int* k1_counts = nullptr;
  int* kb_counts = nullptr;
  int ntile_k = 0, ntile_kb = 0;
  // Halo exchange overlap: the rows a K3 just wrote leave on the comm stream
  // (`cst`, high priority) while the next phase's K1 runs over the deep
  // cells on `st`; `st` joins `ev_halo` before the border cells.
  cudaStream_t cst = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  bool halo_pending = false;
  long long gcount[kMaxLevels] = {};  // owned counts over all ranks
  bool sharded() const { return comm != nullptr; }
  // traversal direction of the next hot kernel (alternating, see k_grad_limit)
  bool alt_dir = true;
  int dir_state = 0;
  int next_dir() {
    if (!alt_dir) return 0;
    dir_state ^= 1;
    return dir_state;
  }

  // stats
  int64_t launches = 0;
  double ms[3] = {0, 0, 0};
  int grid_cap = 148 * 8;

  MeshDev mesh_dev() const {
    return MeshDev{N,    F,   vol,    ivol,   cen,  chl, adj_off, adj_face, adj_nb, lr,
                   periodic ? rcf : nullptr, geo, fcen, slot_geo && slot_n ? sgeo : nullptr,
                   slot_geo && slot_dx ? sdx : nullptr, face_dx ? fdx : nullptr};
  }
  StateDev state_dev() const {
    return StateDev{w, W, wp, grad, tau, cad, phi, isub, iwin, iwin_alias ? ialias : nullptr};
  }

  double* staging(size_t n) {
    if (n > stage_len) {
      if (stage_buf) cudaFree(stage_buf);
      stage_buf = dalloc<double>(n);
      stage_len = n;
    }
    return stage_buf;
  }

  int grid_for(long long n, int block) const {
    long long g = (n + block - 1) / block;
    if (g < 1) g = 1;
    return (int)std::min<long long>(g, grid_cap);
  }

  ~tafv_gpu() { release(); }
  // Frees every device / host resource (destructor; in-place rebuild of a
  // repartitioned shard, tafv_gpu_repartition).
  void release() {
    cudaSetDevice(device);
    delete twin;
    for (auto& g : graphs) {
      cudaGraphExecDestroy(g.second.exec);
      for (auto e : g.second.evs) cudaEventDestroy(e);
    }
    if (plan_graph) cudaGraphExecDestroy(plan_graph);
    if (batch_plans) cudaFreeHost(batch_plans);
    if (iter_graph) cudaGraphExecDestroy(iter_graph);
    if (owns_mesh) {
      void* mesh_ptrs[] = {vol, ivol, cen, chl, fcen, sgeo, sdx, fdx, adj_off, adj_face, adj_nb, lr, rcf, geo,
                           d_cperm, d_fperm, bface, brick_idx, brick_halo, brick_geo, brick_fcen, brick_info,
                           brick_rest, brick_nrest};
      for (void* p : mesh_ptrs)
        if (p) cudaFree(p);
    }
    void* ptrs[] = {w,     W,        wp,       bsum,  lpart,
                    grad, phi,   isub,     iwin,     ialias,   tau,    cad,    raw,      tmpa,    tmpb, sweep_tile,
                    fflag, dt_ticket, dtmax, blockmin, cell_counts, face_counts, clist, flist, partials, dplan,
                    stage_buf, d_send_idx, d_recv_idx, sendbuf, recvbuf, d_cinv,
                    xkey_s, xkey_r, xpos_s, xpos_r, xsorted_s, xsorted_r, xcounts,
                    klist != clist ? klist : nullptr, k1_counts, kblist, kb_counts, filist, fblist, fi_counts,
                    fb_counts};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (hplan) cudaFreeHost(hplan);
    for (int q = 0; q < 2; ++q) {
      if (bin[q]) cudaFree(bin[q]);
      if (bout[q]) cudaFree(bout[q]);
      for (cudaEvent_t e : {ev_in[q], ev_in_free[q], ev_out[q], ev_out_free[q]})
        if (e) cudaEventDestroy(e);
    }
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : evpool) cudaEventDestroy(e);
    for (auto& e : ev_chunk) cudaEventDestroy(e);
    for (auto& e : ev_gather) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
    if (cst) cudaStreamDestroy(cst);
    if (lst) cudaStreamDestroy(lst);
    if (ev_led_fork) cudaEventDestroy(ev_led_fork);
    if (ev_led) cudaEventDestroy(ev_led);
    if (ev_pack) cudaEventDestroy(ev_pack);
    if (ev_halo) cudaEventDestroy(ev_halo);
  }
};


// The compute stream waits for the halo rows in flight on the comm stream.
void halo_join(tafv_gpu& h) {
  if (!h.halo_pending) return;
  CK(cudaStreamWaitEvent(h.st, h.ev_halo, 0));
  h.halo_pending = false;
}

// The device plan into the pinned host copy by a one-block kernel (stores
// over the link into mapped memory): a copy-engine transfer here would queue
// behind any bulk device-to-host copy in flight (run_batch's downloads, a
// caller's copies) and stall the library stream for its duration.
void store_plan(tafv_gpu& h) {
  k_store_plan<<<1, 128, 0, h.st>>>(h.dplan, h.hplan);
  ++h.launches;
}

// ---- transports (comm.h) ------------------------------------------------------
namespace {

#define NK(x)                                                                        \
  do {                                                                               \
    const ncclResult_t r_ = (x);                                                     \
    if (r_ != ncclSuccess) throw Error{TAFV_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

struct NcclComm final : tafv_comm {
  ncclComm_t c = nullptr;
  NcclComm(const void* id, int rank, int n) {
    rank_count = n;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    NK(ncclCommInitRank(&c, n, uid, rank));
  }
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  bool capturable() const override { return true; }
  void allreduce_min_f64(int, double* d, int n, cudaStream_t st) override {
    NK(ncclAllReduce(d, d, n, ncclFloat64, ncclMin, c, st));
  }
  void allreduce_max_i32(int, int* d, int n, cudaStream_t st) override {
    NK(ncclAllReduce(d, d, n, ncclInt32, ncclMax, c, st));
  }
  void allreduce_sum_f64(int, double* d, int n, cudaStream_t st) override {
    NK(ncclAllReduce(d, d, n, ncclFloat64, ncclSum, c, st));
  }
  void allreduce_sum_i64(int, long long* d, int n, cudaStream_t st) override {
    NK(ncclAllReduce(d, d, n, ncclInt64, ncclSum, c, st));
  }
  void exchange(tafv_gpu& h, int bpr, cudaStream_t st, const int* scount, const int* rcount) override {
    // grouped send/recv with every peer (the slab neighbours), one launch
    NK(ncclGroupStart());
    for (size_t q = 0; q < h.peers.size(); ++q) {
      const auto& p = h.peers[q];
      const int ns = scount ? scount[q] : p.nsend, nr = rcount ? rcount[q] : p.nrecv;
      char* sb = reinterpret_cast<char*>(h.sendbuf) + (size_t)p.soff * bpr;
      char* rb = reinterpret_cast<char*>(h.recvbuf) + (size_t)p.roff * bpr;
      if (ns) NK(ncclSend(sb, (size_t)ns * bpr, ncclChar, p.rank, c, st));
      if (nr) NK(ncclRecv(rb, (size_t)nr * bpr, ncclChar, p.rank, c, st));
    }
    NK(ncclGroupEnd());
  }
};

// R in-process ranks (host threads, one stream each). Host barriers order
// the ranks; data moves by device copies on the receiver's stream after the
// producers' streams were synchronised. No device-side waiting.
struct LoopbackComm final : tafv_comm {
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<tafv_gpu*> members;
  std::vector<std::vector<double>> f64;
  std::vector<std::vector<long long>> i64;
  std::vector<std::vector<int>> i32;
  explicit LoopbackComm(int n) : members(n, nullptr), f64(n), i64(n), i32(n) { rank_count = n; }
  bool capturable() const override { return false; }
  void attach(int rank, tafv_gpu* h) override { members[rank] = h; }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == rank_count) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  template <class T, class Op>
  void allreduce(std::vector<std::vector<T>>& slots, int rank, T* d, int n, cudaStream_t st, Op op) {
    slots[rank].resize(n);
    CK(cudaMemcpyAsync(slots[rank].data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    barrier();
    std::vector<T> r = slots[0];
    for (int q = 1; q < rank_count; ++q)
      for (int i = 0; i < n; ++i) r[i] = op(r[i], slots[q][i]);
    CK(cudaMemcpyAsync(d, r.data(), n * sizeof(T), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    barrier();
  }
  void allreduce_min_f64(int rank, double* d, int n, cudaStream_t st) override {
    allreduce(f64, rank, d, n, st, [](double a, double b) { return (b < a) ? b : a; });
  }
  void allreduce_max_i32(int rank, int* d, int n, cudaStream_t st) override {
    allreduce(i32, rank, d, n, st, [](int a, int b) { return a < b ? b : a; });
  }
  void allreduce_sum_f64(int rank, double* d, int n, cudaStream_t st) override {
    allreduce(f64, rank, d, n, st, [](double a, double b) { return a + b; });
  }
  void allreduce_sum_i64(int rank, long long* d, int n, cudaStream_t st) override {
    allreduce(i64, rank, d, n, st, [](long long a, long long b) { return a + b; });
  }
  void exchange(tafv_gpu& h, int bpr, cudaStream_t st, const int* scount, const int* rcount) override {
    CK(cudaStreamSynchronize(st));  // my packed rows are in sendbuf
    barrier();
    for (size_t q = 0; q < h.peers.size(); ++q) {
      const auto& p = h.peers[q];
      const tafv_gpu& g = *members[p.rank];
      const tafv_gpu::Peer* back = nullptr;
      for (const auto& b : g.peers)
        if (b.rank == h.rank) back = &b;
      if (!back || back->nsend != p.nrecv) throw Error{TAFV_ELOGIC, "loopback: mismatched exchange lists"};
      const int nr = rcount ? rcount[q] : p.nrecv;
      if (nr)
        CK(cudaMemcpyAsync(reinterpret_cast<char*>(h.recvbuf) + (size_t)p.roff * bpr,
                           reinterpret_cast<const char*>(g.sendbuf) + (size_t)back->soff * bpr,
                           (size_t)nr * bpr, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaStreamSynchronize(st));  // peers may reuse their send buffers
    barrier();
  }
};

}  // namespace

tafv_comm* make_loopback_comm(int nranks) { return new LoopbackComm(nranks); }
tafv_comm* make_nccl_comm(const void* id, int rank, int nranks) { return new NcclComm(id, rank, nranks); }
int nccl_unique_id(void* out) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return TAFV_ENCCL;
  std::memcpy(out, &id, sizeof id);
  return TAFV_OK;
}

namespace {

// ---- mesh upload -----------------------------------------------------------
// cls (optional): per original cell 0 owned / 1 ring 1 / 2 ring 2 (shards);
// touch (optional): per original face 1 if it has an owned side.
void upload_mesh_host(tafv_gpu& h, const tafv_mesh_view& mv, const uint8_t* cls = nullptr,
                      const uint8_t* touch = nullptr) {
  const int N = mv.n_cells, F = mv.n_faces;
  require(N > 0 && F >= 0, "mesh: empty mesh");
  require(mv.dim >= 1 && mv.dim <= 3, "mesh: dim must be 1, 2 or 3");
  h.N = N;
  h.F = F;
  h.dim = mv.dim;
  for (int f = 0; f < F; ++f) {
    require(mv.face_left[f] >= 0 && mv.face_left[f] < N, "mesh: face left cell out of range");
    require(mv.face_right[f] >= -1 && mv.face_right[f] < N, "mesh: face right cell out of range");
    require(mv.face_partner[f] >= -1 && mv.face_partner[f] < F, "mesh: periodic partner out of range");
    if (mv.face_partner[f] >= 0) h.periodic = true;
  }

  // Cell order: Morton key of the centroid (ties by original id).
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int c = 0; c < N; ++c)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], mv.cell_centroid[3 * (size_t)c + d]);
      hi[d] = std::max(hi[d], mv.cell_centroid[3 * (size_t)c + d]);
    }
  // (class, Morton, id): owned cells first -- those with no halo neighbour
  // ("deep", K1 runs on them while the halo exchange is in flight), then
  // those next to the halo -- then ring 1, then ring 2.
  std::vector<uint8_t> cls4;
  if (cls) {
    cls4.resize(N);
    for (int c = 0; c < N; ++c) cls4[c] = cls[c] == 0 ? 0 : (uint8_t)(cls[c] + 1);
    for (int f = 0; f < F; ++f) {
      const int l = mv.face_left[f];
      const int r = mv.face_right[f] >= 0 ? mv.face_right[f]
                    : mv.face_partner[f] >= 0 ? mv.face_left[mv.face_partner[f]] : -1;
      if (r < 0) continue;
      if (cls[l] == 0 && cls[r] != 0) cls4[l] = 1;
      if (cls[r] == 0 && cls[l] != 0) cls4[r] = 1;
    }
  }
  std::vector<std::pair<std::pair<int, uint64_t>, int>> key(N);
  for (int c = 0; c < N; ++c) {
    uint64_t k = 0;
    for (int d = 0; d < 3; ++d) {
      const double span = hi[d] - lo[d];
      const double u = span > 0 ? (mv.cell_centroid[3 * (size_t)c + d] - lo[d]) / span : 0.0;
      const uint64_t q = (uint64_t)std::min(2097151.0, std::max(0.0, u * 2097151.0));
      k |= spread3(q) << d;
    }
    key[c] = {{cls ? (int)cls4[c] : 0, k}, c};
  }
  std::sort(key.begin(), key.end());
  h.n_deep = h.n_own = h.n_k1 = 0;
  for (int c = 0; c < N; ++c) {
    const int k = cls ? cls4[c] : 0;
    if (k == 0) ++h.n_deep;
    if (k <= 1) ++h.n_own;
    if (k <= 2) ++h.n_k1;
  }
  h.cperm.resize(N);
  std::vector<int> cinv(N);
  for (int i = 0; i < N; ++i) {
    h.cperm[i] = key[i].second;
    cinv[key[i].second] = i;
  }
  key.clear();
  key.shrink_to_fit();

  // Face order: faces touching an owned cell first -- on shards the
  // interior ones (both sides deep owned, or a boundary face of a deep cell:
  // K2 runs them while the halo is in flight) ahead of the border ones --
  // then the rest; within each group by internal left cell, stable in
  // original face id.
  auto face_interior = [&](int f) {
    if (!cls) return true;
    const int l = mv.face_left[f];
    const int r = mv.face_right[f] >= 0 ? mv.face_right[f]
                  : mv.face_partner[f] >= 0 ? mv.face_left[mv.face_partner[f]] : -1;
    return cls4[l] == 0 && (r < 0 || cls4[r] == 0);
  };
  h.F_own = h.F_int = 0;
  for (int f = 0; f < F; ++f) {
    h.F_own += touch ? (touch[f] ? 1 : 0) : 1;
    h.F_int += (!touch || touch[f]) && face_interior(f) ? 1 : 0;
  }
  std::vector<int> fstart(3 * (size_t)N + 1, 0);
  auto fkey = [&](int f) {
    return (touch && !touch[f] ? 2 * N : face_interior(f) ? 0 : N) + cinv[mv.face_left[f]];
  };
  for (int f = 0; f < F; ++f) ++fstart[fkey(f) + 1];
  for (int i = 0; i < 3 * N; ++i) fstart[i + 1] += fstart[i];
  h.fperm.resize(F);
  std::vector<int> finv(F);
  {
    std::vector<int> cur(fstart.begin(), fstart.end() - 1);
    for (int f = 0; f < F; ++f) {
      const int j = cur[fkey(f)]++;
      h.fperm[j] = f;
      finv[f] = j;
    }
  }

  auto resolved_right = [&](int f) {  // kernels.cpp:15-20
    if (mv.face_right[f] >= 0) return mv.face_right[f];
    if (mv.face_partner[f] >= 0) return mv.face_left[mv.face_partner[f]];
    return -1;
  };

  // CSR adjacency (mesh.cpp:241-271) in internal numbering; faces visited in
  // ascending ORIGINAL id so each cell's slots follow the reference order.
  std::vector<int> off(N + 1, 0);
  for (int f = 0; f < F; ++f) {
    ++off[cinv[mv.face_left[f]] + 1];
    if (mv.face_right[f] >= 0) ++off[cinv[mv.face_right[f]] + 1];
  }
  for (int i = 0; i < N; ++i) off[i + 1] += off[i];
  h.M = off[N];
  std::vector<int> adj_face(h.M), adj_nb(h.M);
  std::vector<double> sgn(h.M);
  {
    std::vector<int> cur(off.begin(), off.end() - 1);
    for (int f = 0; f < F; ++f) {
      const int rr = resolved_right(f);
      const int L = cinv[mv.face_left[f]];
      adj_face[cur[L]] = finv[f];
      adj_nb[cur[L]] = rr >= 0 ? cinv[rr] : -1;
      sgn[cur[L]++] = 1.0;
      if (mv.face_right[f] >= 0) {
        const int R = cinv[mv.face_right[f]];
        adj_face[cur[R]] = ~finv[f];
        adj_nb[cur[R]] = L;
        sgn[cur[R]++] = -1.0;
      }
    }
  }
  // Geometric closure (mesh.cpp:273-284), same slot order and expressions,
  // on every cell with a complete face set (a shard's ring 2 has not).
  for (int i = 0; i < h.n_k1; ++i) {
    double s[3] = {0.0, 0.0, 0.0};
    for (int t = off[i]; t < off[i + 1]; ++t) {
      const int j = adj_face[t] >= 0 ? adj_face[t] : ~adj_face[t];
      const int f = h.fperm[j];
      for (int d = 0; d < 3; ++d) s[d] += sgn[t] * mv.face_normal[3 * (size_t)f + d] * mv.face_area[f];
    }
    if (std::abs(s[0]) > 1e-12 || std::abs(s[1]) > 1e-12 || std::abs(s[2]) > 1e-12)
      throw Error{TAFV_ELOGIC, "mesh: geometric closure violated for a cell"};
  }

  // Permuted host arrays -> device.
  std::vector<double> vol(N), cen(3 * (size_t)N), chl(N);
  for (int i = 0; i < N; ++i) {
    const int c = h.cperm[i];
    vol[i] = mv.cell_volume[c];
    chl[i] = mv.cell_char_length[c];
    for (int d = 0; d < 3; ++d) cen[3 * (size_t)i + d] = mv.cell_centroid[3 * (size_t)c + d];
  }
  std::vector<int2> lr(F);
  std::vector<int> bface;  // ledger: transmissive faces touching owned cells
  std::vector<int> rcf(h.periodic ? F : 0);
  std::vector<double4> geo(F);
  std::vector<double> fcen(3 * (size_t)F);
  for (int j = 0; j < F; ++j) {
    const int f = h.fperm[j];
    const int rr = resolved_right(f);
    lr[j] = make_int2(cinv[mv.face_left[f]], rr >= 0 ? cinv[rr] : -1);
    if (rr < 0 && j < h.F_own) bface.push_back(j);
    if (h.periodic) rcf[j] = (mv.face_right[f] < 0 && mv.face_partner[f] >= 0) ? finv[mv.face_partner[f]] : j;
    geo[j] = make_double4(mv.face_normal[3 * (size_t)f], mv.face_normal[3 * (size_t)f + 1],
                          mv.face_normal[3 * (size_t)f + 2], mv.face_area[f]);
    for (int d = 0; d < 3; ++d) fcen[3 * (size_t)j + d] = mv.face_centroid[3 * (size_t)f + d];
  }
  h.vol_host = vol;

  auto up = [&](auto* dst, const auto& src) {
    CK(cudaMemcpy(dst, src.data(), src.size() * sizeof(src[0]), cudaMemcpyHostToDevice));
  };
  h.vol = dalloc<double>(N);
  up(h.vol, vol);
  std::vector<double> ivol(N);
  for (int i = 0; i < N; ++i) ivol[i] = 1.0 / vol[i];  // same IEEE quotient as the device's
  h.ivol = dalloc<double>(N);
  up(h.ivol, ivol);
  // Hex fast path: every cell the hot kernels visit (owned + ring 1, which
  // lead the internal order) has exactly 6 slots.
  h.deg6 = true;
  for (int i = 0; i <= h.n_k1 && h.deg6; ++i) h.deg6 = off[i] == 6 * i;
  if (h.deg6) {
    std::vector<double4> sgeo(h.M);
    std::vector<double4> sdx(h.M, make_double4(0.0, 0.0, 0.0, 0.0));
    for (int i = 0; i < h.n_k1; ++i)
      for (int t = 6 * i; t < 6 * i + 6; ++t) {
        const int j = adj_face[t] >= 0 ? adj_face[t] : ~adj_face[t];
        const double4 g = geo[j];
        sgeo[t] = make_double4(g.x, g.y, g.z, sgn[t] * g.w);
        sdx[t] = make_double4(fcen[3 * (size_t)j] - cen[3 * (size_t)i], fcen[3 * (size_t)j + 1] - cen[3 * (size_t)i + 1],
                              fcen[3 * (size_t)j + 2] - cen[3 * (size_t)i + 2], 0.0);
      }
    h.sgeo = dalloc<double4>(h.M);
    up(h.sgeo, sgeo);
    h.sdx = dalloc<double4>(h.M);
    up(h.sdx, sdx);
  }
  {
    // K2 reconstruction offsets per face (MeshDev::fdx), the kernel's own
    // differences: face centroid minus left centroid, (partner) face centroid
    // minus right centroid
    std::vector<double4> fdx(2 * (size_t)F, make_double4(0.0, 0.0, 0.0, 0.0));
    for (int j = 0; j < F; ++j) {
      const int l = lr[j].x, r = lr[j].y;
      double dl[3], dr[3] = {0.0, 0.0, 0.0};
      for (int d = 0; d < 3; ++d) dl[d] = fcen[3 * (size_t)j + d] - cen[3 * (size_t)l + d];
      if (r >= 0) {
        const int t = h.periodic ? rcf[j] : j;
        for (int d = 0; d < 3; ++d) dr[d] = fcen[3 * (size_t)t + d] - cen[3 * (size_t)r + d];
      }
      fdx[TAFV_FDX_L(j, F)] = make_double4(dl[0], dl[1], dl[2], 0.0);
      fdx[TAFV_FDX_R(j, F)] = make_double4(dr[0], dr[1], dr[2], 0.0);
    }
    h.fdx = dalloc<double4>(2 * (size_t)F);
    up(h.fdx, fdx);
  }
  h.cen = dalloc<double>(3 * (size_t)N);
  up(h.cen, cen);
  h.chl = dalloc<double>(N);
  up(h.chl, chl);
  h.adj_off = dalloc<int>(N + 1);
  up(h.adj_off, off);
  h.adj_face = dalloc<int>(h.M);
  up(h.adj_face, adj_face);
  h.adj_nb = dalloc<int>(h.M);
  up(h.adj_nb, adj_nb);
  h.lr = dalloc<int2>(F);
  up(h.lr, lr);
  if (h.periodic) {
    h.rcf = dalloc<int>(F);
    up(h.rcf, rcf);
  }
  h.geo = dalloc<double4>(F);
  up(h.geo, geo);
  h.fcen = dalloc<double>(3 * (size_t)F);
  up(h.fcen, fcen);
  h.d_cperm = dalloc<int>(N);
  up(h.d_cperm, h.cperm);
  h.d_fperm = dalloc<int>(F);
  up(h.d_fperm, h.fperm);
  h.NB = (int)bface.size();
  h.bface = dalloc<int>(std::max(1, h.NB));
  if (h.NB) up(h.bface, bface);
}

// Device build of the same arrays (meshprep.cuh): the raw mesh goes up once
// and the orderings, CSR, closure check and derived geometry are computed on
// the GPU -- seconds instead of minutes at 80M cells, and no host copies of
// the 32-byte-per-slot streams. Bitwise the host build's arrays
// (test_device_mesh_build_equals_host_build).
void upload_mesh_device(tafv_gpu& h, const tafv_mesh_view& mv, const uint8_t* cls = nullptr,
                        const uint8_t* touch = nullptr) {
  using namespace tafv::prep;
  const int N = mv.n_cells, F = mv.n_faces;
  require(N > 0 && F >= 0, "mesh: empty mesh");
  require(mv.dim >= 1 && mv.dim <= 3, "mesh: dim must be 1, 2 or 3");
  h.N = N;
  h.F = F;
  h.dim = mv.dim;
  cudaStream_t st = h.st;
  std::vector<void*> tmp;  // temporaries, freed on every exit path
  struct Guard {
    std::vector<void*>& t;
    ~Guard() {
      for (void* p : t) cudaFree(p);
    }
  } guard{tmp};
  auto talloc = [&](size_t bytes) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
    tmp.push_back(p);
    return p;
  };
  auto tfree = [&](void* p) {
    auto it = std::find(tmp.begin(), tmp.end(), p);
    if (it != tmp.end()) {
      cudaFree(p);
      tmp.erase(it);
    }
  };
  auto up = [&](const void* src, size_t bytes) {
    void* d = talloc(bytes);
    CK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st));
    return d;
  };
  const int G = h.sms * 8, B = 256;
  int* flags = (int*)talloc(sizeof(int));
  CK(cudaMemsetAsync(flags, 0, sizeof(int), st));
  const int* fl = (const int*)up(mv.face_left, (size_t)F * 4);
  const int* fr = (const int*)up(mv.face_right, (size_t)F * 4);
  const int* fp = (const int*)up(mv.face_partner, (size_t)F * 4);
  k_check_faces<<<G, B, 0, st>>>(fl, fr, fp, N, F, flags);
  int hflags = 0;
  CK(cudaMemcpyAsync(&hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  require(!(hflags & 1), "mesh: face left cell out of range");
  require(!(hflags & 2), "mesh: face right cell out of range");
  require(!(hflags & 4), "mesh: periodic partner out of range");
  h.periodic = (hflags & 8) != 0;
  const double* cen0 = (const double*)up(mv.cell_centroid, (size_t)N * 24);
  const double* vol0 = (const double*)up(mv.cell_volume, (size_t)N * 8);
  const double* chl0 = (const double*)up(mv.cell_char_length, (size_t)N * 8);

  // cell order: (class, Morton, id) -- the class pass only on shards
  std::vector<uint8_t> cls4;
  if (cls) {
    cls4.resize(N);
    for (int c = 0; c < N; ++c) cls4[c] = cls[c] == 0 ? 0 : (uint8_t)(cls[c] + 1);
    for (int f = 0; f < F; ++f) {
      const int l = mv.face_left[f];
      const int r = mv.face_right[f] >= 0 ? mv.face_right[f]
                    : mv.face_partner[f] >= 0 ? mv.face_left[mv.face_partner[f]] : -1;
      if (r < 0) continue;
      if (cls[l] == 0 && cls[r] != 0) cls4[l] = 1;
      if (cls[r] == 0 && cls[l] != 0) cls4[r] = 1;
    }
  }
  h.n_deep = h.n_own = h.n_k1 = 0;
  for (int c = 0; c < N; ++c) {
    const int k = cls ? cls4[c] : 0;
    if (k == 0) ++h.n_deep;
    if (k <= 1) ++h.n_own;
    if (k <= 2) ++h.n_k1;
  }
  double* part = (double*)talloc((size_t)G * 6 * 8);
  double* box = (double*)talloc(6 * 8);
  k_bbox_partial<<<G, 256, 0, st>>>(cen0, N, part);
  k_bbox_final<<<1, 32, 0, st>>>(part, G, box);
  size_t need = 0, have = 0;
  void* sort_tmp = nullptr;
  auto scratch = [&](size_t bytes) {
    if (bytes > have) {
      if (sort_tmp) tfree(sort_tmp);
      sort_tmp = talloc(bytes);
      have = bytes;
    }
    return sort_tmp;
  };
  h.d_cperm = dalloc<int>(N);
  {
    uint64_t* k0 = (uint64_t*)talloc((size_t)N * 8);
    uint64_t* k1 = (uint64_t*)talloc((size_t)N * 8);
    int* v0 = (int*)talloc((size_t)N * 4);
    k_morton<<<G, B, 0, st>>>(cen0, box, N, k0, v0);
    int* sorted = cls ? (int*)talloc((size_t)N * 4) : h.d_cperm;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, need, k0, k1, v0, sorted, N, 0, 63, st));
    CK(cub::DeviceRadixSort::SortPairs(scratch(need), need, k0, k1, v0, sorted, N, 0, 63, st));
    if (cls) {
      uint8_t* dcls = (uint8_t*)up(cls4.data(), N);
      uint32_t* c0 = (uint32_t*)k0;
      uint32_t* c1 = (uint32_t*)k1;
      k_class_keys<<<G, B, 0, st>>>(sorted, dcls, N, c0, v0);
      CK(cub::DeviceRadixSort::SortPairs(nullptr, need, c0, c1, v0, h.d_cperm, N, 0, 2, st));
      CK(cub::DeviceRadixSort::SortPairs(scratch(need), need, c0, c1, v0, h.d_cperm, N, 0, 2, st));
      tfree(sorted);
      tfree(dcls);
    }
    tfree(k0);
    tfree(k1);
    tfree(v0);
  }
  int* cinv = (int*)talloc((size_t)N * 4);
  k_invert<<<G, B, 0, st>>>(h.d_cperm, N, cinv);

  // face order: (touching an owned cell first -- shards: interior ones ahead
  // of border ones --, internal left cell), stable in id
  h.F_own = h.F_int = 0;
  for (int f = 0; f < F; ++f) {
    const bool t = touch ? touch[f] != 0 : true;
    h.F_own += t ? 1 : 0;
    if (t && cls) {
      const int l = mv.face_left[f];
      const int r = mv.face_right[f] >= 0 ? mv.face_right[f]
                    : mv.face_partner[f] >= 0 ? mv.face_left[mv.face_partner[f]] : -1;
      h.F_int += cls4[l] == 0 && (r < 0 || cls4[r] == 0) ? 1 : 0;
    }
  }
  if (!cls) h.F_int = h.F_own;
  h.d_fperm = dalloc<int>(std::max(1, F));
  int* finv = (int*)talloc((size_t)F * 4);
  {
    uint32_t* k0 = (uint32_t*)talloc((size_t)F * 4);
    uint32_t* k1 = (uint32_t*)talloc((size_t)F * 4);
    int* v0 = (int*)talloc((size_t)F * 4);
    const uint8_t* dtouch = touch ? (const uint8_t*)up(touch, F) : nullptr;
    const uint8_t* dcls = cls ? (const uint8_t*)up(cls4.data(), N) : nullptr;
    k_face_keys<<<G, B, 0, st>>>(fl, fr, fp, cinv, dtouch, dcls, N, F, k0, v0);
    int bits = 1;
    while (bits < 32 && (3ull * N) >> bits) ++bits;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, need, k0, k1, v0, h.d_fperm, F, 0, bits, st));
    CK(cub::DeviceRadixSort::SortPairs(scratch(need), need, k0, k1, v0, h.d_fperm, F, 0, bits, st));
    tfree(k0);
    tfree(k1);
    tfree(v0);
    if (dtouch) tfree((void*)dtouch);
    if (dcls) tfree((void*)dcls);
  }
  k_invert<<<G, B, 0, st>>>(h.d_fperm, F, finv);

  // CSR in the reference slot order
  h.adj_off = dalloc<int>(N + 1);
  int* count = (int*)talloc((size_t)(N + 1) * 4);
  CK(cudaMemsetAsync(count, 0, (size_t)(N + 1) * 4, st));
  {
    uint64_t* k0 = (uint64_t*)talloc((size_t)F * 16);
    uint64_t* k1 = (uint64_t*)talloc((size_t)F * 16);
    int* v0 = (int*)talloc((size_t)F * 8);
    int* v1 = (int*)talloc((size_t)F * 8);
    k_slot_keys<<<G, B, 0, st>>>(fl, fr, cinv, finv, F, k0, v0, count);
    CK(cub::DeviceScan::ExclusiveSum(nullptr, need, count, h.adj_off, N + 1, st));
    CK(cub::DeviceScan::ExclusiveSum(scratch(need), need, count, h.adj_off, N + 1, st));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, need, k0, k1, v0, v1, 2 * F, 0, 64, st));
    CK(cub::DeviceRadixSort::SortPairs(scratch(need), need, k0, k1, v0, v1, 2 * F, 0, 64, st));
    int M = 0;
    CK(cudaMemcpyAsync(&M, h.adj_off + N, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    h.M = M;
    h.adj_face = dalloc<int>(std::max(1, M));
    CK(cudaMemcpyAsync(h.adj_face, v1, (size_t)M * 4, cudaMemcpyDeviceToDevice, st));
    tfree(k0);
    tfree(k1);
    tfree(v0);
    tfree(v1);
  }
  tfree(count);

  // per-face arrays (ledger index of transmissive faces by a scan)
  const double* fn0 = (const double*)up(mv.face_normal, (size_t)F * 24);
  const double* fa0 = (const double*)up(mv.face_area, (size_t)F * 8);
  h.lr = dalloc<int2>(std::max(1, F));
  h.rcf = h.periodic ? dalloc<int>(F) : nullptr;
  h.geo = dalloc<double4>(std::max(1, F));
  h.fcen = dalloc<double>(3 * (size_t)std::max(1, F));
  {
    const double* fc0 = (const double*)up(mv.face_centroid, (size_t)F * 24);
    k_face_arrays<<<G, B, 0, st>>>(h.d_fperm, finv, cinv, fl, fr, fp, fn0, fa0, fc0, F, h.periodic ? 1 : 0,
                                   h.lr, h.rcf, h.geo, h.fcen);
    tfree((void*)fc0);
    int* bflag = (int*)talloc((size_t)(F + 1) * 4);
    int* bidx = (int*)talloc((size_t)(F + 1) * 4);
    k_boundary_flags<<<G, B, 0, st>>>(h.d_fperm, fr, fp, F, h.F_own, bflag);
    CK(cudaMemsetAsync(bflag + F, 0, 4, st));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, need, bflag, bidx, F + 1, st));
    CK(cub::DeviceScan::ExclusiveSum(scratch(need), need, bflag, bidx, F + 1, st));
    CK(cudaMemcpyAsync(&h.NB, bidx + F, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    h.bface = dalloc<int>(std::max(1, h.NB));
    k_boundary_list<<<G, B, 0, st>>>(bflag, bidx, F, h.bface);
    CK(cudaStreamSynchronize(st));
    tfree(bflag);
    tfree(bidx);
  }
  h.adj_nb = dalloc<int>(std::max(1, h.M));
  k_slot_nb<<<G, B, 0, st>>>(h.adj_face, h.lr, h.M, h.adj_nb);
  k_closure<<<G, B, 0, st>>>(h.adj_off, h.adj_face, h.d_fperm, fn0, fa0, h.n_k1, flags);
  CK(cudaMemcpyAsync(&hflags, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hflags & 16) throw Error{TAFV_ELOGIC, "mesh: geometric closure violated for a cell"};
  h.deg6 = !(hflags & 32);
  tfree((void*)fn0);
  tfree((void*)fa0);

  // cell arrays
  h.vol = dalloc<double>(N);
  h.ivol = dalloc<double>(N);
  h.chl = dalloc<double>(N);
  h.cen = dalloc<double>(3 * (size_t)N);
  k_cell_arrays<<<G, B, 0, st>>>(h.d_cperm, vol0, chl0, cen0, N, h.vol, h.ivol, h.chl, h.cen);
  if (h.deg6) {
    h.sgeo = dalloc<double4>(std::max(1, h.M));
    h.sdx = dalloc<double4>(std::max(1, h.M));
    CK(cudaMemsetAsync(h.sgeo, 0, (size_t)h.M * sizeof(double4), st));
    CK(cudaMemsetAsync(h.sdx, 0, (size_t)h.M * sizeof(double4), st));
    k_slot_geo<<<G, B, 0, st>>>(h.adj_face, h.geo, h.fcen, h.cen, h.n_k1, h.sgeo, h.sdx);
  }
  h.fdx = dalloc<double4>(2 * (size_t)std::max(1, F));
  k_face_dx<<<G, B, 0, st>>>(h.lr, h.rcf, h.fcen, h.cen, F, h.periodic ? 1 : 0, h.fdx);
  CK(cudaGetLastError());
  // host copies: permutations (boundary calls map ids) and V (internal order)
  h.cperm.resize(N);
  h.fperm.resize(F);
  h.vol_host.resize(N);
  CK(cudaMemcpyAsync(h.cperm.data(), h.d_cperm, (size_t)N * 4, cudaMemcpyDeviceToHost, st));
  if (F) CK(cudaMemcpyAsync(h.fperm.data(), h.d_fperm, (size_t)F * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h.vol_host.data(), h.vol, (size_t)N * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

// The brick K1's static structures (k_brick_build) for the whole bricks of
// the owned cells of a hex mesh; a no-op when they exist or cannot (not hex,
// a shard with halo cells: its identity phases run deep / border lists).
void build_bricks(tafv_gpu& h) {
  if (h.brick_idx || !h.deg6 || h.n_own != h.N || h.N < kBrick) return;
  if (h.brick_declined && h.k1_brick < 0) return;
  const int nb = h.N / kBrick;
  h.nbricks = nb;
  h.brick_info = dalloc<int4>(nb);
  h.brick_nrest = dalloc<int>(2);
  int* esize = dalloc<int>((size_t)nb + 1);
  int* hsize = dalloc<int>((size_t)nb + 1);
  int* eoff = dalloc<int>((size_t)nb + 1);
  int* hoff = dalloc<int>((size_t)nb + 1);
  auto drop = [&] {
    for (void* p : {(void*)esize, (void*)hsize, (void*)eoff, (void*)hoff}) cudaFree(p);
  };
  CK(cudaMemsetAsync(h.brick_nrest, 0, 2 * sizeof(int), h.st));
  CK(cudaMemsetAsync(esize, 0, ((size_t)nb + 1) * sizeof(int), h.st));
  CK(cudaMemsetAsync(hsize, 0, ((size_t)nb + 1) * sizeof(int), h.st));
  k_brick_build<false><<<nb, kBrick, 0, h.st>>>(h.adj_nb, h.adj_face, h.geo, h.fcen, nb, h.nv, h.brick_info, esize,
                                                hsize, nullptr, nullptr, nullptr, nullptr, h.brick_nrest + 1);
  CK(cudaGetLastError());
  // offsets: exclusive scans over nb + 1 sizes (the last entries are the totals)
  size_t need = 0, need2 = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, need, esize, eoff, nb + 1, h.st));
  CK(cub::DeviceScan::ExclusiveSum(nullptr, need2, hsize, hoff, nb + 1, h.st));
  need = std::max(need, need2);
  void* tmp = nullptr;
  CK(cudaMalloc(&tmp, std::max<size_t>(need, 16)));
  CK(cub::DeviceScan::ExclusiveSum(tmp, need, esize, eoff, nb + 1, h.st));
  CK(cub::DeviceScan::ExclusiveSum(tmp, need, hsize, hoff, nb + 1, h.st));
  int cnt[2] = {0, 0}, etot = 0, htot = 0;
  CK(cudaMemcpyAsync(cnt, h.brick_nrest, sizeof cnt, cudaMemcpyDeviceToHost, h.st));
  CK(cudaMemcpyAsync(&etot, eoff + nb, sizeof(int), cudaMemcpyDeviceToHost, h.st));
  CK(cudaMemcpyAsync(&htot, hoff + nb, sizeof(int), cudaMemcpyDeviceToHost, h.st));
  CK(cudaStreamSynchronize(h.st));
  cudaFree(tmp);
  h.brick_ragged = cnt[1];
  // auto mode: the brick kernel pays only when most bricks fit its stage
  // (config 4: 92 % fit, K1 -15 %; config 5: all fit; config 3's
  // corner-stretched mesh: 61 %, K1 +2-7 % with the rest on the general
  // kernel) -- else drop the structures
  if (h.k1_brick < 0 && (double)cnt[1] > TAFV_K1_BRICK_MAX_RAGGED * nb) {
    drop();
    cudaFree(h.brick_info);
    cudaFree(h.brick_nrest);
    h.brick_info = nullptr;
    h.brick_nrest = nullptr;
    h.brick_declined = true;
    return;
  }
  k_brick_offsets<<<h.grid_for(nb, 256), 256, 0, h.st>>>(h.brick_info, eoff, hoff, nb);
  h.brick_idx = dalloc<unsigned short>((size_t)nb * 1536);
  h.brick_halo = dalloc<int>(std::max(1, htot));
  h.brick_geo = dalloc<double>((size_t)std::max(1, etot) * 4);
  h.brick_fcen = dalloc<double>((size_t)std::max(1, etot) * 3);
  CK(cudaMemsetAsync(h.brick_halo, 0, (size_t)std::max(1, htot) * sizeof(int), h.st));
  CK(cudaMemsetAsync(h.brick_geo, 0, (size_t)std::max(1, etot) * 4 * sizeof(double), h.st));
  CK(cudaMemsetAsync(h.brick_fcen, 0, (size_t)std::max(1, etot) * 3 * sizeof(double), h.st));
  k_brick_build<true><<<nb, kBrick, 0, h.st>>>(h.adj_nb, h.adj_face, h.geo, h.fcen, nb, h.nv, h.brick_info, esize,
                                               hsize, h.brick_idx, h.brick_halo, h.brick_geo, h.brick_fcen, nullptr);
  CK(cudaGetLastError());
  const size_t cap = (size_t)cnt[1] * kBrick + (size_t)(h.N - nb * kBrick);
  h.brick_rest = dalloc<int>(std::max<size_t>(1, cap));
  k_brick_ragged_cells<<<h.grid_for(h.N, 256), 256, 0, h.st>>>(h.brick_info, nb, h.N, h.brick_rest, h.brick_nrest);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(cnt, h.brick_nrest, sizeof(int), cudaMemcpyDeviceToHost, h.st));
  CK(cudaStreamSynchronize(h.st));
  drop();
  h.brick_rest_host = cnt[0];
  h.brick_entries = etot;
  if ((size_t)cnt[0] != cap) throw std::logic_error("brick K1: ragged cell count mismatch");
}

void upload_mesh(tafv_gpu& h, const tafv_mesh_view& mv, const uint8_t* cls = nullptr,
                 const uint8_t* touch = nullptr) {
  if (getenv("TAFV_HOST_UPLOAD") != nullptr) upload_mesh_host(h, mv, cls, touch);
  else upload_mesh_device(h, mv, cls, touch);
  if (h.k1_brick > 0 || (h.k1_brick < 0 && h.n_own >= (TAFV_K1_BRICK_AUTO))) build_bricks(h);
}

void alloc_state(tafv_gpu& h) {
  const size_t N = h.N, F = h.F, nv = h.nv;
  // + 2: load_row's aligned 16-byte pairs reach one double past the last row
  h.w = dalloc<double>(N * nv + 2);
  h.W = dalloc<double>(N * nv + 2);
  h.wp = dalloc<double>(N * nv + 2);
  h.gs = (nv * 3 + 3) / 4 * 4;  // GradRow<NV>::S
  h.grad = dalloc<double>(N * h.gs);
  h.fs = (nv + 1) / 2 * 2;  // FaceRow<NV>::S
  h.phi = dalloc<double>(F * h.fs);
  h.isub = dalloc<double>(F * h.fs);
  h.iwin = dalloc<double>(F * h.fs);
  CK(cudaMemset(h.w, 0, N * nv * sizeof(double)));
  CK(cudaMemset(h.W, 0, N * nv * sizeof(double)));
  CK(cudaMemset(h.wp, 0, N * nv * sizeof(double)));
  CK(cudaMemset(h.grad, 0, N * h.gs * sizeof(double)));
  CK(cudaMemset(h.phi, 0, F * h.fs * sizeof(double)));
  CK(cudaMemset(h.isub, 0, F * h.fs * sizeof(double)));
  CK(cudaMemset(h.iwin, 0, F * h.fs * sizeof(double)));
  h.ialias = dalloc<uint8_t>(F);
  CK(cudaMemset(h.ialias, 0, F));
  h.bsum = dalloc<double>(std::max<size_t>(1, (size_t)h.NB * nv));
  CK(cudaMemset(h.bsum, 0, std::max<size_t>(1, (size_t)h.NB * nv) * sizeof(double)));
  h.nblk_led = (int)std::max<long long>(1, std::min<long long>(2LL * h.sms, ((long long)h.NB + 1023) / 1024));
  h.lpart = dalloc<DD>((size_t)nv * h.nblk_led);
  h.tau = dalloc<int8_t>(N);
  h.raw = dalloc<int8_t>(N);
  h.sweep_tile = dalloc<uint8_t>((size_t)kMaxLevels * ((N + kTile - 1) / kTile + 1));
  h.tmpa = dalloc<int8_t>(N);
  h.tmpb = dalloc<int8_t>(N);
  h.fflag = dalloc<uint8_t>(((size_t)N + 3) & ~(size_t)3);  // word-addressed by k_face_cadence
  CK(cudaMemset(h.fflag, 0, ((size_t)N + 3) & ~(size_t)3));
  h.dt_ticket = dalloc<unsigned>(1);
  CK(cudaMemset(h.dt_ticket, 0, sizeof(unsigned)));
  h.cad = dalloc<int8_t>(F);
  CK(cudaMemset(h.tau, 0, N));
  CK(cudaMemset(h.cad, 0, F));
  h.dtmax = dalloc<double>(N);
#ifndef TAFV_DT_BPS
#define TAFV_DT_BPS 4
#endif
  h.nblk_dt = h.sms * TAFV_DT_BPS;
  h.blockmin = dalloc<double>(h.nblk_dt);
  h.ntile_c = (int)((h.n_own + kTile - 1) / kTile);
  h.ntile_f = (int)((h.F_own + kTile - 1) / kTile);
  h.cell_counts = dalloc<int>((size_t)std::max(1, h.ntile_c) * kMaxLevels);
  h.face_counts = dalloc<int>((size_t)std::max(1, h.ntile_f) * kMaxLevels);
  h.clist = dalloc<int>(N);
  h.flist = dalloc<int>(F);
  if (h.n_k1 != h.n_own || h.n_deep != h.n_own) {
    h.klist = dalloc<int>(std::max(1, h.n_deep));
    h.ntile_k = (int)((h.n_deep + kTile - 1) / kTile);
    h.k1_counts = dalloc<int>((size_t)std::max(1, h.ntile_k) * kMaxLevels);
    h.kblist = dalloc<int>(std::max(1, h.n_k1 - h.n_deep));
    h.ntile_kb = (int)((h.n_k1 - h.n_deep + kTile - 1) / kTile);
    h.kb_counts = dalloc<int>((size_t)std::max(1, h.ntile_kb) * kMaxLevels);
    h.ntile_fi = (int)((h.F_int + kTile - 1) / kTile);
    h.ntile_fb = (int)((h.F_own - h.F_int + kTile - 1) / kTile);
    h.filist = dalloc<int>(std::max(1, h.F_int));
    h.fblist = dalloc<int>(std::max(1, h.F_own - h.F_int));
    h.fi_counts = dalloc<int>((size_t)std::max(1, h.ntile_fi) * kMaxLevels);
    h.fb_counts = dalloc<int>((size_t)std::max(1, h.ntile_fb) * kMaxLevels);
  } else {
    h.klist = h.clist;
  }
  if (h.sharded() && h.peers.size() <= (size_t)kMaxPeers && getenv("TAFV_FULL_HALO") == nullptr) {
    h.xfilter = true;
    h.xkey_s = dalloc<int8_t>(std::max(1, h.send_total));
    h.xkey_r = dalloc<int8_t>(std::max(1, h.recv_total));
    h.xpos_s = dalloc<int>(std::max(1, h.send_total));
    h.xpos_r = dalloc<int>(std::max(1, h.recv_total));
    h.xsorted_s = dalloc<int>(std::max(1, h.send_total));
    h.xsorted_r = dalloc<int>(std::max(1, h.recv_total));
    int maxseg = 1;
    for (const auto& p : h.peers) maxseg = std::max(maxseg, std::max(p.nsend, p.nrecv));
    h.xtile_stride = ((maxseg + kTile - 1) / kTile) * kMaxLevels;
    h.xcounts = dalloc<int>((size_t)std::max<size_t>(1, 2 * h.peers.size()) * h.xtile_stride);
  }
  h.nblk_last = h.sms * 16;
  h.partials = dalloc<DD>((size_t)h.nblk_last * 8);
  h.dplan = dalloc<PlanDev>(1);
  CK(cudaMemset(h.dplan, 0, sizeof(PlanDev)));
  CK(cudaMallocHost(&h.hplan, sizeof(PlanDev)));
  std::memset(h.hplan, 0, sizeof(PlanDev));
  for (auto& e : h.ev) CK(cudaEventCreate(&e));
  CK(cudaStreamCreateWithFlags(&h.lst, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&h.ev_led_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h.ev_led, cudaEventDisableTiming));
}

// Fixed grids for graph capture: every SM filled to the kernel's occupancy.
template <class P, int DEG>
void set_grids_t(tafv_gpu& h) {
  int b1 = 0, b2 = 0, b3 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_grad_limit<P, DEG, false>, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_face_flux<P, true>, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b3, k_gather_update<P, true, false, DEG>, 128, 0));
  h.grid_k1 = h.sms * std::max(1, b1);
  if (DEG == 6) {
    // brick K1: dynamic shared memory (one stage per block), carve-out at its maximum
    constexpr int smem = BrickSmem<P::NV>::bytes;
    CK(cudaFuncSetAttribute(k_grad_limit_brick<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_grad_limit_brick<P>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            cudaSharedmemCarveoutMaxShared));
    int bb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bb, k_grad_limit_brick<P>, kBrick, smem));
    h.grid_k1b = h.sms * std::max(1, bb);
  }
  // trailing corrector: exactly one wave of resident blocks (its partials
  // buffer holds sms * 16 blocks)
  int bl = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bl, k_gather_update<P, false, true, DEG>, 128, 0));
  h.nblk_last = h.sms * std::max(1, std::min(16, bl));
  h.grid_k2 = h.sms * std::max(1, b2);
  h.grid_k3 = h.sms * std::max(1, b3);
}

template <class P>
void set_grids_p(tafv_gpu& h) {
  if (h.deg6) set_grids_t<P, 6>(h);
  else set_grids_t<P, 0>(h);
}

void set_grids(tafv_gpu& h) {
  switch (h.model) {
    case TAFV_ADVECTION: set_grids_p<Advection2D>(h); break;
    case TAFV_BURGERS: set_grids_p<Burgers2D>(h); break;
    default: set_grids_p<Euler3D>(h); break;
  }
}

// ---- optional per-kernel timing ---------------------------------------------
template <class F>
void timed(tafv_gpu& h, int kind, F&& launch, long long cells = 0, long long faces = 0,
           long long fringe = 0) {
  if (!h.ktime) {
    launch();
    return;
  }
  if (h.cap) {  // inside a graph capture: dedicated events become graph nodes
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    // external records: real event-record nodes (a plain record inside a
    // capture only expresses a dependency and carries no timestamp)
    CK(cudaEventRecordWithFlags(a, h.st, cudaEventRecordExternal));
    launch();
    CK(cudaEventRecordWithFlags(b, h.st, cudaEventRecordExternal));
    h.cap->evs.push_back(a);
    h.cap->evs.push_back(b);
    h.cap->kinds.push_back(kind);
    h.cap->items.push_back({cells, faces, fringe});
    return;
  }
  h.kitems[kind][0] += cells;
  h.kitems[kind][1] += faces;
  h.kitems[kind][2] += fringe;
  const size_t i = h.evkind.size();
  while (h.evpool.size() < 2 * (i + 1)) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    h.evpool.push_back(e);
  }
  CK(cudaEventRecord(h.evpool[2 * i], h.st));
  launch();
  CK(cudaEventRecord(h.evpool[2 * i + 1], h.st));
  h.evkind.push_back(kind);
}

// After a host sync: fold the recorded pairs into the per-kind totals.
void collect_times(tafv_gpu& h) {
  if (h.pending_graph) {
    const auto& g = *h.pending_graph;
    for (size_t i = 0; i < g.kinds.size(); ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, g.evs[2 * i], g.evs[2 * i + 1]));
      // per-launch log (kind, active cells / faces / fringe at capture, us):
      // tools/klog_summary.py, tools/small_phase_probe.py
      if (h.klog)
        fprintf(stderr, "KLOG %d %lld %lld %lld %.4f\n", g.kinds[i], g.items[i][0], g.items[i][1], g.items[i][2],
                ms * 1e3);
      h.kms[g.kinds[i]] += ms;
      h.kcnt[g.kinds[i]] += 1;
      for (int j = 0; j < 3; ++j) h.kitems[g.kinds[i]][j] += g.items[i][j];
    }
    h.pending_graph = nullptr;
  }
  for (size_t i = 0; i < h.evkind.size(); ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h.evpool[2 * i], h.evpool[2 * i + 1]));
    h.kms[h.evkind[i]] += ms;
    h.kcnt[h.evkind[i]] += 1;
  }
  h.evkind.clear();
}

// ---- halo exchange (shards) -------------------------------------------------
// Owned rows listed for the peers -> sendbuf -> comm -> recvbuf -> halo rows.
// The pack runs on the compute stream right behind the K3 that wrote the
// rows; the exchange and the unpack run on the comm stream, so the next
// phase's K1 over the deep cells (which read no halo row) overlaps them.
// join_now: the compute stream waits for the halo at once (trailing
// corrector: the plan follows); otherwise the next K1 joins it before its
// border cells (halo_join).
// level >= 0 (level-sorted lists): only the rows of cells with tau <= level,
// the ones the phase just updated, move.
void halo_rows(tafv_gpu& h, double* arr, int width, bool join_now, int level = -1) {
  if (!h.sharded()) return;
  if (h.xfilter && level >= 0) {
    int sc[kMaxPeers], rc[kMaxPeers];
    for (size_t q = 0; q < h.peers.size(); ++q) {
      const auto& pe = h.peers[q];
      sc[q] = h.xs[q][level];
      rc[q] = h.xr[q][level];
      if (sc[q])
        k_pack_rows<<<h.grid_for((long long)sc[q] * width, 256), 256, 0, h.st>>>(
            arr, h.xsorted_s + pe.soff, sc[q], width, h.sendbuf + (size_t)pe.soff * width);
    }
    CK(cudaEventRecord(h.ev_pack, h.st));
    CK(cudaStreamWaitEvent(h.cst, h.ev_pack, 0));
    h.comm->exchange(h, width * (int)sizeof(double), h.cst, sc, rc);
    for (size_t q = 0; q < h.peers.size(); ++q) {
      const auto& pe = h.peers[q];
      if (rc[q])
        k_unpack_rows<<<h.grid_for((long long)rc[q] * width, 256), 256, 0, h.cst>>>(
            h.recvbuf + (size_t)pe.roff * width, h.xsorted_r + pe.roff, rc[q], width, arr);
    }
    h.launches += 2 * (int64_t)h.peers.size();
  } else {
    if (h.send_total)
      k_pack_rows<<<h.grid_for((long long)h.send_total * width, 256), 256, 0, h.st>>>(
          arr, h.d_send_idx, h.send_total, width, h.sendbuf);
    CK(cudaEventRecord(h.ev_pack, h.st));
    CK(cudaStreamWaitEvent(h.cst, h.ev_pack, 0));
    h.comm->exchange(h, width * (int)sizeof(double), h.cst);
    if (h.recv_total)
      k_unpack_rows<<<h.grid_for((long long)h.recv_total * width, 256), 256, 0, h.cst>>>(
          h.recvbuf, h.d_recv_idx, h.recv_total, width, arr);
    h.launches += 2;
  }
  CK(cudaEventRecord(h.ev_halo, h.cst));
  h.halo_pending = true;
  if (join_now) halo_join(h);
}

void halo_i8(tafv_gpu& h, int8_t* arr) {
  if (!h.sharded()) return;
  int8_t* sb = reinterpret_cast<int8_t*>(h.sendbuf);
  int8_t* rb = reinterpret_cast<int8_t*>(h.recvbuf);
  if (h.send_total)
    k_pack_i8<<<h.grid_for(h.send_total, 256), 256, 0, h.st>>>(arr, h.d_send_idx, h.send_total, sb);
  h.comm->exchange(h, 1, h.st);
  if (h.recv_total)
    k_unpack_i8<<<h.grid_for(h.recv_total, 256), 256, 0, h.st>>>(rb, h.d_recv_idx, h.recv_total, arr);
  h.launches += 2;
}

// ---- plan ------------------------------------------------------------------
template <class P>
void launch_dt_max(tafv_gpu& h, double cfl, double dt_cap, const int8_t* tau_scale, bool reset) {
  k_dt_max<P><<<h.nblk_dt, 256, 0, h.st>>>(h.mesh_dev(), h.state_dev(), h.pp, cfl, dt_cap, h.dtmax,
                                          h.blockmin, tau_scale, h.n_own, h.dt_ticket, h.dplan,
                                          reset ? 1 : 0);
  ++h.launches;
  // global stable step: exact min over ranks (RankComm::allreduce_min,
  // exchange.cpp:155-192)
  if (h.sharded()) h.comm->allreduce_min_f64(h.rank, &h.dplan->dt_min, 1, h.st);
}

// reset: also clear the plan's error flag and counts (plan_iteration); dt_min
// is written, nonfinite/totals (the previous sweep's, read back with this
// plan) are kept.
void dispatch_dt_max(tafv_gpu& h, double cfl, double dt_cap, const int8_t* tau_scale, bool reset) {
  switch (h.model) {
    case TAFV_ADVECTION: launch_dt_max<Advection2D>(h, cfl, dt_cap, tau_scale, reset); break;
    case TAFV_BURGERS: launch_dt_max<Burgers2D>(h, cfl, dt_cap, tau_scale, reset); break;
    default: launch_dt_max<Euler3D>(h, cfl, dt_cap, tau_scale, reset); break;
  }
}

// Face cadences, fringe counts and the level-sorted cell / face lists, then
// the asynchronous read-back of the plan (and of the previous sweep's flags).
// cells_counted: the last level sweep already left the cell tile counts and
// cleared the fringe flags (single-domain plan).
void enqueue_finish_plan(tafv_gpu& h, int nkeys, bool cells_counted) {
  const MeshDev md = h.mesh_dev();
  const int ntc = std::max(1, h.ntile_c);
  if (!cells_counted) {
    CK(cudaMemsetAsync(h.fflag, 0, h.N, h.st));
    k_tile_count<<<ntc, kCompactThreads, 0, h.st>>>(h.tau, h.n_own, nkeys, h.cell_counts);
    ++h.launches;
  }
  const bool k1 = h.klist != h.clist;  // shards: deep and border K1 lists
  if (k1) {
    k_tile_count<<<std::max(1, h.ntile_k), kCompactThreads, 0, h.st>>>(h.tau, h.n_deep, nkeys, h.k1_counts);
    k_tile_count<<<std::max(1, h.ntile_kb), kCompactThreads, 0, h.st>>>(h.tau + h.n_deep, h.n_k1 - h.n_deep,
                                                                        nkeys, h.kb_counts);
    h.launches += 2;
  }
  k_face_cadence<<<std::max(1, (h.F + kTile - 1) / kTile), kCompactThreads, 0, h.st>>>(
      md, h.tau, h.cad, reinterpret_cast<unsigned*>(h.fflag), h.dplan, h.n_own, h.F_own, nkeys, h.face_counts,
      h.ntile_f);
  if (k1) {  // shards: interior / border face lists
    k_tile_count<<<std::max(1, h.ntile_fi), kCompactThreads, 0, h.st>>>(h.cad, h.F_int, nkeys, h.fi_counts);
    k_tile_count<<<std::max(1, h.ntile_fb), kCompactThreads, 0, h.st>>>(h.cad + h.F_int, h.F_own - h.F_int,
                                                                        nkeys, h.fb_counts);
    h.launches += 2;
  }
  // K3 list (owned cells by level), K2 list (faces touching owned by cadence),
  // shards' K1 list: prefixes of each are the active sets of every level
  CompactJobs jobs{};
  // single domain: the top level's entries are never read (identity phases)
  h.lists_skip_top = !h.sharded() && h.skip_top_lists;
  const long long* top_of = h.lists_skip_top ? &h.dplan->cell_count[0] : nullptr;
  jobs.j[0] = CompactJob{h.tau, h.n_own, ntc, h.cell_counts, h.clist, &h.dplan->cell_count[0],
                         &h.dplan->ncell_prefix[0], 0, top_of};
  jobs.j[1] = CompactJob{h.cad, h.F_own, h.ntile_f, h.face_counts, h.flist, &h.dplan->face_count[0],
                         &h.dplan->nface_prefix[0], 0, top_of};
  jobs.njobs = 2;
  if (k1) {
    jobs.j[2] = CompactJob{h.tau, h.n_deep, std::max(1, h.ntile_k), h.k1_counts, h.klist,
                           &h.dplan->k1_count[0], &h.dplan->nk1_prefix[0], 0, nullptr};
    jobs.j[3] = CompactJob{h.tau + h.n_deep, h.n_k1 - h.n_deep, std::max(1, h.ntile_kb), h.kb_counts,
                           h.kblist, &h.dplan->kb_count[0], &h.dplan->nkb_prefix[0], h.n_deep, nullptr};
    jobs.j[4] = CompactJob{h.cad, h.F_int, std::max(1, h.ntile_fi), h.fi_counts, h.filist,
                           &h.dplan->fi_count[0], &h.dplan->nfi_prefix[0], 0, nullptr};
    jobs.j[5] = CompactJob{h.cad + h.F_int, h.F_own - h.F_int, std::max(1, h.ntile_fb), h.fb_counts, h.fblist,
                           &h.dplan->fb_count[0], &h.dplan->nfb_prefix[0], h.F_int, nullptr};
    jobs.njobs = 6;
  }
  if (h.xfilter) {  // the exchange lists of every peer, sorted by level
    if (h.send_total)
      k_gather_keys<<<h.grid_for(h.send_total, 256), 256, 0, h.st>>>(h.tau, h.d_send_idx, h.send_total, h.xkey_s);
    if (h.recv_total)
      k_gather_keys<<<h.grid_for(h.recv_total, 256), 256, 0, h.st>>>(h.tau, h.d_recv_idx, h.recv_total, h.xkey_r);
    h.launches += 2;
    for (size_t q = 0; q < h.peers.size(); ++q) {
      const auto& pe = h.peers[q];
      for (int side = 0; side < 2; ++side) {
        const int n = side ? pe.nrecv : pe.nsend, off = side ? pe.roff : pe.soff;
        const int nt = std::max(1, (n + kTile - 1) / kTile);
        int* cnt = h.xcounts + (2 * q + side) * (size_t)h.xtile_stride;
        const int8_t* key = (side ? h.xkey_r : h.xkey_s) + off;
        k_tile_count<<<nt, kCompactThreads, 0, h.st>>>(key, n, nkeys, cnt);
        ++h.launches;
        jobs.j[jobs.njobs++] = CompactJob{key, n, nt, cnt, (side ? h.xpos_r : h.xpos_s) + off,
                                          side ? &h.dplan->xr_count[q][0] : &h.dplan->xs_count[q][0],
                                          side ? &h.dplan->xr_prefix[q][0] : &h.dplan->xs_prefix[q][0], off,
                                          nullptr};
      }
    }
  }
  int tiles = 0;
  for (int q = 0; q < jobs.njobs; ++q) tiles += jobs.j[q].ntiles;
  k_tile_scan<<<jobs.njobs, 1024, 0, h.st>>>(jobs, nkeys, h.dplan, k1 ? 0 : 1);
  if (nkeys <= 5) k_tile_scatter_packed<<<tiles, kCompactThreads, 0, h.st>>>(jobs, nkeys);
  else k_tile_scatter<<<tiles, kCompactThreads, 0, h.st>>>(jobs, nkeys);
  if (h.xfilter) {
    if (h.send_total)
      k_permute_list<<<h.grid_for(h.send_total, 256), 256, 0, h.st>>>(h.d_send_idx, h.xpos_s, h.send_total,
                                                                        h.xsorted_s);
    if (h.recv_total)
      k_permute_list<<<h.grid_for(h.recv_total, 256), 256, 0, h.st>>>(h.d_recv_idx, h.xpos_r, h.recv_total,
                                                                        h.xsorted_r);
    h.launches += 2;
  }
  h.launches += 3;
  if (h.sharded()) h.comm->allreduce_sum_i64(h.rank, &h.dplan->gcell_count[0], kMaxLevels, h.st);
  CK(cudaGetLastError());
  store_plan(h);
  h.plan_nkeys = nkeys;
}

// Host side of the plan once its read-back landed (after a stream sync).
void parse_plan(tafv_gpu& h);

void accept_plan(tafv_gpu& h) {
  {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h.ev[2], h.ev[3]));
    h.ms[1] += ms;
    if (h.ktime) {
      h.kms[tafv_gpu::kPlan] += ms;
      h.kcnt[tafv_gpu::kPlan] += 1;
    }
  }
  parse_plan(h);
}

// The host copy of a plan (h.hplan) -> levels, counts, dt; error flags throw.
void parse_plan(tafv_gpu& h) {
  const PlanDev& p = *h.hplan;
  const int nkeys = h.plan_nkeys;
  h.has_plan = false;
  if (p.err & 2) throw Error{TAFV_EINVAL, "level map: level outside [0, 15]"};
  if (p.err & 1)
    throw Error{TAFV_ELOGIC, "plan: neighbouring levels differ by more than one (unsmoothed level map)"};
  h.dt = p.dt_min;
  h.theta = 0;
  for (int l = 0; l < kMaxLevels; ++l) {
    h.ccount[l] = l < nkeys ? p.cell_count[l] : 0;
    h.fcount[l] = l < nkeys ? p.face_count[l] : 0;
    h.frcount[l] = p.fringe_count[l];
    h.gcount[l] = l < nkeys ? p.gcell_count[l] : 0;
    if (h.gcount[l] > 0) h.theta = l;  // theta = max level over all ranks
  }
  if (h.xfilter)
    for (size_t q = 0; q < h.peers.size(); ++q)
      for (int l = 0; l < kMaxLevels; ++l) {
        h.xs[q][l] = p.xs_prefix[q][l];
        h.xr[q][l] = p.xr_prefix[q][l];
      }
  h.has_plan = true;
}

void fill_plan_info(const tafv_gpu& h, tafv_plan_info* out) {
  if (!out) return;
  std::memset(out, 0, sizeof *out);
  out->theta = h.theta;
  out->n_levels = h.theta + 1;
  out->dt = h.dt;
  long long cost = 0, fe = 0, re = 0;
  for (int l = 0; l <= h.theta; ++l) {
    out->cells_per_level[l] = h.gcount[l];
    out->faces_per_cadence[l] = h.fcount[l];
    cost += (1ll << (h.theta - l)) * h.gcount[l];
    fe += (1ll << (h.theta - l)) * h.fcount[l];
  }
  for (int l = 0; l < h.theta; ++l) {
    out->fringe_per_level[l] = h.frcount[l];
    re += (1ll << (h.theta - l)) * h.frcount[l];
  }
  out->c_eff = cost;
  out->f_eff = fe;
  out->r_eff = re;
  // LevelMap::cost_ratio (levels.cpp:73-79)
  const long long ncells = h.sharded() ? h.N_global : h.N;
  out->cost_ratio = cost == 0 ? 1.0 : (double)((1ll << h.theta) * ncells) / (double)cost;
}

void plan_kernels(tafv_gpu& h, const tafv_options& opt);

// plan_iteration on the device: either the captured plan graph of these
// options (kernels + the read-back copy, one launch) or direct launches.
// Raw levels of the last regular plan from its dt_max and dt_min (bitwise the
// values the fused sweep used: the same classify_raw on the same operands).
void materialise_raw(tafv_gpu& h) {
  k_classify<<<h.grid_for(h.N, 256), 256, 0, h.st>>>(h.N, h.dtmax, h.dplan, h.plan_nkeys - 1, h.raw);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h.st));
  h.raw_lazy = false;
}

void enqueue_plan(tafv_gpu& h, const tafv_options& opt) {
  h.raw_lazy = !h.sharded();  // single domain: raw levels fused away (materialised on read)
  const Range r("tafv.plan");
  require(opt.theta_max >= 0, "classify: theta_max must be >= 0");
  require(opt.theta_max < kMaxLevels, "classify: theta_max above the supported 15");
  require(h.state_set, "plan: state not set");
  h.has_plan = false;
  CK(cudaEventRecord(h.ev[2], h.st));
  if (!h.use_graph || !h.plan_graph_on || (h.sharded() && !h.comm->capturable())) {
    plan_kernels(h, opt);
  } else {
    const bool same = h.plan_graph && h.plan_opt.theta_max == opt.theta_max &&
                      h.plan_opt.cfl == opt.cfl && h.plan_opt.dt_cap == opt.dt_cap;
    if (!same) {
      if (h.plan_graph) CK(cudaGraphExecDestroy(h.plan_graph));
      h.plan_graph = nullptr;
      cudaGraph_t g;
      const int64_t l0 = h.launches;
      h.capturing = true;
      CK(cudaStreamBeginCapture(h.st, cudaStreamCaptureModeThreadLocal));
      plan_kernels(h, opt);
      const cudaError_t e = cudaStreamEndCapture(h.st, &g);
      h.capturing = false;
      CK(e);
      CK(cudaGraphInstantiate(&h.plan_graph, g, 0));
      CK(cudaGraphDestroy(g));
      h.plan_opt = opt;
      h.plan_graph_launches = h.launches - l0;
      h.launches = l0;
    }
    CK(cudaGraphLaunch(h.plan_graph, h.st));
    h.launches += h.plan_graph_launches;
    h.plan_nkeys = opt.theta_max + 1;
  }
  CK(cudaEventRecord(h.ev[3], h.st));
}

void plan_kernels(tafv_gpu& h, const tafv_options& opt) {
  dispatch_dt_max(h, opt.cfl, opt.dt_cap, nullptr, true);
  const MeshDev md = h.mesh_dev();
  const int nkeys = opt.theta_max + 1;
  if (!h.sharded()) {
    // classification fused into the first Jacobi sweep, tile counts into the
    // last (k_level_sweep). The fixpoint is min_d raw(d) + dist(c, d); a cell
    // more than theta_max hops away cannot lower raw(c) <= theta_max, so
    // theta_max sweeps reach it exactly (levels.cpp:33-51).
    const int ntc = std::max(1, h.ntile_c);
    const int sweeps = std::max(1, opt.theta_max);
    // per-sweep tile marks (k_level_sweep): sweep i + 1 only re-evaluates the
    // tiles a level change of sweep i can reach
    const bool marks = h.sweep_marks && sweeps > 1;
    if (marks) CK(cudaMemsetAsync(h.sweep_tile, 0, (size_t)sweeps * ntc, h.st));
    const int gs = marks ? ntc : h.grid_for(h.n_own, 256);
    const int8_t* src = nullptr;
    for (int i = 0; i < sweeps; ++i) {
      const bool first = i == 0, last = i == sweeps - 1;
      int8_t* dst = last ? h.tau : (i % 2 == 0 ? h.tmpa : h.tmpb);
      const int sm = opt.theta_max > 0 ? 1 : 0;
      uint8_t* clr = first ? h.fflag : nullptr;
      const uint8_t* tp = marks && !first ? h.sweep_tile + (size_t)(i - 1) * ntc : nullptr;
      uint8_t* tc = marks && !last ? h.sweep_tile + (size_t)i * ntc : nullptr;
      if (first && last)
        k_level_sweep<true, true><<<ntc, kCompactThreads, 0, h.st>>>(md, src, h.dtmax, h.dplan, opt.theta_max,
                                                                     sm, dst, h.n_own, nkeys, h.cell_counts, clr, i, h.deg6 ? 6 : 0, tp, tc);
      else if (first)
        k_level_sweep<true, false><<<gs, kCompactThreads, 0, h.st>>>(md, src, h.dtmax, h.dplan, opt.theta_max,
                                                                     sm, dst, h.n_own, nkeys, h.cell_counts, clr, i, h.deg6 ? 6 : 0, tp, tc);
      else if (last)
        k_level_sweep<false, true><<<ntc, kCompactThreads, 0, h.st>>>(md, src, h.dtmax, h.dplan, opt.theta_max,
                                                                      sm, dst, h.n_own, nkeys, h.cell_counts, clr, i, h.deg6 ? 6 : 0, tp, tc);
      else
        k_level_sweep<false, false><<<gs, kCompactThreads, 0, h.st>>>(md, src, h.dtmax, h.dplan, opt.theta_max,
                                                                      sm, dst, h.n_own, nkeys, h.cell_counts, clr, i, h.deg6 ? 6 : 0, tp, tc);
      ++h.launches;
      src = dst;
    }
    enqueue_finish_plan(h, nkeys, true);
    return;
  }
  k_classify<<<h.grid_for(h.n_own, 256), 256, 0, h.st>>>(h.n_own, h.dtmax, h.dplan, opt.theta_max, h.raw);
  ++h.launches;
  halo_i8(h, h.raw);
  // Jacobi smoothing (levels.cpp:33-51), theta_max sweeps as above; shards
  // sweep the owned cells, then refresh the halo levels (the replicated-array
  // Jacobi of the reference, levels.hpp:32-37)
  if (opt.theta_max == 0) {
    CK(cudaMemcpyAsync(h.tau, h.raw, h.N, cudaMemcpyDeviceToDevice, h.st));  // raw halo already fresh
  } else {
    const int8_t* src = h.raw;
    for (int i = 0; i < opt.theta_max; ++i) {
      int8_t* dst = i == opt.theta_max - 1 ? h.tau : (i % 2 == 0 ? h.tmpa : h.tmpb);
      k_smooth<<<h.grid_for(h.n_own, 256), 256, 0, h.st>>>(md, src, dst, h.n_own);
      ++h.launches;
      halo_i8(h, dst);
      src = dst;
    }
  }
  enqueue_finish_plan(h, nkeys, false);
}

// After the plan read-back: levels, counts and the stable-step check
// (reference.cpp:93).
void check_plan(tafv_gpu& h) {
  accept_plan(h);
  h.levels_made = true;
  if (!(std::isfinite(h.dt) && h.dt > 0.0)) {
    h.has_plan = false;
    throw Error{TAFV_EINVAL, "integrate: stable step collapsed"};
  }
}

void plan(tafv_gpu& h, const tafv_options& opt) {
  enqueue_plan(h, opt);
  CK(cudaStreamSynchronize(h.st));
  check_plan(h);
}

void inject(tafv_gpu& h, const int32_t* tau_in, double dt, const tafv_options* opt) {
  // the reference leaves raw_level as the last plan_iteration computed it:
  // materialise it before dt_max / dt_min are overwritten
  if (h.raw_lazy) materialise_raw(h);
  require(h.state_set || dt > 0.0, "inject_levels: state not set");
  // shards take the GLOBAL level map and keep their local cells' entries
  std::vector<int32_t> local;
  const int32_t* tau_host = tau_in;
  if (h.sharded()) {
    local.resize(h.N);
    for (int i = 0; i < h.N; ++i) local[i] = tau_in[h.shard_cells[i]];
    tau_host = local.data();
  }
  int maxl = 0;
  const int nchk = h.sharded() ? h.N_global : h.N;
  for (int c = 0; c < nchk; ++c) {
    require(tau_in[c] >= 0, "level map: negative level");
    maxl = std::max(maxl, (int)tau_in[c]);
  }
  require(maxl < kMaxLevels, "level map: level above the supported 15");
  h.has_plan = false;
  CK(cudaEventRecord(h.ev[2], h.st));
  CK(cudaMemsetAsync(h.dplan, 0, sizeof(PlanDev), h.st));
  int32_t* stage = reinterpret_cast<int32_t*>(h.staging(((size_t)h.N + 1) / 2));
  CK(cudaMemcpyAsync(stage, tau_host, (size_t)h.N * sizeof(int32_t), cudaMemcpyHostToDevice, h.st));
  k_gather_i8<<<h.grid_for(h.N, 256), 256, 0, h.st>>>(stage, h.d_cperm, h.N, h.tau, h.dplan, kMaxLevels - 1);
  ++h.launches;
  if (dt > 0.0) {
    h.hplan->dt_min = dt;
    CK(cudaMemcpyAsync(&h.dplan->dt_min, &h.hplan->dt_min, sizeof(double), cudaMemcpyHostToDevice, h.st));
  } else {
    require(opt != nullptr, "inject_levels: dt <= 0 needs options for the stable step");
    dispatch_dt_max(h, opt->cfl, opt->dt_cap, h.tau, false);
  }
  enqueue_finish_plan(h, maxl + 1, false);
  CK(cudaEventRecord(h.ev[3], h.st));
  CK(cudaStreamSynchronize(h.st));
  accept_plan(h);
  if (!(std::isfinite(h.dt) && h.dt > 0.0)) {  // levels.cpp:54
    h.has_plan = false;
    throw Error{TAFV_EINVAL, "level map: dt must be positive"};
  }
}

// ---- conservation ledger (k_ledger) on the side stream -----------------------
// After a corrector's K2 the ledger kernel forks onto `lst` (it reads only
// int_substep and cadences, which nothing touches until the next corrector's
// K2); the library stream joins it before that K2 and before k_totals. In a
// captured sweep the fork / join are graph edges: the ledger is off the
// critical path.
template <int NV>
void ledger_fork(tafv_gpu& h, int level) {
  if (h.NB == 0) return;
  CK(cudaEventRecord(h.ev_led_fork, h.st));
  CK(cudaStreamWaitEvent(h.lst, h.ev_led_fork, 0));
  const int g = std::max(1, std::min(h.sms * 4, (h.NB + 255) / 256));
  k_ledger<NV><<<g, 256, 0, h.lst>>>(h.bface, h.NB, h.cad, level, h.isub, (int)h.fs, h.bsum);
  CK(cudaEventRecord(h.ev_led, h.lst));
  h.led_pending = true;
  ++h.launches;
}
void ledger_join(tafv_gpu& h) {
  if (!h.led_pending) return;
  CK(cudaStreamWaitEvent(h.st, h.ev_led, 0));
  h.led_pending = false;
}

// ---- the subiteration sweep ------------------------------------------------
template <class P, int DEG>
void phase_t(tafv_gpu& h, bool pred, bool last, int level, int front) {
  long long na = 0, nf = 0, nk = 0;
  for (int l = 0; l <= level; ++l) {
    na += h.ccount[l];
    nf += h.fcount[l];
  }
  nk = h.klist == h.clist ? na : h.n_deep;  // shards: deep cells (upper bound); border below
  // Level theta activates every cell and face (tau <= theta): identity lists
  // (owned / owned + ring 1 / faces touching owned lead the internal order).
  const bool all = level == h.theta;
  const int* cl = all ? nullptr : h.clist;
  const int* kl = all ? nullptr : h.klist;
  const int* fl = all ? nullptr : h.flist;
  const int* ncp = &h.dplan->ncell_prefix[level];
  const int* nkp = &h.dplan->nk1_prefix[level];
  const int* nkbp = &h.dplan->nkb_prefix[level];
  const int* kbl = all ? nullptr : h.kblist;
  const int* nfp = &h.dplan->nface_prefix[level];
  const MeshDev md = h.mesh_dev();
  const StateDev sd = h.state_dev();
  // Graph mode: fixed occupancy-sized grids (the capture must not depend on
  // the counts); direct mode: grids sized from the host-known counts.
  const bool fixed = h.capturing;
  constexpr int CPB = (32 / P::NV) * 4;  // cells per 128-thread block in K3
  const int g1 = fixed ? h.grid_k1 : h.grid_for(nk, 128);
  const int g2 = fixed ? h.grid_k2 : h.grid_for(nf, 128);
  const int g3 = fixed ? h.grid_k3 : h.grid_for((na + CPB - 1) / CPB * 128, 128);
  const long long nfr = level < h.theta ? h.frcount[level] : 0;
  timed(h, tafv_gpu::kK1, [&] {
    // identity phases (kl == nullptr) of hex meshes: the bulk-copy brick kernel
    // (single list: cells [0, n) lead the internal order), else the Morton-brick instance
    if (DEG == 6 && kl == nullptr && !(h.sharded() && h.klist != h.clist) && h.use_k1_brick()) {
      k_grad_limit_brick<P><<<fixed ? h.grid_k1b : std::min<long long>(h.grid_k1b, (nk + kBrick - 1) / kBrick),
                              kBrick, BrickSmem<P::NV>::bytes, h.st>>>(md, sd, h.brick_dev(), nkp, pred ? 1 : 0,
                                                                      h.next_dir());
      if (h.brick_rest_host > 0) {  // ragged bricks and the tail cells: the general kernel over their list
        k_grad_limit<P, DEG, false><<<h.grid_for(h.brick_rest_host, 128), 128, 0, h.st>>>(
            md, sd, h.brick_rest, h.brick_nrest, 0, front, pred ? 1 : 0, 0);
        ++h.launches;
      }
    } else if (DEG == 6 && kl == nullptr && h.use_k1_tile())
      k_grad_limit<P, DEG, true><<<g1, 128, 0, h.st>>>(md, sd, kl, nkp, 0, front, pred ? 1 : 0, h.next_dir());
    else
      k_grad_limit<P, DEG, false><<<g1, 128, 0, h.st>>>(md, sd, kl, nkp, 0, front, pred ? 1 : 0, h.next_dir());
  }, na, nf, nfr);
  const PlanDev* cpl = h.dplan;
  // shards with a halo: deep / border K1 lists and interior / border K2
  // lists (a shard without halo cells -- one rank -- runs the single-domain
  // lists and only joins the (empty) exchange)
  const bool split = h.sharded() && h.klist != h.clist;
  if (h.sharded() && !split) halo_join(h);
  if (split) {
    // interior faces while the halo is in flight
    timed(h, pred ? tafv_gpu::kK2P : tafv_gpu::kK2C, [&] {
      const int* fil = all ? nullptr : h.filist;
      const int* nfip = &h.dplan->nfi_prefix[level];
      if (pred) k_face_flux<P, true><<<g2, 128, 0, h.st>>>(md, sd, h.pp, fil, nfip, 0, front, cpl, 0);
      else k_face_flux<P, false><<<g2, 128, 0, h.st>>>(md, sd, h.pp, fil, nfip, 0, front, cpl, 0);
    }, 0, 0, 0);
    ++h.launches;
    // border cells (owned next to the halo, ring 1) once the halo landed
    halo_join(h);
    const int gb = fixed ? h.grid_k1 : h.grid_for(h.n_k1 - h.n_deep, 128);
    timed(h, tafv_gpu::kK1, [&] {
      if (DEG == 6 && kbl == nullptr && h.use_k1_tile())
        k_grad_limit<P, DEG, true><<<gb, 128, 0, h.st>>>(md, sd, kbl, nkbp, h.n_deep, front, pred ? 1 : 0, 0);
      else
        k_grad_limit<P, DEG, false><<<gb, 128, 0, h.st>>>(md, sd, kbl, nkbp, h.n_deep, front, pred ? 1 : 0, 0);
    }, 0, 0, 0);
    ++h.launches;
  }
  if (!pred) ledger_join(h);  // int_substep is about to be overwritten
  timed(h, pred ? tafv_gpu::kK2P : tafv_gpu::kK2C, [&] {
    const int r2 = h.next_dir();
    if (split) {  // the border faces, after the halo landed
      const int* fbl = all ? nullptr : h.fblist;
      const int* nfbp = &h.dplan->nfb_prefix[level];
      const int gb2 = fixed ? h.grid_k2 : h.grid_for(h.F_own - h.F_int, 128);
      if (pred) k_face_flux<P, true><<<gb2, 128, 0, h.st>>>(md, sd, h.pp, fbl, nfbp, h.F_int, front, cpl, r2);
      else k_face_flux<P, false><<<gb2, 128, 0, h.st>>>(md, sd, h.pp, fbl, nfbp, h.F_int, front, cpl, r2);
    } else {
      if (pred) k_face_flux<P, true><<<g2, 128, 0, h.st>>>(md, sd, h.pp, fl, nfp, 0, front, cpl, r2);
      else k_face_flux<P, false><<<g2, 128, 0, h.st>>>(md, sd, h.pp, fl, nfp, 0, front, cpl, r2);
    }
  }, na, nf, nfr);
  if (!pred) ledger_fork<P::NV>(h, level);
  if (last) {
    timed(h, tafv_gpu::kK3C, [&] {
      k_gather_update<P, false, true, DEG><<<h.nblk_last, 128, 0, h.st>>>(md, sd, nullptr, ncp,
                                                                          h.dplan, h.partials, 0);
    }, na, nf, 0);
    ledger_join(h);
    if (h.NB) {  // the ledger's outflow partials (a last-block merge into k_totals measured slower)
      k_ledger_reduce<P::NV><<<h.nblk_led, 256, 0, h.st>>>(h.bsum, h.NB, h.lpart);
      ++h.launches;
    }
    k_totals<<<P::NV, 256, 0, h.st>>>(h.partials, h.nblk_last, h.dplan, h.NB ? h.lpart : nullptr, h.nblk_led);
    h.launches += 4;  // K1, K2, K3 and the totals
    if (h.sharded()) {
      h.comm->allreduce_sum_f64(h.rank, h.dplan->totals, P::NV, h.st);
      h.comm->allreduce_sum_f64(h.rank, h.dplan->bflux, P::NV, h.st);
      h.comm->allreduce_max_i32(h.rank, &h.dplan->nonfinite, 1, h.st);
    }
    halo_rows(h, h.w, P::NV, true);  // the next iteration stages the halo's new w
  } else {
    timed(h, pred ? tafv_gpu::kK3P : tafv_gpu::kK3C, [&] {
      const int r3 = h.next_dir();
      if (pred)
        k_gather_update<P, true, false, DEG><<<g3, 128, 0, h.st>>>(md, sd, cl, ncp, h.dplan, h.partials, r3);
      else
        k_gather_update<P, false, false, DEG><<<g3, 128, 0, h.st>>>(md, sd, cl, ncp, h.dplan, h.partials, r3);
    }, na, nf, 0);
    h.launches += 3;
    // shards: the just-updated rows of owned cells to the peers' halos
    // (w_pred after a predictor, w after a corrector)
    halo_rows(h, pred ? h.wp : h.w, P::NV, false, level);
  }
}

template <class P>
void phase(tafv_gpu& h, bool pred, bool last, int level, int front) {
  const Range r(pred ? "tafv.phase.predictor" : (last ? "tafv.phase.trailing" : "tafv.phase.corrector"));
  if (h.deg6) phase_t<P, 6>(h, pred, last, level, front);
  else phase_t<P, 0>(h, pred, last, level, front);
}

template <class P>
void sweep(tafv_gpu& h) {
  const int subs = 1 << h.theta;
  for (int s = 1; s <= subs; ++s) {  // reference.cpp:108-120
    const int level = subiteration_level(s, h.theta);
    const int front = s - 1;
    if (s > 1) phase<P>(h, false, false, level, front);
    phase<P>(h, true, false, level, front);
  }
  phase<P>(h, false, true, h.theta, subs);  // trailing corrector, reference.cpp:121
}

void enqueue_sweep_direct(tafv_gpu& h) {
  h.dir_state = 1;  // the sweep's first kernel walks forwards (fixed per graph)
  CK(cudaMemsetAsync(&h.dplan->nonfinite, 0, sizeof(int), h.st));
  switch (h.model) {
    case TAFV_ADVECTION: sweep<Advection2D>(h); break;
    case TAFV_BURGERS: sweep<Burgers2D>(h); break;
    default: sweep<Euler3D>(h); break;
  }
  CK(cudaGetLastError());
}

// The whole 2^theta subiteration sweep as one CUDA graph per theta: every
// launch reads its active count and dt from the device plan, so the graph
// captured once replays for every later iteration with the same theta.
void run_sweep(tafv_gpu& h) {
  const Range r(h.sharded() ? "tafv.sweep.shard" : "tafv.sweep");
  // shards with level-sorted exchanges: the message sizes change with every
  // plan, so the sweep is launched directly (NCCL counts are fixed in a graph)
  if (!h.use_graph || (h.sharded() && (!h.comm->capturable() || h.xfilter))) {
    enqueue_sweep_direct(h);
    return;
  }
  const int key = 2 * h.theta + (h.ktime ? 1 : 0);
  auto it = h.graphs.find(key);
  if (it == h.graphs.end()) {
    tafv_gpu::GraphRec rec;
    cudaGraph_t g;
    h.capturing = true;
    h.cap = &rec;
    const int64_t l0 = h.launches;
    CK(cudaStreamBeginCapture(h.st, cudaStreamCaptureModeThreadLocal));
    enqueue_sweep_direct(h);
    const cudaError_t e = cudaStreamEndCapture(h.st, &g);
    h.capturing = false;
    h.cap = nullptr;
    CK(e);
    // node priorities: the halo exchange captured from the high-priority
    // comm stream keeps its priority over the K1 it overlaps
    CK(cudaGraphInstantiate(&rec.exec, g, cudaGraphInstantiateFlagUseNodePriority));
    CK(cudaGraphDestroy(g));
    rec.launches = h.launches - l0;
    h.launches = l0;
    it = h.graphs.emplace(key, std::move(rec)).first;
  }
  CK(cudaGraphLaunch(it->second.exec, h.st));
  h.launches += it->second.launches;
  if (h.ktime) h.pending_graph = &it->second;
}

void close_iteration(tafv_gpu& h, tafv_record* rec) {
  if (h.hplan->nonfinite) {
    h.has_plan = false;
    throw Error{TAFV_EDIVERGED, "integrate: solution diverged to a non-finite state"};
  }
  const double t_start = h.t0;
  h.t0 = t_start + h.dt * (double)(1 << h.theta);
  h.iteration += 1;
  if (rec) {
    tafv_plan_info pi;
    fill_plan_info(h, &pi);
    std::memset(rec, 0, sizeof *rec);
    rec->iteration = h.iteration;
    rec->t_start = t_start;
    rec->dt = h.dt;
    rec->theta = h.theta;
    rec->advance = h.dt * (double)(1 << h.theta);
    rec->cost_ratio = pi.cost_ratio;
    rec->nv = h.nv;
    for (int k = 0; k < h.nv; ++k) rec->total_extensive[k] = h.hplan->totals[k];
    for (int k = 0; k < h.nv; ++k) rec->boundary_flux[k] = h.hplan->bflux[k];
    rec->n_levels = h.theta + 1;
    for (int l = 0; l <= h.theta; ++l) rec->level_cells[l] = h.gcount[l];
  }
}

void run_iteration(tafv_gpu& h, tafv_record* rec) {
  require(h.has_plan, "run_iteration: no plan (call tafv_gpu_plan or tafv_gpu_inject_levels)");
  CK(cudaEventRecord(h.ev[0], h.st));
  run_sweep(h);
  CK(cudaEventRecord(h.ev[1], h.st));
  store_plan(h);
  CK(cudaStreamSynchronize(h.st));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h.ev[0], h.ev[1]));
  h.ms[2] += ms;
  collect_times(h);
  close_iteration(h, rec);
}

// reference_integrate as a pipelined loop: the plan of iteration i+1 is
// enqueued right behind sweep i and ONE read-back carries both plan i+1 and
// sweep i's divergence flag and totals, so the host waits once per iteration.
// Semantics match the sequential loop: iteration i's divergence is reported
// before plan i+1's errors, and the state is left as the reference leaves it.
void integrate_pipelined(tafv_gpu& h, const tafv_options& opt, int n, tafv_record* out,
                         bool keep_all) {
  if (n <= 0) return;
  enqueue_plan(h, opt);
  CK(cudaStreamSynchronize(h.st));
  check_plan(h);
  for (int i = 0; i < n; ++i) {
    // snapshot the plan that drives sweep i (the next plan overwrites h.*)
    const int theta = h.theta;
    const double dt = h.dt;
    long long cc[kMaxLevels], gc[kMaxLevels];
    std::memcpy(cc, h.ccount, sizeof cc);
    std::memcpy(gc, h.gcount, sizeof gc);
    run_sweep(h);
    const bool more = i + 1 < n;
    if (more) {
      enqueue_plan(h, opt);
    } else {
      store_plan(h);
    }
    CK(cudaStreamSynchronize(h.st));
    collect_times(h);
    // close iteration i with its own plan
    const int th_next = h.theta;
    const double dt_next = h.dt;
    long long cc_next[kMaxLevels], gc_next[kMaxLevels];
    std::memcpy(cc_next, h.ccount, sizeof cc_next);
    std::memcpy(gc_next, h.gcount, sizeof gc_next);
    h.theta = theta;
    h.dt = dt;
    std::memcpy(h.ccount, cc, sizeof cc);
    std::memcpy(h.gcount, gc, sizeof gc);
    close_iteration(h, (keep_all || !more) && out ? (keep_all ? out + i : out) : nullptr);
    if (more) {
      h.theta = th_next;
      h.dt = dt_next;
      std::memcpy(h.ccount, cc_next, sizeof cc_next);
      std::memcpy(h.gcount, gc_next, sizeof gc_next);
      check_plan(h);
    }
  }
}

// Whole-call device time: events on the library stream bracket every
// iteration, host syncs (the per-iteration plan read-back) included.
template <class F>
void timed_call(tafv_gpu& h, F&& body) {
  h.launches = 0;
  h.ms[0] = h.ms[1] = h.ms[2] = 0;
  CK(cudaEventRecord(h.ev[4], h.st));
  body();
  CK(cudaEventRecord(h.ev[5], h.st));
  CK(cudaEventSynchronize(h.ev[5]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h.ev[4], h.ev[5]));
  h.ms[0] = ms;
}

template <class F>
int guard(tafv_gpu* h, F&& f) {
  if (!h) return TAFV_EINVAL;
  try {
    CK(cudaSetDevice(h->device));
    f();
    return TAFV_OK;
  } catch (const Error& e) {
    h->err = e.what;
    return e.code;
  } catch (const std::bad_alloc&) {
    h->err = "host allocation failed";
    return TAFV_ECUDA;
  } catch (const std::exception& e) {
    h->err = e.what();
    return TAFV_ECUDA;
  }
}

}  // namespace

extern "C" {

// Shared by tafv_gpu_create and tafv_gpu_create_shard. `shard` (optional)
// makes the handle a rank of a decomposed run.
// Builds a handle's device resources in place (throws). `shard` (optional)
// makes the handle a rank of a decomposed run. Shared by tafv_gpu_create,
// tafv_gpu_create_shard and the in-place rebuild of tafv_gpu_repartition.
static void init_handle(tafv_gpu* h, const tafv_mesh_view* mesh, const tafv_physics* physics, int device,
                        const tafv::Shard* shard, tafv_comm* comm, int n_global) {
  h->device = device;
  h->phys = *physics;
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
  {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&h->cst, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&h->ev_pack, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming));
  }
  CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device));
  h->grid_cap = h->sms * 16;
  h->model = physics->model;
  switch (physics->model) {
    case TAFV_ADVECTION:
      h->nv = 1;
      h->pp.ax = physics->a[0];
      h->pp.ay = physics->a[1];
      break;
    case TAFV_BURGERS: {  // parse_flux_model (physics.cpp:13-17)
      h->nv = 1;
      const double len = std::sqrt(physics->a[0] * physics->a[0] + physics->a[1] * physics->a[1]);
      require(len > 0.0, "physics: burgers direction must be nonzero");
      h->pp.ax = physics->a[0] / len;
      h->pp.ay = physics->a[1] / len;
      break;
    }
    case TAFV_EULER:
      require(physics->gamma > 1.0, "physics: gamma must exceed 1");
      h->nv = 5;
      h->pp.gamma = physics->gamma;
      h->pp.gm1 = physics->gamma - 1.0;
      break;
    default:
      require(false, "physics: unknown model");
  }
  if (h->model != TAFV_EULER) require(mesh->dim <= 2, "physics: scalar models run on 1D/2D meshes");
  else require(mesh->dim == 3, "physics: Euler runs on 3D meshes");
  if (shard) {
    std::vector<uint8_t> touch(shard->touch_own.begin(), shard->touch_own.end());
    upload_mesh(*h, *mesh, shard->cls.data(), touch.data());
    h->comm = comm;
    h->rank = shard->rank;
    h->nranks = shard->nranks;
    h->N_global = n_global;
    h->shard_cells = shard->cells;
    // exchange lists in internal ids, peer segments in shard order
    std::vector<int> cinv(h->N);
    for (int i = 0; i < h->N; ++i) cinv[h->cperm[i]] = i;
    std::vector<int> sidx, ridx;
    for (size_t p = 0; p < shard->peers.size(); ++p) {
      tafv_gpu::Peer pe{shard->peers[p], (int)shard->send[p].size(), (int)shard->recv[p].size(),
                        (int)sidx.size(), (int)ridx.size()};
      for (int c : shard->send[p]) sidx.push_back(cinv[c]);
      for (int c : shard->recv[p]) ridx.push_back(cinv[c]);
      h->peers.push_back(pe);
    }
    h->send_total = (int)sidx.size();
    h->recv_total = (int)ridx.size();
    h->d_send_idx = dalloc<int>(sidx.size());
    h->d_recv_idx = dalloc<int>(ridx.size());
    if (!sidx.empty()) CK(cudaMemcpy(h->d_send_idx, sidx.data(), sidx.size() * 4, cudaMemcpyHostToDevice));
    if (!ridx.empty()) CK(cudaMemcpy(h->d_recv_idx, ridx.data(), ridx.size() * 4, cudaMemcpyHostToDevice));
    const int width = std::max(h->nv, 1);
    h->sendbuf = dalloc<double>((size_t)std::max(1, h->send_total) * width);
    h->recvbuf = dalloc<double>((size_t)std::max(1, h->recv_total) * width);
    comm->attach(h->rank, h);
  } else {
    upload_mesh(*h, *mesh);
  }
  alloc_state(*h);
  set_grids(*h);
}

static int create_handle(const tafv_mesh_view* mesh, const tafv_physics* physics, int device,
                         const tafv::Shard* shard, tafv_comm* comm, int n_global, tafv_gpu** out) {
  if (!out || !mesh || !physics) {
    g_create_error = "tafv_gpu_create: null argument";
    return TAFV_EINVAL;
  }
  *out = nullptr;
  auto* h = new tafv_gpu;
  h->device = device;
  try {
    init_handle(h, mesh, physics, device, shard, comm, n_global);
  } catch (const Error& e) {
    g_create_error = e.what;
    delete h;
    return e.code;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    delete h;
    return TAFV_ECUDA;
  }
  *out = h;
  return TAFV_OK;
}

int tafv_gpu_create(const tafv_mesh_view* mesh, const tafv_physics* physics, int device,
                    tafv_gpu** out) {
  return create_handle(mesh, physics, device, nullptr, nullptr, 0, out);
}

int tafv_comm_create_loopback(int32_t nranks, tafv_comm** out) {
  if (!out || nranks < 1) return TAFV_EINVAL;
  *out = make_loopback_comm(nranks);
  return TAFV_OK;
}

int tafv_comm_nccl_unique_id(uint8_t* out128) {
  if (!out128) return TAFV_EINVAL;
  return nccl_unique_id(out128);
}

int tafv_comm_create_nccl(const uint8_t* id128, int32_t rank, int32_t nranks, int device,
                          tafv_comm** out) {
  if (!out || !id128 || rank < 0 || rank >= nranks) return TAFV_EINVAL;
  try {
    CK(cudaSetDevice(device));
    *out = make_nccl_comm(id128, rank, nranks);
  } catch (const Error& e) {
    g_create_error = e.what;
    return e.code;
  }
  return TAFV_OK;
}

void tafv_comm_destroy(tafv_comm* c) { delete c; }

int tafv_gpu_create_shard(const tafv_mesh_view* global_mesh, const tafv_physics* physics, int device,
                          const int32_t* rank_of_cell, int32_t rank, tafv_comm* comm, tafv_gpu** out) {
  if (!global_mesh || !rank_of_cell || !comm || !out) {
    g_create_error = "tafv_gpu_create_shard: null argument";
    return TAFV_EINVAL;
  }
  try {
    const tafv::Shard sh = tafv::build_shard(*global_mesh, rank_of_cell, rank, comm->nranks());
    const tafv_mesh_view lv = sh.view(global_mesh->dim);
    return create_handle(&lv, physics, device, &sh, comm, global_mesh->n_cells, out);
  } catch (const std::invalid_argument& e) {
    g_create_error = e.what();
    return TAFV_EINVAL;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    return TAFV_ELOGIC;
  }
}

void tafv_gpu_destroy(tafv_gpu* h) { delete h; }

const char* tafv_gpu_last_error(const tafv_gpu* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

int tafv_gpu_set_state(tafv_gpu* h, const double* w_in, const double* W_in, double t0,
                       int32_t iteration) {
  return guard(h, [&] {
    require(w_in != nullptr || W_in != nullptr, "set_state: w and W are both null");
    // shards take the GLOBAL state and keep their local cells' rows
    std::vector<double> wl, Wl;
    const double* w = w_in;
    const double* W = W_in;
    if (h->sharded()) {
      auto local = [&](const double* src, std::vector<double>& dst) {
        dst.resize((size_t)h->N * h->nv);
        for (int i = 0; i < h->N; ++i)
          std::memcpy(&dst[(size_t)i * h->nv], src + (size_t)h->shard_cells[i] * h->nv, h->nv * sizeof(double));
        return dst.data();
      };
      if (w_in) w = local(w_in, wl);
      if (W_in) W = local(W_in, Wl);
    }
    const size_t n = (size_t)h->N * h->nv;
    double* stage = h->staging(n);
    if (w) {
      CK(cudaMemcpyAsync(stage, w, n * sizeof(double), cudaMemcpyHostToDevice, h->st));
      k_gather_rows<<<h->grid_for((long long)n, 256), 256, 0, h->st>>>(stage, h->d_cperm, h->N, h->nv, h->w);
    }
    if (W) {
      CK(cudaMemcpyAsync(stage, W, n * sizeof(double), cudaMemcpyHostToDevice, h->st));
      k_gather_rows<<<h->grid_for((long long)n, 256), 256, 0, h->st>>>(stage, h->d_cperm, h->N, h->nv, h->W);
      if (!w)  // w = W / V, the relation every corrector leaves (kernels.cpp:237-241)
        k_intensive<<<h->grid_for((long long)n, 256), 256, 0, h->st>>>(h->W, h->vol, h->N, h->nv, h->w);
    } else {
      k_sync_extensive<<<h->grid_for((long long)n, 256), 256, 0, h->st>>>(h->w, h->vol, h->N, h->nv, h->W);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->st));
    h->t0 = t0;
    h->iteration = iteration;
    h->state_set = true;
    h->has_plan = false;
  });
}

int tafv_gpu_get_state(tafv_gpu* h, double* w_out, double* W_out, double* t0, int32_t* iteration) {
  return guard(h, [&] {
    const size_t n = (size_t)h->N * h->nv;
    // shards write their OWNED rows into the global arrays
    std::vector<double> wl, Wl;
    double* w = w_out;
    double* W = W_out;
    if (h->sharded()) {
      if (w_out) {
        wl.resize(n);
        w = wl.data();
      }
      if (W_out) {
        Wl.resize(n);
        W = Wl.data();
      }
    }
    double* stage = h->staging(n);
    if (w) {
      k_scatter_rows<<<h->grid_for((long long)n, 256), 256, 0, h->st>>>(h->w, h->d_cperm, h->N, h->nv, stage);
      CK(cudaMemcpyAsync(w, stage, n * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    }
    if (W) {
      k_scatter_rows<<<h->grid_for((long long)n, 256), 256, 0, h->st>>>(h->W, h->d_cperm, h->N, h->nv, stage);
      CK(cudaMemcpyAsync(W, stage, n * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    }
    CK(cudaStreamSynchronize(h->st));
    if (h->sharded()) {
      std::vector<int> cinv(h->N);
      for (int i = 0; i < h->N; ++i) cinv[h->cperm[i]] = i;
      for (int c = 0; c < h->N; ++c) {
        if (cinv[c] >= h->n_own) continue;  // owned cells lead the internal order
        const size_t g = (size_t)h->shard_cells[c] * h->nv;
        if (w_out) std::memcpy(w_out + g, &wl[(size_t)c * h->nv], h->nv * sizeof(double));
        if (W_out) std::memcpy(W_out + g, &Wl[(size_t)c * h->nv], h->nv * sizeof(double));
      }
    }
    if (t0) *t0 = h->t0;
    if (iteration) *iteration = h->iteration;
  });
}

int tafv_gpu_plan(tafv_gpu* h, const tafv_options* opt, tafv_plan_info* out) {
  return guard(h, [&] {
    require(opt != nullptr, "plan: null options");
    h->launches = 0;
    plan(*h, *opt);
    fill_plan_info(*h, out);
  });
}

int tafv_gpu_inject_levels(tafv_gpu* h, const int32_t* tau, double dt, const tafv_options* opt,
                           tafv_plan_info* out) {
  return guard(h, [&] {
    require(tau != nullptr, "inject_levels: tau is null");
    inject(*h, tau, dt, opt);
    fill_plan_info(*h, out);
  });
}

int tafv_gpu_get_plan_lists(tafv_gpu* h, int32_t* tau_out, int32_t* cad_out, int32_t* cells_flat,
                            int32_t* faces_flat, int32_t* fringe_flat) {
  return guard(h, [&] {
    require(h->has_plan, "get_plan_lists: no plan");
    std::vector<int8_t> tau(h->N), cad(h->F);
    CK(cudaMemcpy(tau.data(), h->tau, h->N, cudaMemcpyDeviceToHost));
    if (h->F) CK(cudaMemcpy(cad.data(), h->cad, h->F, cudaMemcpyDeviceToHost));
    if (tau_out)
      for (int i = 0; i < h->N; ++i) tau_out[h->cperm[i]] = tau[i];
    if (cad_out)
      for (int j = 0; j < h->F; ++j) cad_out[h->fperm[j]] = cad[j];
    const int L = h->theta + 1;
    // Device lists (internal ids, level-sorted) -> original ids, ascending per level.
    auto export_list = [&](const int* dlist, long long n_total, const long long* counts,
                           const std::vector<int>& perm, int32_t* out, const std::vector<int8_t>& key,
                           long long n_items) {
      std::vector<int> lst(n_total);
      if (n_total) CK(cudaMemcpy(lst.data(), dlist, n_total * sizeof(int), cudaMemcpyDeviceToHost));
      if (h->lists_skip_top) {
        // the device list has no entries for the top level theta (never read
        // there): the items with key == theta in ascending internal id, which
        // is what the stable compaction would have written
        long long o = 0;
        for (int l = 0; l < h->theta; ++l) o += counts[l];
        for (long long i = 0; i < n_items; ++i)
          if (key[i] == h->theta) lst[o++] = (int)i;
        if (o != n_total) throw std::logic_error("plan lists: top-level count mismatch");
      }
      long long o = 0;
      for (int l = 0; l < L; ++l) {
        for (long long i = o; i < o + counts[l]; ++i) out[i] = perm[lst[i]];
        std::sort(out + o, out + o + counts[l]);
        o += counts[l];
      }
    };
    long long nc = 0, nf = 0;
    for (int l = 0; l < L; ++l) {
      nc += h->ccount[l];
      nf += h->fcount[l];
    }
    if (cells_flat) export_list(h->clist, nc, h->ccount, h->cperm, cells_flat, tau, h->n_own);
    if (faces_flat) export_list(h->flist, nf, h->fcount, h->fperm, faces_flat, cad, h->F_own);
    if (fringe_flat) {
      // fringe[l]: cells of level l+1 flagged by a level-l face neighbour
      // (levels.cpp:139-153), from the device flags.
      std::vector<uint8_t> flag(h->N);
      CK(cudaMemcpy(flag.data(), h->fflag, h->N, cudaMemcpyDeviceToHost));
      std::vector<std::vector<int>> fr(std::max(0, h->theta));
      for (int i = 0; i < h->N; ++i)
        if (flag[i] && tau[i] > 0 && tau[i] - 1 < h->theta) fr[tau[i] - 1].push_back(h->cperm[i]);
      long long o = 0;
      for (auto& v : fr) {
        std::sort(v.begin(), v.end());
        std::copy(v.begin(), v.end(), fringe_flat + o);
        o += (long long)v.size();
      }
    }
  });
}

int tafv_gpu_run_iteration(tafv_gpu* h, tafv_record* out) {
  return guard(h, [&] {
    h->launches = 0;
    h->ms[0] = h->ms[1] = h->ms[2] = 0;
    run_iteration(*h, out);
  });
}

// ---- in-library repartition (DistDriver::repartition, exchange.cpp:595-609)
// Every rank publishes its owned rows of W (as bit patterns, so the sum
// with the other ranks' zeros is exact, signed zeros included) and its owned
// cells' levels into global device buffers; all-reduces over the shard
// communicator give every rank the global committed state and the last
// plan's level map (the reference's sync_doubles of w / W); the level cost
// 2^(theta - tau) cuts new slabs (exchange.cpp:598-603) unless the caller
// passes a partition; the handle is rebuilt IN PLACE from the global mesh
// (shard description, device mesh build, state, graphs) and restored to the
// same W (w = W / V, the relation every corrector leaves), t0 and iteration.
__global__ void k_publish_owned(const double* __restrict__ W, const int8_t* __restrict__ tau,
                                const int* __restrict__ gid, int n_own, int nv, long long* gW, int* gtau) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_own; i += gridDim.x * blockDim.x) {
    const size_t g = (size_t)gid[i];
    for (int k = 0; k < nv; ++k) gW[g * nv + k] = __double_as_longlong(W[(size_t)i * nv + k]);
    gtau[g] = tau[i];
  }
}

static void repartition(tafv_gpu* h, const tafv_mesh_view* gm, const int32_t* roc_in, int axis,
                        int32_t* roc_out) {
  const auto t_start = std::chrono::steady_clock::now();
  require(h->sharded(), "repartition: the handle is not a shard (tafv_gpu_create_shard)");
  require(gm != nullptr && gm->n_cells == h->N_global, "repartition: global mesh differs from the shard's");
  if (!h->levels_made) throw Error{TAFV_ELOGIC, "dist: repartition before any iteration"};
  require(h->state_set, "repartition: no state");
  const int NG = h->N_global, nv = h->nv;
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->st));
  // 1. global committed state and last plan's levels on every rank
  std::vector<int> gid(h->n_own);
  for (int i = 0; i < h->n_own; ++i) gid[i] = h->shard_cells[h->cperm[i]];
  int* dgid = dalloc<int>(std::max(1, h->n_own));
  long long* gWb = dalloc<long long>((size_t)NG * nv);
  int* gtau = dalloc<int>(NG);
  std::vector<long long> hW((size_t)NG * nv);
  std::vector<int> htau(NG);
  try {
    if (h->n_own) CK(cudaMemcpy(dgid, gid.data(), gid.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemsetAsync(gWb, 0, (size_t)NG * nv * 8, h->st));
    CK(cudaMemsetAsync(gtau, 0xff, (size_t)NG * 4, h->st));
    k_publish_owned<<<h->grid_for(h->n_own, 256), 256, 0, h->st>>>(h->W, h->tau, dgid, h->n_own, nv, gWb, gtau);
    CK(cudaGetLastError());
    h->comm->allreduce_sum_i64(h->rank, gWb, NG * nv, h->st);
    h->comm->allreduce_max_i32(h->rank, gtau, NG, h->st);
    CK(cudaMemcpyAsync(hW.data(), gWb, hW.size() * 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaMemcpyAsync(htau.data(), gtau, htau.size() * 4, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
  } catch (...) {
    cudaFree(dgid);
    cudaFree(gWb);
    cudaFree(gtau);
    throw;
  }
  cudaFree(dgid);
  cudaFree(gWb);
  cudaFree(gtau);
  for (int c = 0; c < NG; ++c) require(htau[c] >= 0, "repartition: a cell is owned by no rank");
  // 2. the new partition: the caller's, or level-cost slabs
  std::vector<int32_t> roc(NG);
  if (roc_in) {
    for (int c = 0; c < NG; ++c) {
      require(roc_in[c] >= 0 && roc_in[c] < h->nranks, "repartition: rank_of_cell out of range");
      roc[c] = roc_in[c];
    }
  } else {
    int theta = 0;
    for (int c = 0; c < NG; ++c) theta = std::max(theta, htau[c]);
    std::vector<double> wgt(NG);
    for (int c = 0; c < NG; ++c) wgt[c] = (double)(1ll << (theta - htau[c]));
    tafv::partition_slabs(*gm, h->nranks, axis, wgt.data(), roc.data());
  }
  if (roc_out) std::memcpy(roc_out, roc.data(), (size_t)NG * 4);
  // 3. the new shard (host description first: a bad partition leaves the
  // handle untouched), then the in-place rebuild
  const tafv::Shard sh = tafv::build_shard(*gm, roc.data(), h->rank, h->nranks);
  const tafv_mesh_view lv = sh.view(gm->dim);
  std::vector<double> Wg((size_t)NG * nv);
  std::memcpy(Wg.data(), hW.data(), Wg.size() * 8);
  hW.clear();
  hW.shrink_to_fit();
  const double t0 = h->t0;
  const int iteration = h->iteration;
  tafv_comm* comm = h->comm;
  const int device = h->device;
  const tafv_physics phys = h->phys;
  const bool use_graph = h->use_graph, plan_graph_on = h->plan_graph_on, slot_geo = h->slot_geo,
             slot_n = h->slot_n, slot_dx = h->slot_dx, face_dx = h->face_dx, alt_dir = h->alt_dir,
             iwin_alias = h->iwin_alias;
  const int dl_stream = h->dl_stream, batch_lanes = h->batch_lanes, k1_tile = h->k1_tile;
  const tafv_mesh_view* rep_mesh = h->rep_mesh;
  const int rep_every = h->rep_every, rep_axis = h->rep_axis;
  h->release();
  *h = tafv_gpu{};
  h->use_graph = use_graph;
  h->plan_graph_on = plan_graph_on;
  h->slot_geo = slot_geo;
  h->slot_n = slot_n;
  h->slot_dx = slot_dx;
  h->face_dx = face_dx;
  h->alt_dir = alt_dir;
  h->iwin_alias = iwin_alias;
  h->dl_stream = dl_stream;
  h->batch_lanes = batch_lanes;
  h->k1_tile = k1_tile;
  h->rep_mesh = rep_mesh;
  h->rep_every = rep_every;
  h->rep_axis = rep_axis;
  init_handle(h, &lv, &phys, device, &sh, comm, NG);
  const int rc = tafv_gpu_set_state(h, nullptr, Wg.data(), t0, iteration);
  if (rc != TAFV_OK) throw Error{rc, h->err};
  h->levels_made = true;  // the next plan_iteration rebuilds them; tau is the old map
  h->rep_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
}

int tafv_gpu_repartition(tafv_gpu* h, const tafv_mesh_view* global_mesh, const int32_t* rank_of_cell,
                         int32_t axis, int32_t* rank_of_cell_out) {
  return guard(h, [&] { repartition(h, global_mesh, rank_of_cell, axis, rank_of_cell_out); });
}

int tafv_gpu_set_repartition(tafv_gpu* h, const tafv_mesh_view* global_mesh, int32_t every, int32_t axis) {
  return guard(h, [&] {
    require(every >= 0, "repartition_every must be >= 0");
    require(every == 0 || h->sharded(), "repartition_every: the handle is not a shard");
    require(every == 0 || (global_mesh != nullptr && global_mesh->n_cells == h->N_global),
            "repartition_every: global mesh differs from the shard's");
    require(axis >= 0 && axis <= 2, "repartition_every: axis must be 0, 1 or 2");
    h->rep_mesh = every ? global_mesh : nullptr;
    h->rep_every = every;
    h->rep_axis = axis;
  });
}

int tafv_gpu_iterate(tafv_gpu* h, const tafv_options* opt, int32_t n, tafv_record* out) {
  return guard(h, [&] {
    require(opt != nullptr, "iterate: null options");
    require(n >= 0, "integrate: negative iteration count");
    if (h->rep_every > 0 && h->sharded()) {
      // DistDriver::integrate (exchange.cpp:611-618): repartition before
      // iteration i whenever i > 0 and i % repartition_every == 0
      int64_t launches = 0;
      double ms3[3] = {0, 0, 0};
      for (int i = 0; i < n; i += h->rep_every) {
        if (i > 0) repartition(h, h->rep_mesh, nullptr, h->rep_axis, nullptr);
        const int m = std::min<int>(h->rep_every, n - i);
        timed_call(*h, [&] { integrate_pipelined(*h, *opt, m, out ? out + i : nullptr, true); });
        launches += h->launches;
        for (int q = 0; q < 3; ++q) ms3[q] += h->ms[q];
      }
      h->launches = launches;
      for (int q = 0; q < 3; ++q) h->ms[q] = ms3[q];
      return;
    }
    timed_call(*h, [&] { integrate_pipelined(*h, *opt, n, out, true); });
  });
}

int tafv_gpu_advance(tafv_gpu* h, const tafv_options* opt, int32_t n, tafv_record* last) {
  return guard(h, [&] {
    require(opt != nullptr, "advance: null options");
    require(n >= 0, "integrate: negative iteration count");
    timed_call(*h, [&] { integrate_pipelined(*h, *opt, n, last, false); });
  });
}

// One whole iteration as ONE graph (single domain): the plan graph's
// kernels, a selector kernel that sets a switch condition to theta (or past
// the last case when the plan failed: stable step collapsed / level error),
// and a SWITCH node whose case theta is the captured sweep of that theta. No
// host round trip between plan and sweep.
void build_iter_graph(tafv_gpu& h, const tafv_options& opt) {
  if (h.iter_graph) CK(cudaGraphExecDestroy(h.iter_graph));
  h.iter_graph = nullptr;
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  CK(cudaGraphConditionalHandleCreate(&h.iter_cond, g, (unsigned)opt.theta_max + 1, cudaGraphCondAssignDefault));
  const int64_t l0 = h.launches;
  const int theta0 = h.theta;
  h.capturing = true;
  CK(cudaStreamBeginCaptureToGraph(h.st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  plan_kernels(h, opt);
  k_select_sweep<<<1, 32, 0, h.st>>>(h.dplan, h.iter_cond, opt.theta_max);
  CK(cudaStreamEndCapture(h.st, &g));
  size_t nn = 0;
  CK(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn), leaves;
  CK(cudaGraphGetNodes(g, nodes.data(), &nn));
  for (cudaGraphNode_t nd : nodes) {
    size_t nd_out = 0;
    CK(cudaGraphNodeGetDependentNodes(nd, nullptr, &nd_out));
    if (nd_out == 0) leaves.push_back(nd);
  }
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h.iter_cond;
  cp.conditional.type = cudaGraphCondTypeSwitch;
  cp.conditional.size = (unsigned)opt.theta_max + 1;
  cudaGraphNode_t cn;
  CK(cudaGraphAddNode(&cn, g, leaves.data(), leaves.size(), &cp));
  for (int th = 0; th <= opt.theta_max; ++th) {
    h.theta = th;  // the sweep's level sequence; counts come from the device plan
    CK(cudaStreamBeginCaptureToGraph(h.st, cp.conditional.phGraph_out[th], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    enqueue_sweep_direct(h);
    cudaGraph_t body;
    CK(cudaStreamEndCapture(h.st, &body));
  }
  h.capturing = false;
  h.theta = theta0;
  CK(cudaGraphInstantiate(&h.iter_graph, g, 0));
  CK(cudaGraphDestroy(g));
  h.iter_opt = opt;
  h.launches = l0;
}

// The run_batch twin of a single-domain handle (see tafv_gpu::twin), or
// null when the device lacks the memory for a second state.
tafv_gpu* make_twin(const tafv_gpu& h) {
  const size_t state_bytes = (size_t)h.N * (3 * h.nv + h.gs + 8) * sizeof(double) +
                             (size_t)h.F * (3 * h.fs + 4) * sizeof(double) +
                             2 * 2 * (size_t)h.N * h.nv * sizeof(double);
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  if (free_b < state_bytes + state_bytes / 2 + ((size_t)1 << 30)) return nullptr;
  auto* t = new tafv_gpu;
  try {
    t->device = h.device;
    CK(cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking));
    t->model = h.model;
    t->nv = h.nv;
    t->dim = h.dim;
    t->pp = h.pp;
    t->N = h.N;
    t->F = h.F;
    t->M = h.M;
    t->periodic = h.periodic;
    t->sms = h.sms;
    t->grid_cap = h.grid_cap;
    t->vol_host = h.vol_host;
    t->owns_mesh = false;
    t->vol = h.vol;
    t->ivol = h.ivol;
    t->cen = h.cen;
    t->chl = h.chl;
    t->fcen = h.fcen;
    t->deg6 = h.deg6;
    t->adj_off = h.adj_off;
    t->adj_face = h.adj_face;
    t->adj_nb = h.adj_nb;
    t->lr = h.lr;
    t->rcf = h.rcf;
    t->geo = h.geo;
    t->sgeo = h.sgeo;
    t->sdx = h.sdx;
    t->fdx = h.fdx;
    t->brick_idx = h.brick_idx;
    t->brick_halo = h.brick_halo;
    t->brick_geo = h.brick_geo;
    t->brick_fcen = h.brick_fcen;
    t->brick_info = h.brick_info;
    t->brick_rest = h.brick_rest;
    t->brick_nrest = h.brick_nrest;
    t->brick_rest_host = h.brick_rest_host;
    t->nbricks = h.nbricks;
    t->k1_brick = h.k1_brick;
    t->d_cperm = h.d_cperm;
    t->d_fperm = h.d_fperm;
    t->slot_geo = h.slot_geo;
    t->slot_n = h.slot_n;
    t->k1_tile = h.k1_tile;
    t->slot_dx = h.slot_dx;
    t->face_dx = h.face_dx;
    t->iwin_alias = h.iwin_alias;
    t->alt_dir = h.alt_dir;
    t->use_graph = h.use_graph;
    t->plan_graph_on = h.plan_graph_on;
    t->dl_stream = h.dl_stream;
    t->n_deep = h.n_deep;
    t->n_own = h.n_own;
    t->n_k1 = h.n_k1;
    t->F_own = h.F_own;
    t->F_int = h.F_int;
    t->N_global = h.N_global;
    t->NB = h.NB;
    t->bface = h.bface;
    alloc_state(*t);
    set_grids(*t);
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

// Run-batch staging of one lane: copy streams, double-buffered device
// input / output rows, their events; one-graph iteration and plan copies.
void batch_setup(tafv_gpu& g, const tafv_options& opt, size_t n_plans, bool one_graph) {
  const size_t n = (size_t)g.N * g.nv;
  if (!g.cin) {
    CK(cudaStreamCreateWithFlags(&g.cin, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&g.cout, cudaStreamNonBlocking));
    for (int q = 0; q < 2; ++q) {
      g.bin[q] = dalloc<double>(n);
      g.bout[q] = dalloc<double>(n);
      for (cudaEvent_t* e : {&g.ev_in[q], &g.ev_in_free[q], &g.ev_out[q], &g.ev_out_free[q]}) {
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CK(cudaEventRecord(*e, g.st));  // initially complete
      }
    }
  }
  if (one_graph) {
    const bool same = g.iter_graph && g.iter_opt.theta_max == opt.theta_max && g.iter_opt.cfl == opt.cfl &&
                      g.iter_opt.dt_cap == opt.dt_cap;
    if (!same) build_iter_graph(g, opt);
    if (n_plans > g.batch_cap) {
      if (g.batch_plans) CK(cudaFreeHost(g.batch_plans));
      CK(cudaMallocHost(&g.batch_plans, n_plans * sizeof(PlanDev)));
      g.batch_cap = n_plans;
    }
  }
}

// A batch of independent inputs through one handle, each `iterations`
// iterations from its own extensive state (w = W / V); input j+1 uploads on
// a copy stream while input j computes on the library stream.
int tafv_gpu_run_batch(tafv_gpu* h, const tafv_options* opt, int32_t n_inputs, int32_t iterations,
                       const double* const* W_in, double* const* W_out, tafv_record* last) {
  return guard(h, [&] {
    require(opt != nullptr && W_in != nullptr && W_out != nullptr, "run_batch: null argument");
    require(n_inputs >= 0 && iterations >= 1, "run_batch: counts");
    const size_t n = (size_t)h->N * h->nv, bytes = n * sizeof(double);
    // single domain: every iteration is one graph launch (plan + switch to
    // the sweep of its theta), no host synchronisation inside the batch, and
    // the inputs alternate between two lanes (this handle and its twin) that
    // run concurrently; the last input runs on this handle, so its state is
    // the last input's afterwards
    const bool one_graph = !h->sharded() && h->use_graph && h->plan_graph_on && !h->ktime;
    std::vector<tafv_gpu*> lanes{h};
    if (one_graph && n_inputs >= 2 && h->batch_lanes >= 2) {
      if (!h->twin) {
        try {
          h->twin = make_twin(*h);
        } catch (const Error&) {  // no room for a second state: one lane
          h->twin = nullptr;
          cudaGetLastError();
        }
      }
      if (h->twin) lanes.push_back(h->twin);
    }
    const int nl = (int)lanes.size();
    auto lane_of = [&](int j) { return (n_inputs - 1 - j) % nl; };
    std::vector<std::vector<int>> mine(nl);  // each lane's inputs, in order
    for (int j = 0; j < n_inputs; ++j) mine[lane_of(j)].push_back(j);
    for (int L = 0; L < nl; ++L) batch_setup(*lanes[L], *opt, mine[L].size() * (size_t)iterations, one_graph);

    auto upload = [&](int L, int i) {  // lane-local input i
      tafv_gpu& g = *lanes[L];
      const int q = i & 1;
      CK(cudaStreamWaitEvent(g.cin, g.ev_in_free[q], 0));
      // not under the previous download either (they share the link: measured)
      CK(cudaStreamWaitEvent(g.cin, g.ev_out_free[q], 0));  // download i - 2 of this slot pair = the one in flight
      CK(cudaMemcpyAsync(g.bin[q], W_in[mine[L][i]], bytes, cudaMemcpyHostToDevice, g.cin));
      CK(cudaEventRecord(g.ev_in[q], g.cin));
    };
    const int grid = h->grid_for((long long)n, 256);
    auto process = [&](int L, int i) {
      tafv_gpu& g = *lanes[L];
      const int j = mine[L][i];
      const int q = i & 1;
      if (i + 1 < (int)mine[L].size()) upload(L, i + 1);
      // state j: W from the staged input, w = W / V (kernels.cpp:237-241)
      CK(cudaStreamWaitEvent(g.st, g.ev_in[q], 0));
      k_load_extensive<<<grid, 256, 0, g.st>>>(g.bin[q], g.d_cperm, g.vol, g.N, g.nv, g.W, g.w);
      CK(cudaEventRecord(g.ev_in_free[q], g.st));
      g.t0 = 0.0;
      g.iteration = 0;
      g.state_set = true;
      g.has_plan = false;
      if (one_graph) {
        for (int it = 0; it < iterations; ++it) {
          CK(cudaGraphLaunch(g.iter_graph, g.st));
          // this iteration's plan + its sweep's flags and totals, stored by a
          // kernel into the pinned (device-mapped) host array: a copy-engine
          // transfer would queue behind the bulk downloads on the same engine
          k_store_plan<<<1, 128, 0, g.st>>>(g.dplan, &g.batch_plans[(size_t)i * iterations + it]);
        }
      } else {
        integrate_pipelined(g, *opt, iterations, j + 1 == n_inputs ? last : nullptr, false);
      }
      // output j: W in original order -> staging -> host on the download
      // copy stream, under the next input's compute. (A copy-engine read-back
      // of the plan on the library stream queued behind these downloads and
      // stalled it; the plan goes to the host by a kernel, store_plan.)
      CK(cudaStreamWaitEvent(g.st, g.ev_out_free[q], 0));
      k_scatter_rows<<<grid, 256, 0, g.st>>>(g.W, g.d_cperm, g.N, g.nv, g.bout[q]);
      if (g.dl_stream) {
        CK(cudaEventRecord(g.ev_out[q], g.st));
        CK(cudaStreamWaitEvent(g.cout, g.ev_out[q], 0));
        CK(cudaMemcpyAsync(W_out[j], g.bout[q], bytes, cudaMemcpyDeviceToHost, g.cout));
        CK(cudaEventRecord(g.ev_out_free[q], g.cout));
      } else {
        CK(cudaMemcpyAsync(W_out[j], g.bout[q], bytes, cudaMemcpyDeviceToHost, g.st));
        CK(cudaEventRecord(g.ev_out_free[q], g.st));
      }
    };
    try {
      for (int L = 0; L < nl; ++L)
        if (!mine[L].empty()) upload(L, 0);
      const int rounds = n_inputs == 0 ? 0 : (int)mine[0].size();
      for (int i = 0; i < rounds; ++i)
        for (int L = nl - 1; L >= 0; --L)  // input order: the twin's input precedes this handle's
          if (i < (int)mine[L].size()) process(L, i);
    } catch (...) {
      // copies from / into the CALLER's buffers may still be in flight on
      // the copy streams: drain every lane before the error reaches the
      // caller (who may free or reuse those buffers at once); secondary
      // errors are dropped, the first one is reported
      for (tafv_gpu* g : lanes)
        for (cudaStream_t q : {g->cin, g->cout, g->st})
          if (q) cudaStreamSynchronize(q);
      cudaGetLastError();
      throw;
    }
    for (tafv_gpu* g : lanes) {
      CK(cudaStreamSynchronize(g->cout));
      CK(cudaStreamSynchronize(g->cin));
      CK(cudaStreamSynchronize(g->st));
    }
    if (one_graph) {  // the plans and flags of every iteration, in input order
      std::vector<int> local(n_inputs);
      for (int L = 0; L < nl; ++L)
        for (size_t i = 0; i < mine[L].size(); ++i) local[mine[L][i]] = (int)i;
      for (int j = 0; j < n_inputs; ++j) {
        tafv_gpu& g = *lanes[lane_of(j)];
        g.t0 = 0.0;
        g.iteration = 0;
        for (int it = 0; it < iterations; ++it) {
          *g.hplan = g.batch_plans[(size_t)local[j] * iterations + it];
          g.plan_nkeys = opt->theta_max + 1;
          parse_plan(g);
          if (!(std::isfinite(g.dt) && g.dt > 0.0)) {
            g.has_plan = false;
            throw Error{TAFV_EINVAL, "integrate: stable step collapsed"};
          }
          close_iteration(g, j + 1 == n_inputs && it + 1 == iterations ? last : nullptr);
        }
        g.has_plan = false;
        g.raw_lazy = true;  // the last plan's raw levels, materialised on read
      }
    }
  });
}


// reference_integrate on a HOST-resident state (the caller's SolverState,
// state.hpp:17-50, kept on the host between iterations): every iteration
// uploads W from the caller's buffer (w = W / V on the device), runs one
// plan + sweep, and writes the new W back into the same buffer. The copies
// are chunked: chunk c of iteration i+1's upload starts as soon as chunk c
// of iteration i's download has landed in the host buffer, so the two
// directions of the link overlap (the bytes still make the full round trip
// through the caller's memory every iteration). W_host in the batch layout
// (original cell order; shards: local cells in shard order).
int tafv_gpu_iterate_host(tafv_gpu* h, const tafv_options* opt, int32_t n, double* W_host, tafv_record* out) {
  return guard(h, [&] {
    require(opt != nullptr && W_host != nullptr, "iterate_host: null argument");
    require(n >= 0, "integrate: negative iteration count");
    batch_setup(*h, *opt, 0, false);
    const size_t total = (size_t)h->N * h->nv;
    size_t chunk_mb = 64;
    if (const char* e = getenv("TAFV_E2E_CHUNK_MB")) chunk_mb = std::max(1, atoi(e));  // A/B
    // whole rows per chunk: each chunk is loaded / gathered on its own,
    // overlapped with the neighbouring chunks' copies
    const size_t crow = std::max<size_t>(1, (chunk_mb << 20) / (sizeof(double) * h->nv));
    const size_t chunk = std::min<size_t>(total, crow * h->nv);
    const int nchunks = (int)((total + chunk - 1) / chunk);
    while ((int)h->ev_chunk.size() < nchunks) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, h->cout));  // initially complete
      h->ev_chunk.push_back(e);
    }
    while ((int)h->ev_gather.size() < nchunks) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      h->ev_gather.push_back(e);
    }
    if (!h->d_cinv) {
      h->d_cinv = dalloc<int>(std::max(1, h->N));
      prep::k_invert<<<h->grid_for(h->N, 256), 256, 0, h->st>>>(h->d_cperm, h->N, h->d_cinv);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(h->st));
    }
    h->ms[0] = h->ms[1] = h->ms[2] = 0.0;
    h->launches = 0;
    // TAFV_E2E_TRACE: per-iteration stage times on stderr (upload, load,
    // plan + sweep, scatter, download), from events on the stages' streams
    const char* trace_env = getenv("TAFV_E2E_TRACE");
    const bool trace = trace_env != nullptr && atoi(trace_env) == 1;
    // TAFV_E2E_TRACE=2: an unsynchronised timeline (event per stage boundary
    // per iteration, printed at the end relative to the first)
    const bool tline = trace_env != nullptr && atoi(trace_env) == 2;
    std::vector<std::pair<const char*, cudaEvent_t>> tl;
    auto mark = [&](const char* what, cudaStream_t q) {
      if (!tline) return;
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      CK(cudaEventRecord(e, q));
      tl.emplace_back(what, e);
    };
    cudaEvent_t tev[6] = {};
    if (trace)
      for (auto& e : tev) CK(cudaEventCreate(&e));
    try {
      for (int it = 0; it < n; ++it) {
        mark("upload start", h->cin);
        if (trace) CK(cudaEventRecord(tev[0], h->cin));
        for (int c = 0; c < nchunks; ++c) {
          // upload chunk c once its previous download landed (which also
          // means its rows were gathered, so they may be overwritten), then
          // load it (W, w = W / V) behind the copy while chunk c + 1 uploads
          const size_t a = (size_t)c * chunk, len = std::min(chunk, total - a);
          CK(cudaStreamWaitEvent(h->cin, h->ev_chunk[c], 0));
          CK(cudaMemcpyAsync(h->bin[0] + a, W_host + a, len * sizeof(double), cudaMemcpyHostToDevice, h->cin));
          CK(cudaEventRecord(h->ev_gather[c], h->cin));  // (reused: chunk c landed)
          CK(cudaStreamWaitEvent(h->st, h->ev_gather[c], 0));
          k_load_extensive_chunk<<<h->grid_for((long long)len, 256), 256, 0, h->st>>>(
              h->bin[0] + a, h->d_cinv, h->vol, (long long)(a / h->nv), (long long)(len / h->nv), h->nv, h->W, h->w);
          CK(cudaGetLastError());
        }
        mark("uploads done", h->cin);
        mark("loads done", h->st);
        if (trace) CK(cudaEventRecord(tev[1], h->st));
        if (trace) CK(cudaEventRecord(tev[2], h->st));
        h->state_set = true;
        h->has_plan = false;
        const int64_t l0 = h->launches;
        double ms0[3] = {h->ms[0], h->ms[1], h->ms[2]};
        timed_call(*h, [&] { integrate_pipelined(*h, *opt, 1, out ? out + it : nullptr, true); });
        for (int q = 0; q < 3; ++q) h->ms[q] += ms0[q];
        h->launches += l0;
        mark("sweep done", h->st);
        if (trace) CK(cudaEventRecord(tev[3], h->st));
        // gather chunk c into original order on the library stream and
        // download it on the copy stream while chunk c + 1 is gathered
        for (int c = 0; c < nchunks; ++c) {
          const size_t a = (size_t)c * chunk, len = std::min(chunk, total - a);
          k_gather_orig_chunk<<<h->grid_for((long long)len, 256), 256, 0, h->st>>>(
              h->W, h->d_cinv, (long long)(a / h->nv), (long long)(len / h->nv), h->nv, h->bout[0] + a);
          CK(cudaGetLastError());
          CK(cudaEventRecord(h->ev_gather[c], h->st));
          CK(cudaStreamWaitEvent(h->cout, h->ev_gather[c], 0));
          if (c == 0) {
            if (trace) CK(cudaEventRecord(tev[4], h->cout));
            mark("first chunk gathered / downloads start", h->cout);
          }
          CK(cudaMemcpyAsync(W_host + a, h->bout[0] + a, len * sizeof(double), cudaMemcpyDeviceToHost, h->cout));
          CK(cudaEventRecord(h->ev_chunk[c], h->cout));
        }
        mark("downloads done", h->cout);
        if (trace) {
          CK(cudaEventRecord(tev[5], h->cout));
          CK(cudaEventSynchronize(tev[5]));
          float d[5];
          for (int q = 0; q < 5; ++q) CK(cudaEventElapsedTime(&d[q], tev[q], tev[q + 1]));
          fprintf(stderr, "E2E it %d upload %.2f load %.2f plan+sweep %.2f scatter %.2f download %.2f ms\n", it,
                  d[0], d[1], d[2], d[3], d[4]);
        }
      }
      if (trace)
        for (auto& e : tev) cudaEventDestroy(e);
      if (tline) {
        CK(cudaStreamSynchronize(h->cout));
        for (auto& m : tl) {
          float t = 0.f;
          CK(cudaEventElapsedTime(&t, tl[0].second, m.second));
          fprintf(stderr, "E2E %9.2f ms  %s\n", t, m.first);
        }
        for (auto& m : tl) cudaEventDestroy(m.second);
      }
      CK(cudaStreamSynchronize(h->cout));
    } catch (...) {
      // the caller's buffer may still be the target of a copy in flight
      for (cudaStream_t q : {h->cin, h->cout, h->st})
        if (q) cudaStreamSynchronize(q);
      cudaGetLastError();
      throw;
    }
  });
}

int tafv_gpu_get_array(tafv_gpu* h, const char* name, void* out) {
  return guard(h, [&] {
    require(name && out, "get_array: null argument");
    const std::string n = name;
    auto rows = [&](const double* src, int count, int width, const int* dperm) {
      const size_t total = (size_t)count * width;
      double* stage = h->staging(total);
      k_scatter_rows<<<h->grid_for((long long)total, 256), 256, 0, h->st>>>(src, dperm, count, width, stage);
      CK(cudaMemcpyAsync(out, stage, total * sizeof(double), cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
    };
    if (n == "w") rows(h->w, h->N, h->nv, h->d_cperm);
    else if (n == "W") rows(h->W, h->N, h->nv, h->d_cperm);
    else if (n == "repartition_ms") *static_cast<double*>(out) = h->rep_ms;
    else if (n == "brick_counts") {  // [nbricks][4] int32: face entries (-e - 1: ragged), halo rows, offsets
      if (h->brick_info)
        CK(cudaMemcpy(out, h->brick_info, (size_t)h->nbricks * sizeof(int4), cudaMemcpyDeviceToHost));
    } else if (n == "brick_info") {  // bricks, ragged bricks, cells left to the general K1, built
      double* o = static_cast<double*>(out);
      o[0] = h->nbricks;
      o[1] = h->brick_ragged;
      o[2] = h->brick_rest_host;
      o[3] = h->brick_idx != nullptr;
    }
    else if (n == "w_pred") rows(h->wp, h->N, h->nv, h->d_cperm);
    else if (n == "grad") {  // unpadded rows of nv*3
      const size_t w3 = (size_t)h->nv * 3;
      double* dense = dalloc<double>((size_t)h->N * w3);
      CK(cudaMemcpy2DAsync(dense, w3 * sizeof(double), h->grad, h->gs * sizeof(double), w3 * sizeof(double),
                           h->N, cudaMemcpyDeviceToDevice, h->st));
      rows(dense, h->N, (int)w3, h->d_cperm);
      cudaFree(dense);
    }
    else if (n == "dt_max") rows(h->dtmax, h->N, 1, h->d_cperm);
    else if (n == "phi_pred" || n == "int_substep") {  // padded rows -> nv wide
      double* dense = dalloc<double>((size_t)h->F * h->nv);
      CK(cudaMemcpy2DAsync(dense, h->nv * sizeof(double), n == "phi_pred" ? h->phi : h->isub,
                           h->fs * sizeof(double), h->nv * sizeof(double), h->F, cudaMemcpyDeviceToDevice, h->st));
      rows(dense, h->F, h->nv, h->d_fperm);
      cudaFree(dense);
    }
    else if (n == "int_window") {
      double* win = dalloc<double>((size_t)h->F * h->nv);
      k_window_rows<<<h->grid_for((long long)h->F * h->nv, 256), 256, 0, h->st>>>(h->iwin, h->isub,
                                                                             h->iwin_alias ? h->ialias : nullptr,
                                                                             h->F, h->nv, (int)h->fs, win);
      rows(win, h->F, h->nv, h->d_fperm);
      cudaFree(win);
    }
    else if (n == "mesh_digest") {
      // FNV-1a 64 of every internal mesh array (debug: host vs device build)
      auto fnv = [&](const void* dptr, size_t bytes) -> uint64_t {
        std::vector<unsigned char> v(bytes);
        if (bytes) CK(cudaMemcpy(v.data(), dptr, bytes, cudaMemcpyDeviceToHost));
        uint64_t x = 1469598103934665603ull;
        for (unsigned char c : v) x = (x ^ c) * 1099511628211ull;
        return x;
      };
      uint64_t* o = static_cast<uint64_t*>(out);
      const size_t N = h->N, F = h->F, M = h->M;
      const void* ptrs[] = {h->vol, h->ivol, h->cen, h->chl, h->adj_off, h->adj_face, h->adj_nb, h->lr,
                            h->geo, h->fcen, h->sgeo, h->sdx, h->fdx, h->d_cperm, h->d_fperm, h->bface};
      const size_t sizes[] = {N * 8, N * 8, N * 24, N * 8, (N + 1) * 4, M * 4, M * 4, F * 8,
                              F * 32, F * 24, h->sgeo ? M * 32 : 0, h->sdx ? M * 32 : 0, F * 64, N * 4, F * 4,
                              (size_t)h->NB * 4};
      for (int i = 0; i < 16; ++i) o[i] = ptrs[i] ? fnv(ptrs[i], sizes[i]) : 0;
      o[16] = (uint64_t)h->M;
      o[17] = (uint64_t)h->NB;
      o[18] = (uint64_t)(h->deg6 ? 1 : 0) | (uint64_t)(h->periodic ? 2 : 0);
      o[19] = h->periodic ? fnv(h->rcf, F * 4) : 0;
    }
    else if (n == "raw_level" || n == "tau") {
      if (n == "raw_level" && h->raw_lazy) materialise_raw(*h);
      std::vector<int8_t> v(h->N);
      CK(cudaMemcpy(v.data(), n == "tau" ? h->tau : h->raw, h->N, cudaMemcpyDeviceToHost));
      int32_t* o = static_cast<int32_t*>(out);
      // shards: OWNED entries into the global array (like get_state)
      for (int i = 0; i < h->N; ++i) {
        if (h->sharded() && i >= h->n_own) continue;
        o[h->sharded() ? h->shard_cells[h->cperm[i]] : h->cperm[i]] = v[i];
      }
    } else {
      require(false, "get_array: unknown array");
    }
  });
}

// Every captured graph (sweeps, plan, one-graph iteration) and the run_batch
// twin: dropped whenever a flag changes what a capture records, so the next
// call re-captures with the new settings on every path (iterate AND
// run_batch).
void drop_graphs(tafv_gpu& h) {
  for (auto& g : h.graphs) {
    cudaGraphExecDestroy(g.second.exec);
    for (auto e : g.second.evs) cudaEventDestroy(e);
  }
  h.graphs.clear();
  if (h.plan_graph) cudaGraphExecDestroy(h.plan_graph);
  h.plan_graph = nullptr;
  if (h.iter_graph) cudaGraphExecDestroy(h.iter_graph);
  h.iter_graph = nullptr;
}

int tafv_gpu_set_flag(tafv_gpu* h, const char* name, int64_t value) {
  return guard(h, [&] {
    const std::string n = name ? name : "";
    delete h->twin;  // rebuilt with the new settings by the next run_batch
    h->twin = nullptr;
    if (n == "grid_cap") {
      h->grid_cap = (int)std::max<int64_t>(1, std::min<int64_t>(value, h->nblk_last));
      drop_graphs(*h);
    } else if (n == "skip_top_lists") {
      h->skip_top_lists = value != 0;
      drop_graphs(*h);
    } else if (n == "sweep_marks") {
      h->sweep_marks = value != 0;
      drop_graphs(*h);
    } else if (n == "k1_tile") {
      h->k1_tile = (int)value;
      drop_graphs(*h);
    } else if (n == "k1_brick") {
      h->k1_brick = (int)value;
      if (value > 0) build_bricks(*h);
      drop_graphs(*h);
    } else if (n == "slot_n") {
      h->slot_n = value != 0;
      drop_graphs(*h);
    } else if (n == "slot_dx") {
      h->slot_dx = value != 0;
      drop_graphs(*h);
    } else if (n == "slot_geo") {
      h->slot_geo = value != 0;
      drop_graphs(*h);
    } else if (n == "alt_dir") {
      h->alt_dir = value != 0;
      drop_graphs(*h);
    } else if (n == "iwin_alias") {
      h->iwin_alias = value != 0;
      // no face is aliased any more: int_window holds every face's window
      // from here on (K2 accumulates all of them), so stale alias bytes
      // must not redirect the read-out -- but windows opened while aliased
      // hold no int_window yet: materialise them first
      if (!h->iwin_alias && h->ialias) {
        k_materialise_alias<<<h->grid_for((long long)h->F, 256), 256, 0, h->st>>>(h->iwin, h->isub, h->ialias,
                                                                                h->F, h->nv, (int)h->fs);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->st));
      }
      drop_graphs(*h);
    } else if (n == "dl_stream") {
      h->dl_stream = (int)value;
    } else if (n == "face_dx") {
      h->face_dx = value != 0;
      drop_graphs(*h);
    } else if (n == "batch_lanes") {
      h->batch_lanes = (int)value;
    } else if (n == "plan_graph") {
      h->plan_graph_on = value != 0;
    } else if (n == "use_graph") {
      h->use_graph = value != 0;
    } else if (n == "kernel_timing") {
      h->ktime = value != 0;
      for (int k = 0; k < tafv_gpu::kNumKinds; ++k) {
        h->kms[k] = 0.0;
        h->kcnt[k] = 0;
        h->kitems[k][0] = h->kitems[k][1] = h->kitems[k][2] = 0;
      }
      h->evkind.clear();
    }
    else require(false, "set_flag: unknown flag");
  });
}

int tafv_gpu_kernel_times(tafv_gpu* h, double* ms, int64_t* counts, int64_t* items) {
  if (!h) return TAFV_EINVAL;
  for (int k = 0; k < tafv_gpu::kNumKinds; ++k) {
    if (ms) ms[k] = h->kms[k];
    if (counts) counts[k] = h->kcnt[k];
    if (items)
      for (int j = 0; j < 3; ++j) items[3 * k + j] = h->kitems[k][j];
  }
  return TAFV_OK;
}

int tafv_gpu_mesh_info(tafv_gpu* h, int64_t* info4) {
  if (!h || !info4) return TAFV_EINVAL;
  info4[0] = h->N;
  info4[1] = h->F;
  info4[2] = h->M;
  info4[3] = h->nv;
  return TAFV_OK;
}

int tafv_gpu_stats(tafv_gpu* h, int64_t* launches, double* ms3) {
  if (!h) return TAFV_EINVAL;
  if (launches) *launches = h->launches;
  if (ms3)
    for (int i = 0; i < 3; ++i) ms3[i] = h->ms[i];
  return TAFV_OK;
}

}  // extern "C"
