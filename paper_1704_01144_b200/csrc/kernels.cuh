// sm_100a kernels of the LTS finite-volume hot path.
//
// One phase of the reference (corrector_phase / predictor_phase,
// proj/core/src/reference.cpp:41-70) runs as three kernels, the minimum the
// data dependencies allow (gradients need every neighbour's staged value,
// fluxes need both sides' limited gradients, residuals need every face flux):
//
//   K1 k_grad_limit   stage (committed / predicted / time-interpolated fringe,
//                     kernels.cpp:31-63) fused into Green-Gauss
//                     (kernels.cpp:65-89) + Barth-Jespersen (kernels.cpp:91-121).
//                     Staging is a pure function of (w, w_pred, tau, front,
//                     phase), so w_eval is never materialised: every consumer
//                     recomputes it bitwise-identically.
//   K2 k_face_flux    window reset (kernels.cpp:123-130) + reconstruction
//                     (kernels.cpp:132-159) + Rusanov (physics.hpp:42-47) +
//                     riemann_predict / riemann_correct (kernels.cpp:161-186);
//                     face states live in registers only.
//   K3 k_gather_update flux sum in the CSR slot order = ascending ORIGINAL
//                     face id (kernels.cpp:188-216) + extensive/intensive
//                     predict or correct (kernels.cpp:218-241). A gather, not
//                     a scatter: deterministic, no atomics.
//
// Plan kernels restate plan_iteration (reference.cpp:89-98): dt_max
// (kernels.cpp:247-254), min (kernels.cpp:260-264), ilogb classification
// (levels.cpp:18-25), Jacobi smoothing (levels.cpp:33-51), face cadence and
// fringe (levels.cpp:123-155), and a stable per-level compaction giving the
// prefix-union active sets of build_active_sets (reference.cpp:27-39).
//
// All item loops are grid-stride over an explicit list (or the identity when
// every item is active), so one launch shape serves any active-set size.
#pragma once

#include <cstdint>

#include "physics.cuh"

namespace tafv {

constexpr int kMaxLevels = 16;
constexpr int kMaxPeers = 4;  // level-sorted halo exchange lists (slab shards have <= 2 peers)

// ---- device views --------------------------------------------------------
struct MeshDev {
  int n_cells, n_faces;
  const double* __restrict__ vol;   // [N]
  const double* __restrict__ ivol;  // [N] 1.0 / vol (host IEEE division == device)
  const double* __restrict__ cen;   // [N][3]
  const double* __restrict__ chl;   // [N]
  const int* __restrict__ adj_off;  // [N+1]
  const int* __restrict__ adj_face; // [M] face id (~f when the cell is the face's right side)
  const int* __restrict__ adj_nb;   // [M] neighbour cell (-1 across transmissive faces)
  const int2* __restrict__ lr;      // [F] {left, resolved right (-1 transmissive)}
  const int* __restrict__ rcf;      // [F] face whose centroid the right side uses (periodic), or null
  const double4* __restrict__ geo;  // [F] {nx, ny, nz, area}
  const double* __restrict__ fcen;  // [F][3]
  // Hex fast path (DEG 6) per-slot geometry, contiguous per cell so K1's
  // geometry loads do not wait on the adjacency: {n.x, n.y, n.z, sign*area}
  // and the limiter's face-centroid offset fc - cc (same IEEE values the
  // kernel would compute: sign*area is exact, the subtraction is the same).
  const double4* __restrict__ sgeo;  // [N*6]
  const double4* __restrict__ sdx;   // [N*6] {dx, dy, dz, 0}: one 256-bit load per slot
  // [2F] or null: K2's reconstruction offsets per face, fc - c_left and
  // fc' - c_right (fc' = the partner's centroid across a periodic link), as
  // {dLx, dLy, dLz, 0}, {dRx, dRy, dRz, 0}: the same IEEE differences the
  // kernel would form, loaded by face index instead of gathered by cell.
  // TAFV_FDX_SPLIT: the left offsets of every face, then the right ones (a
  // warp's load covers 8 lines instead of 16), else interleaved per face.
  const double4* __restrict__ fdx;
};
#ifndef TAFV_FDX_SPLIT
#define TAFV_FDX_SPLIT 1
#endif
#if TAFV_FDX_SPLIT
#define TAFV_FDX_L(f, F) ((size_t)(f))
#define TAFV_FDX_R(f, F) ((size_t)(F) + (size_t)(f))
#else
#define TAFV_FDX_L(f, F) (2 * (size_t)(f))
#define TAFV_FDX_R(f, F) (2 * (size_t)(f) + 1)
#endif

struct StateDev {
  double* w;     // [N][NV] committed intensive
  double* W;     // [N][NV] committed extensive
  double* wp;    // [N][NV] predicted intensive (window end)
  double* grad;  // [N][NV][3] limited gradient (frozen for fringe cells)
  int8_t* tau;   // [N]
  int8_t* cad;   // [F]
  double* phi;   // [F][NV] phi_pred
  double* isub;  // [F][NV] int_substep
  double* iwin;  // [F][NV] int_window
  // [F] or null. Equal-level faces (both sides at the face's cadence, or a
  // boundary face) open a window at every one of their substeps, so their
  // int_window is always 0.0 + int_substep and no gather ever reads it (K3
  // reads int_window only on the coarser side of a fringe face). With
  // `ialias` set K2 skips those faces' window reset and accumulation and
  // records alias = 1; get_array("int_window") materialises isub + 0.0.
  uint8_t* ialias;
};

struct PlanDev {
  double dt_min;        // global stable step (or injected dt)
  int err;              // bit 0: |dtau| > 1 across a face; bit 1: injected tau out of range
  int nonfinite;        // divergence flag of the last trailing corrector
  long long cell_count[kMaxLevels];
  long long face_count[kMaxLevels];
  long long fringe_count[kMaxLevels];
  double totals[8];     // sum of W per component after the last iteration
  double bflux[8];      // boundary outflow per component over the last iteration (ledger)
  int ncell_prefix[kMaxLevels];  // |{c owned : tau_c <= l}|: K3 active cells of level l
  int nface_prefix[kMaxLevels];  // |{f touching owned : cadence_f <= l}|: K2 active faces
  // K1 active cells. Single domain: the K3 list. Shards: two lists, so the
  // cells that read no halo row run while the halo exchange is in flight:
  int nk1_prefix[kMaxLevels];    // |{c owned, no halo neighbour : tau_c <= l}| ("deep")
  int nkb_prefix[kMaxLevels];    // |{c owned with a halo neighbour, or ring 1 : tau_c <= l}| ("border")
  long long k1_count[kMaxLevels];    // per-level counts of the deep K1 list
  long long kb_count[kMaxLevels];    // per-level counts of the border K1 list
  long long gcell_count[kMaxLevels]; // owned counts summed over ranks (records, theta)
  int nfi_prefix[kMaxLevels];        // shards: |{interior f : cadence_f <= l}| (K2 before the halo join)
  int nfb_prefix[kMaxLevels];        // shards: |{border f touching owned : cadence_f <= l}|
  long long fi_count[kMaxLevels];
  long long fb_count[kMaxLevels];
  int sweep_changed[kMaxLevels];     // single-domain plan: Jacobi sweep i changed a level
  // shards: the exchange lists of every peer sorted by level; prefix counts
  // |{listed cells : tau <= l}| = the rows a phase at level l updates
  int xs_prefix[kMaxPeers][kMaxLevels];
  int xr_prefix[kMaxPeers][kMaxLevels];
  long long xs_count[kMaxPeers][kMaxLevels];
  long long xr_count[kMaxPeers][kMaxLevels];
};

// ---- staging: pure function of the committed/predicted state ---------------
// Reproduces w_eval of stage_committed / stage_predicted / stage_interpolated
// (kernels.cpp:31-63): at `front`, a cell whose window boundary lies on the
// front (offset 0) stages w (predictor) or w_pred (corrector); a fringe cell
// straddling the front stages w + theta_f (w_pred - w), theta_f = offset/2^tau.
// The row an offset-0 cell stages (w in a predictor, w_pred in a corrector)
// is loaded together with tau, so the common case costs one dependent load,
// not two; a cell straddling the front then loads its other row and
// interpolates. Returns tau.
// A cell's state row (NV doubles at arr + x NV). With an odd NV >= 3 (Euler:
// 40-byte rows) the row starts on a 16-byte boundary for even x and 8 bytes
// past one for odd x: WIDE loads the (NV + 1) / 2 aligned 16-byte pairs that
// cover it (one double before the row for odd x, one past it for even x; the
// state arrays are allocated with that slack) and selects, so a warp's row
// load is 3 instructions of 3 L1 wavefronts per line touched instead of 5
// (K2 runs at ~80 % of the L1 data pipe; profiles/r2_k2_l1.md).
#ifndef TAFV_ROW128
#define TAFV_ROW128 1  // 0 off, 1 K2, 2 K2 and K1
#endif
template <int NV, bool WIDE>
__device__ __forceinline__ void load_row(const double* __restrict__ arr, int x, double* out) {
  if constexpr (WIDE && NV >= 3 && (NV & 1)) {
    const size_t e0 = (size_t)x * NV;
    const bool odd = e0 & 1;
    const double2* p = reinterpret_cast<const double2*>(arr + (e0 & ~(size_t)1));
    double v[NV + 1];
#pragma unroll
    for (int q = 0; q < (NV + 1) / 2; ++q) {
      const double2 t = __ldg(p + q);
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = odd ? v[k + 1] : v[k];
  } else {
    const double* base = arr + (size_t)x * NV;
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = __ldg(base + k);
  }
}

template <int NV, bool WIDE = false>
__device__ __forceinline__ int stage_spec(const StateDev& s, int x, int front, bool pred, double* out) {
  load_row<NV, WIDE>(pred ? s.w : s.wp, x, out);
  const int tx = __ldg(s.tau + x);
  const int win = 1 << tx;
  const int off = front & (win - 1);
  if (off != 0) {
    const double th = (double)off / (double)win;
    if constexpr (WIDE && NV >= 3 && (NV & 1)) {
      double o[NV];
      load_row<NV, true>(pred ? s.wp : s.w, x, o);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const double a = pred ? out[k] : o[k];   // w
        const double b = pred ? o[k] : out[k];   // w_pred
        out[k] = a + th * (b - a);
      }
    } else {
      const double* other = (pred ? s.wp : s.w) + (size_t)x * NV;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const double o = __ldg(other + k);
        const double a = pred ? out[k] : o;   // w
        const double b = pred ? o : out[k];   // w_pred
        out[k] = a + th * (b - a);
      }
    }
  }
  return tx;
}

// One 256-bit load of a 32-byte aligned double4 (sm_100), read-only path.
#ifndef TAFV_V4
#define TAFV_V4 2
#endif
__device__ __forceinline__ double4 ld4(const double4* p) {
  double4 r;
#if TAFV_V4 == 2
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
#elif TAFV_V4 == 1
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
#else
  r = *p;
#endif
  return r;
}

// 256-bit load through L1 (rows reused by neighbouring items) and store.
__device__ __forceinline__ double4 ld4a(const double* p) {
  double4 r;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// Gradient rows are padded to a multiple of 4 doubles (Euler: 15 -> 16) so
// K1 writes and K2 reads them with 256-bit accesses.
template <int NV>
struct GradRow {
  static constexpr int S = (NV * 3 + 3) / 4 * 4;
};
// Face integral rows (phi_pred, int_substep, int_window) padded to an even
// number of doubles (Euler: 5 -> 6, 48 B) for 128-bit stores / loads.
template <int NV>
struct FaceRow {
  static constexpr int S = (NV + 1) / 2 * 2;
};
__device__ __forceinline__ void st2(double* p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(a), "d"(b) : "memory");
}

__device__ __forceinline__ int slot_face(int e) { return e >= 0 ? e : ~e; }
__device__ __forceinline__ double slot_sign(int e) { return e >= 0 ? 1.0 : -1.0; }

#ifndef TAFV_BJ2
#define TAFV_BJ2 1
#endif
#ifndef TAFV_BJZ
#define TAFV_BJZ 1
#endif
// Barth-Jespersen update alpha = min(alpha, minmod(delta, head) / delta)
// (kernels.cpp:111-117) with the division evaluated only where its value can
// matter. Exactly equivalent, including signed zeros and NaN:
//   same-sign, |head| >= |delta|  -> delta/delta = 1 (or NaN for inf/inf):
//                                    smin(alpha <= 1, .) leaves alpha unchanged;
//   opposite sign / zero / NaN head -> 0.0/delta = +-0 by the sign of delta;
//   delta NaN                      -> NaN ratio: smin leaves alpha unchanged;
//   delta == 0                     -> skipped by the reference.
__device__ __forceinline__ double bj_update(double alpha, double delta, double hp, double hn) {
#if TAFV_BJ2
  // In magnitudes: A = the headroom on delta's side, sign-normalised (hp =
  // w_max - w_c for delta > 0, hn = -(w_min - w_c) for delta < 0, exact).
  //   A > 0, |delta| > A      -> head / delta = A / |delta| (IEEE division is
  //                              sign-symmetric: the same quotient)
  //   A > 0, |delta| <= A     -> 1 (or NaN for inf/inf): no-op
  //   A <= 0 or NaN           -> +-0 by the sign of delta
  //   delta == 0 or NaN       -> skipped / no-op
  const bool pos = delta > 0.0, neg = delta < 0.0;
  const double A = pos ? hp : hn;
  const bool aok = A > 0.0;
  const double ad = fabs(delta);
#if TAFV_BJZ
  // the zero outcome as word selects: smin(alpha, +-0) is +-0 exactly when
  // alpha > 0 (alpha is never negative), and +-0 has a zero low word
  const bool upd = (pos || neg) && !aok && alpha > 0.0;
  const int hi = upd ? (neg ? (int)0x80000000 : 0) : __double2hiint(alpha);
  const int lo = upd ? 0 : __double2loint(alpha);
  alpha = __hiloint2double(hi, lo);
#else
  if ((pos || neg) && !aok) alpha = smin(alpha, pos ? 0.0 : -0.0);
#endif
  if (aok && ad > A) alpha = smin(alpha, A / ad);
  return alpha;
#else
  const double head = delta > 0.0 ? hp : -hn;
  // zero outcome (opposite signs, head == 0 or NaN): +0 for delta > 0, -0 for
  // delta < 0 -- predicated; the quotient only where |head| < |delta|.
  const bool pos = delta > 0.0, neg = delta < 0.0;
  const bool same = pos ? head > 0.0 : head < 0.0;
  const bool lim = same && (pos ? head < delta : delta < head);
  if ((pos || neg) && !same) alpha = smin(alpha, pos ? 0.0 : -0.0);
  if (lim) alpha = smin(alpha, head / delta);
  return alpha;
#endif
}

// ---- bulk copies into shared memory (TMA engine, mbarrier completion) ------
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// One elected thread: expect `bytes` on the barrier and start the copy.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst before the async write
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// ---- K1: stage + Green-Gauss + Barth-Jespersen ----------------------------
// Thread per cell, all NV components in registers (measured faster than a
// component-parallel layout, which multiplies the shared index/geometry
// instructions by NV). Per component the arithmetic is the reference's, slot
// by slot in CSR order. DEG = 6 is the hex fast path (implicit offsets, fully
// unrolled slot loop); DEG = 0 reads the CSR offsets. The active count comes
// from device memory so the launch is graph-capturable.
#ifndef TAFV_K1_TILE
#define TAFV_K1_TILE 1  // identity phases: Morton-brick staging in shared memory
#endif
#ifndef TAFV_K1_TILE_SDX
#define TAFV_K1_TILE_SDX 0  // with TILE: the brick's limiter offsets by one bulk copy (A/B)
#endif
#ifndef TAFV_K1_MINB
#define TAFV_K1_MINB 5  // min resident 128-thread blocks/SM for K1 (register cap 102; measured best)
#endif
// TILE: the identity-phase instance (list == nullptr, Morton-brick staging);
// a separate instantiation so each path is register-allocated on its own.
template <class P, int DEG, bool TILE>
__global__ void __launch_bounds__(128, TAFV_K1_MINB) k_grad_limit(MeshDev m, StateDev s,
                                                    const int* __restrict__ list,
                                                    const int* __restrict__ n_dev, int base, int front,
                                                    int pred, int rev) {
  constexpr int NV = P::NV, D = P::DIM;
  const int n = *n_dev;
  const int stride = gridDim.x * blockDim.x;
  // One active cell c with its staged row we: Green-Gauss + Barth-Jespersen.
  // Neighbours in [lo, hi) were staged into srow by their own threads.
  // sdx_tile (tile path): the brick's limiter offsets, bulk-copied into
  // shared memory at the brick's start (complete when `bar` flips `parity`)
  auto cell = [&](int c, const double* we, int lo, int hi, const double* srow, const double4* sdx_tile,
                  uint64_t* bar, unsigned parity) {
    double g[NV][D];
    double wmin[NV], wmax[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
      for (int d = 0; d < D; ++d) g[k][d] = 0.0;
      wmin[k] = __longlong_as_double(0x7ff0000000000000ll);
      wmax[k] = __longlong_as_double((long long)0xfff0000000000000ull);
    }
    bool any = false;
    const int s0 = DEG ? DEG * c : m.adj_off[c];
    const int s1 = DEG ? s0 + DEG : m.adj_off[c + 1];
#pragma unroll
    for (int t = s0; t < s1; ++t) {
      const int nb = m.adj_nb[t];
      double4 gm;
      double scale;
      if (DEG == 6 && m.sgeo) {
#ifdef TAFV_EXP_NO_SGEO
        gm = make_double4(0.5 + 1e-3 * t, 0.25, 0.125, 1e-4 * (t & 7));  // timing experiment only
#else
        gm = ld4(m.sgeo + t);
#endif
        scale = gm.w;
      } else {
        const int ef = m.adj_face[t];
        gm = ld4(m.geo + slot_face(ef));
        scale = slot_sign(ef) * gm.w;
      }
      double wf[NV];
      if (nb >= 0) {
        double wn[NV];
#ifdef TAFV_EXP_NO_GATHER
        for (int k = 0; k < NV; ++k) wn[k] = we[k] * (1.0 + 1e-3 * t);  // timing experiment only
#else
        if (nb >= lo && nb < hi) {  // staged by its own thread in this tile
#pragma unroll
          for (int k = 0; k < NV; ++k) wn[k] = srow[(nb - lo) * NV + k];
        } else {
          stage_spec<NV, (TAFV_ROW128 >= 2)>(s, nb, front, pred, wn);
        }
#endif
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          wf[k] = 0.5 * (we[k] + wn[k]);
          wmin[k] = smin(wmin[k], wn[k]);
          wmax[k] = smax(wmax[k], wn[k]);
        }
        any = true;
      } else {
#pragma unroll
        for (int k = 0; k < NV; ++k) wf[k] = we[k];
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        g[k][0] += wf[k] * gm.x * scale;
        g[k][1] += wf[k] * gm.y * scale;
        if (D == 3) g[k][D - 1] += wf[k] * gm.z * scale;
      }
    }
    const double inv_v = m.ivol[c];
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int d = 0; d < D; ++d) g[k][d] = g[k][d] * inv_v;
#ifdef TAFV_EXP_NO_LIMIT
    any = false;  // timing experiment only
#endif
    if (any) {
      const double* cp = m.cen + 3 * (size_t)c;
      const double cc0 = cp[0], cc1 = cp[1], cc2 = cp[2];
      double alpha[NV];
      // headroom operands are the same for every slot (kernels.cpp:115-116)
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        alpha[k] = 1.0;
        wmax[k] = wmax[k] - we[k];     // hp: headroom above
        wmin[k] = -(wmin[k] - we[k]);  // hn: headroom below, negated (exact)
      }
      if (DEG == 6 && sdx_tile) mbar_wait(bar, parity);
#pragma unroll
      for (int t = s0; t < s1; ++t) {
        double dx0, dx1, dx2;
        if (DEG == 6 && m.sdx) {
#ifdef TAFV_EXP_NO_SDX
          const double4 d = make_double4(1e-3 * (t & 15), 1e-3, -1e-3, 0.0);  // timing experiment only
#else
          const double4 d = sdx_tile ? sdx_tile[(size_t)DEG * (c - lo) + (t - s0)] : ld4(m.sdx + t);
#endif
          dx0 = d.x;
          dx1 = d.y;
          dx2 = d.z;
        } else {
          const int f = slot_face(m.adj_face[t]);
          const double* fc = m.fcen + 3 * (size_t)f;
          dx0 = fc[0] - cc0;
          dx1 = fc[1] - cc1;
          dx2 = fc[2] - cc2;
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          double delta = g[k][0] * dx0 + g[k][1] * dx1;
          if (D == 3) delta = delta + g[k][D - 1] * dx2;
          alpha[k] = bj_update(alpha[k], delta, wmax[k], wmin[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int d = 0; d < D; ++d) g[k][d] *= alpha[k];
    }
    constexpr int GS = GradRow<NV>::S;
    double row[GS];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      row[3 * k] = g[k][0];
      row[3 * k + 1] = g[k][1];
      row[3 * k + 2] = D == 3 ? g[k][D - 1] : 0.0;
    }
#pragma unroll
    for (int q = 3 * NV; q < GS; ++q) row[q] = 0.0;
    double* go = s.grad + (size_t)c * GS;
#pragma unroll
    for (int q = 0; q < GS; q += 4) st4(go + q, row[q], row[q + 1], row[q + 2], row[q + 3]);
  };
#if TAFV_K1_TILE
  if constexpr (TILE && DEG == 6) {
    // Identity phase (every cell of [base, base + n) active): a block takes
    // 128 consecutive cells (a Morton brick), each thread stages its own cell
    // into shared memory once, and the neighbours inside the brick (~80 % of
    // the slots) read it there instead of re-staging it from global memory.
    __shared__ double srow[128 * NV];
#if TAFV_K1_TILE_SDX
    // and the brick's limiter offsets arrive by one bulk copy per brick
    // (cp.async.bulk, TMA engine) while the gradient loop runs
    __shared__ __align__(128) double4 sdx_tile[128 * 6];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0 && m.sdx) mbar_init(&bar, 1);
    __syncthreads();
    unsigned parity = 0;
#endif
    for (int t0 = blockIdx.x * blockDim.x; t0 < n; t0 += stride) {
      const int cnt = min((int)blockDim.x, n - t0);
      // rev: walk the items backwards (see below); the tile is contiguous either way
      const int lo = base + (rev ? n - t0 - cnt : t0), hi = lo + cnt;
#if TAFV_K1_TILE_SDX
      if (threadIdx.x == 0 && m.sdx)
        bulk_g2s(sdx_tile, m.sdx + (size_t)DEG * lo, (unsigned)(cnt * DEG * sizeof(double4)), &bar);
#endif
      const int ii = t0 + threadIdx.x;
      int c = -1;
      double we[NV];
      if (ii < n) {
        c = base + (rev ? n - 1 - ii : ii);
        stage_spec<NV, (TAFV_ROW128 >= 2)>(s, c, front, pred, we);
#pragma unroll
        for (int k = 0; k < NV; ++k) srow[(c - lo) * NV + k] = we[k];
      }
      __syncthreads();
#if TAFV_K1_TILE_SDX
      if (c >= 0) cell(c, we, lo, hi, srow, m.sdx ? sdx_tile : nullptr, &bar, parity);
      parity ^= 1u;
#else
      if (c >= 0) cell(c, we, lo, hi, srow, nullptr, nullptr, 0);
#endif
      // the next brick overwrites srow (a second buffer without this barrier
      // measured slower: the barrier keeps the block's warps on one brick)
      __syncthreads();
    }
  } else
#endif
  {
    for (int ii = blockIdx.x * blockDim.x + threadIdx.x; ii < n; ii += stride) {
      // rev: walk the items backwards, so this kernel starts on the rows its
      // predecessor wrote last (still in L2); consecutive kernels alternate.
      const int i = rev ? n - 1 - ii : ii;
      const int c = list ? list[i] : base + i;
      double we[NV];
      stage_spec<NV, (TAFV_ROW128 >= 2)>(s, c, front, pred, we);
      cell(c, we, 0, 0, nullptr, nullptr, nullptr, 0);
    }
  }
}

// ---- K1 for identity phases of hex meshes: precomputed bricks ---------------
// A block takes a Morton brick of 128 consecutive cells whose every operand
// arrives in shared memory without a dependent global load:
//  * built once per mesh (k_brick_build): per slot a 16-bit row index into the
//    brick's stage (own rows 0..127, halo rows 128.., 0xffff = no neighbour) and
//    a 16-bit face entry (bit 15 = the slot sees the face from its right side),
//    the brick's halo cell list, and the brick's faces {n, area}, centroid
//    PACKED per brick (a face shared by two bricks is stored in both: ~3.6
//    entries of 56 B per cell instead of the 6 x 64 B per-slot streams);
//  * per brick, ONE elected thread starts bulk copies (cp.async.bulk, the TMA
//    engine, one mbarrier) of the contiguous streams -- the cells' staged rows
//    (in an identity phase the staged row IS w in a predictor / w_pred in a
//    corrector, kernels.cpp:31-44), centroids, 1/V, the index table, the
//    packed faces -- and prefetches the next brick's into L2; every thread
//    gathers its share of the halo rows with cp.async (the halo list of brick
//    b was fetched while brick b - 1 was computed);
//  * then k_grad_limit's per-cell arithmetic (per-face geometry: scale =
//    sign * area, offset = face centroid - cell centroid, the values the
//    per-slot streams store) from shared memory only.
// Bricks whose halo or faces exceed the stage (ragged Morton bricks) are left
// to k_grad_limit over a list of their cells. Other resident blocks compute
// while a block waits for its copies (one stage per block).
#ifndef TAFV_K1B_MINB
#define TAFV_K1B_MINB 4
#endif
// Stage capacity: 128-cell runs of the Morton order are ragged (config 4:
// 500 +- 20 face entries, 235 +- 40 halo rows per brick against 464 / 160 for
// an 8x4x4 box; tools/brick_probe.py), so the halo rows and the packed faces
// share ONE pool of the stage -- a brick fits when 40 B per halo row + 56 B
// per face entry fit the pool (and the halo list its buffer) -- sized for 4
// blocks per SM; larger stages (3 blocks per SM) measured slower.
#ifndef TAFV_K1B_HALO
#define TAFV_K1B_HALO 320  // halo rows per brick at most (list buffers)
#endif
#ifndef TAFV_K1B_POOL
#define TAFV_K1B_POOL 41856  // bytes of halo rows + face entries per brick
#endif
constexpr int kBrick = 128;  // cells per brick = threads per block
constexpr int kBrickHalo = TAFV_K1B_HALO;
constexpr int kBrickPool = TAFV_K1B_POOL;
// pool bytes of a brick with e face entries (padded to even) and h halo rows of nv doubles
__host__ __device__ constexpr int brick_pool_bytes(int e, int h, int nv) {
  return ((h * nv * 8 + 31) & ~31) + ((e + 1) & ~1) * 56;
}
struct BrickDev {
  const unsigned short* idx;  // [nbricks][2][768]: row indices, then face entries
  const int4* info;           // [nbricks] {face entries (< 0: ragged, not staged), halo rows, entry offset, halo offset}
  const int* halo;            // halo cell ids, brick after brick (each padded to 4)
  const double* geo;          // [entries][4] {n, area}, brick after brick (each padded to even)
  const double* fcen;         // [entries][3]
};
template <int NV>
struct BrickSmem {  // byte offsets into the dynamic shared memory (16-byte aligned parts)
  static constexpr int row = 0;  // [128][NV] own rows, then the pool: halo rows, {n, area}, centroids
  static constexpr int pool = row + kBrick * NV * 8;
  static constexpr int cen = pool + kBrickPool;
  static constexpr int ivol = cen + kBrick * 24;
  static constexpr int idx = ivol + kBrick * 8;  // [2][768] u16
  static constexpr int hl = idx + 2 * 768 * 2;   // [2][halo] halo lists (this brick's, the next one's)
  static constexpr int bytes = hl + 2 * kBrickHalo * 4;
  static_assert(pool % 32 == 0 && kBrickPool % 32 == 0, "the pool holds 32-byte aligned face rows");
};
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic accesses of the stage before the async writes
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
}
// cells [0, *n_dev) active (an identity phase: n = every owned cell), all with 6 slots.
template <class P>
__global__ void __launch_bounds__(kBrick, TAFV_K1B_MINB) k_grad_limit_brick(MeshDev m, StateDev s, BrickDev bk,
                                                                           const int* __restrict__ n_dev,
                                                                           int pred, int rev) {
  constexpr int NV = P::NV, D = P::DIM, B = kBrick;
  using L = BrickSmem<NV>;
  extern __shared__ __align__(128) unsigned char brick_smem[];
  double* s_row = reinterpret_cast<double*>(brick_smem + L::row);
  double* s_cen = reinterpret_cast<double*>(brick_smem + L::cen);
  double* s_ivol = reinterpret_cast<double*>(brick_smem + L::ivol);
  unsigned short* s_ri = reinterpret_cast<unsigned short*>(brick_smem + L::idx);
  unsigned short* s_fi = s_ri + 768;
  int* s_hl = reinterpret_cast<int*>(brick_smem + L::hl);
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  unsigned parity = 0;
  const int n = *n_dev;
  const int nbricks = n / B;  // whole bricks only; the tail cells go with the ragged bricks' list
  const double* __restrict__ src = pred ? s.w : s.wp;
  auto brick_of = [&](int b) { return rev ? nbricks - 1 - b : b; };
  // the first brick's halo list (later ones arrive one brick ahead)
  int buf = 0;
  if ((int)blockIdx.x < nbricks) {
    const int4 c0 = bk.info[brick_of(blockIdx.x)];
    if (c0.x >= 0)
      for (int i = tid; i < c0.y; i += B) s_hl[i] = bk.halo[(size_t)c0.w + i];
  }
  __syncthreads();
  for (int b = blockIdx.x; b < nbricks; b += gridDim.x) {
    const int bb = brick_of(b);
    const int lo = bb * B;
    const int4 cnt = bk.info[bb];
    const int bn = b + (int)gridDim.x;
    const int nbb = bn < nbricks ? brick_of(bn) : -1;
    const int ne = (cnt.x + 1) & ~1;  // an even number of entries: 16-byte multiples of the 24-byte centroids
    // the pool of this brick: halo rows, then {n, area}, then centroids
    double* s_geo = reinterpret_cast<double*>(brick_smem + L::pool + ((cnt.y * NV * 8 + 31) & ~31));
    double* s_fcen = s_geo + 4 * ne;
    if (cnt.x >= 0) {
      if (tid == 0) {
        mbar_expect(&bar, (unsigned)(B * NV * 8 + B * 24 + B * 8 + 3072 + ne * 56));
        bulk_copy(s_ri, bk.idx + (size_t)bb * 1536, 3072, &bar);
        bulk_copy(s_row, src + (size_t)lo * NV, B * NV * 8, &bar);
        if (ne) {
          bulk_copy(s_geo, bk.geo + (size_t)cnt.z * 4, (unsigned)ne * 32, &bar);
          bulk_copy(s_fcen, bk.fcen + (size_t)cnt.z * 3, (unsigned)ne * 24, &bar);
        }
        bulk_copy(s_cen, m.cen + 3 * (size_t)lo, B * 24, &bar);
        bulk_copy(s_ivol, m.ivol + lo, B * 8, &bar);
      }
      // halo rows: 8-byte asynchronous copies, every thread its share
      const int* hl = s_hl + buf * kBrickHalo;
      for (int i = tid; i < cnt.y * NV; i += B) {
        const int h = i / NV, k = i - h * NV;
        cp_async8(s_row + (B + h) * NV + k, src + (size_t)hl[h] * NV + k);
      }
    }
    if (nbb >= 0) {  // the next brick: its halo list into the other buffer, its streams towards L2
      const int4 c2 = bk.info[nbb];
      if (c2.x >= 0) {
        int* hn = s_hl + (buf ^ 1) * kBrickHalo;
        for (int i = tid; i < c2.y; i += B) hn[i] = bk.halo[(size_t)c2.w + i];
        if (tid == 32) {
          const int n2 = (c2.x + 1) & ~1;
          bulk_prefetch_l2(bk.idx + (size_t)nbb * 1536, 3072);
          bulk_prefetch_l2(src + (size_t)nbb * B * NV, B * NV * 8);
          if (n2) {
            bulk_prefetch_l2(bk.geo + (size_t)c2.z * 4, (unsigned)n2 * 32);
            bulk_prefetch_l2(bk.fcen + (size_t)c2.z * 3, (unsigned)n2 * 24);
          }
          bulk_prefetch_l2(m.cen + 3 * (size_t)nbb * B, B * 24);
        }
      }
    }
    if (cnt.x >= 0) {
      cp_async_wait_all();
      mbar_wait(&bar, parity);
      parity ^= 1u;
    }
    __syncthreads();  // halo rows of every thread, the next halo list
    if (cnt.x >= 0) {
      const int c = lo + tid;
      double we[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) we[k] = s_row[tid * NV + k];
      double g[NV][D];
      double wmin[NV], wmax[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int d = 0; d < D; ++d) g[k][d] = 0.0;
        wmin[k] = __longlong_as_double(0x7ff0000000000000ll);
        wmax[k] = __longlong_as_double((long long)0xfff0000000000000ull);
      }
      bool any = false;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const unsigned li = s_ri[tid * 6 + t];
        const unsigned fe = s_fi[tid * 6 + t];
        const unsigned le = fe & 0x7fffu;
        const double2 g01 = *reinterpret_cast<const double2*>(s_geo + 4 * le);
        const double2 g23 = *reinterpret_cast<const double2*>(s_geo + 4 * le + 2);
        const double scale = (fe & 0x8000u) ? -g23.y : g23.y;  // sign * area, exact
        double wf[NV];
        if (li != 0xffffu) {
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            const double wn = s_row[li * NV + k];
            wf[k] = 0.5 * (we[k] + wn);
            wmin[k] = smin(wmin[k], wn);
            wmax[k] = smax(wmax[k], wn);
          }
          any = true;
        } else {
#pragma unroll
          for (int k = 0; k < NV; ++k) wf[k] = we[k];
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          g[k][0] += wf[k] * g01.x * scale;
          g[k][1] += wf[k] * g01.y * scale;
          if (D == 3) g[k][D - 1] += wf[k] * g23.x * scale;
        }
      }
      const double inv_v = s_ivol[tid];
#pragma unroll
      for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int d = 0; d < D; ++d) g[k][d] = g[k][d] * inv_v;
      if (any) {
        const double cc0 = s_cen[3 * tid], cc1 = s_cen[3 * tid + 1], cc2 = s_cen[3 * tid + 2];
        double alpha[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          alpha[k] = 1.0;
          wmax[k] = wmax[k] - we[k];     // hp: headroom above
          wmin[k] = -(wmin[k] - we[k]);  // hn: headroom below, negated (exact)
        }
#pragma unroll
        for (int t = 0; t < 6; ++t) {
          const unsigned le = s_fi[tid * 6 + t] & 0x7fffu;
          const double dx0 = s_fcen[3 * le] - cc0, dx1 = s_fcen[3 * le + 1] - cc1, dx2 = s_fcen[3 * le + 2] - cc2;
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            double delta = g[k][0] * dx0 + g[k][1] * dx1;
            if (D == 3) delta = delta + g[k][D - 1] * dx2;
            alpha[k] = bj_update(alpha[k], delta, wmax[k], wmin[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < NV; ++k)
#pragma unroll
          for (int d = 0; d < D; ++d) g[k][d] *= alpha[k];
      }
      constexpr int GS = GradRow<NV>::S;
      double row[GS];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        row[3 * k] = g[k][0];
        row[3 * k + 1] = g[k][1];
        row[3 * k + 2] = D == 3 ? g[k][D - 1] : 0.0;
      }
#pragma unroll
      for (int q = 3 * NV; q < GS; ++q) row[q] = 0.0;
      double* go = s.grad + (size_t)c * GS;
#pragma unroll
      for (int q = 0; q < GS; q += 4) st4(go + q, row[q], row[q + 1], row[q + 2], row[q + 3]);
    }
    buf ^= 1;
    __syncthreads();  // every read of the stage before the next brick's copies
  }
}

// The static brick structures (BrickDev) of cells [0, 128 nbricks), one block
// per brick, in two passes around an exclusive scan of the bricks' sizes: a
// slot whose face this cell owns as the left side (or whose left cell lies
// outside the brick) takes a packed face entry, the other side of a face
// inside the brick shares its left cell's entry; every out-of-brick neighbour
// takes a halo row. FILL = false: sizes only (info.x < 0: the brick does not
// fit the stage; esize / hsize = its padded sizes, 0 when ragged); FILL = true:
// info.z / .w hold the offsets and the tables are written.
template <bool FILL>
__global__ void __launch_bounds__(kBrick) k_brick_build(const int* __restrict__ adj_nb,
                                                        const int* __restrict__ adj_face,
                                                        const double4* __restrict__ geo,
                                                        const double* __restrict__ fcen, int nbricks, int nv,
                                                        int4* info, int* esize, int* hsize, unsigned short* idx,
                                                        int* halo, double* bgeo, double* bfcen,
                                                        int* ragged_count) {
  __shared__ int s_nb[768], s_af[768], s_ent[768];
  __shared__ int s_e[kBrick + 1], s_h[kBrick + 1];
  const int b = blockIdx.x, tid = threadIdx.x, lo = b * kBrick;
  if (b >= nbricks) return;
  if (FILL && info[b].x < 0) return;
  for (int i = tid; i < 768; i += kBrick) {
    s_nb[i] = adj_nb[6 * (size_t)lo + i];
    s_af[i] = adj_face[6 * (size_t)lo + i];
  }
  __syncthreads();
  int ne = 0, nh = 0;
  for (int t = 0; t < 6; ++t) {
    const int nb = s_nb[tid * 6 + t], ef = s_af[tid * 6 + t];
    const bool inside = nb >= lo && nb < lo + kBrick;
    if (nb >= 0 && !inside) ++nh;
    if (ef >= 0 || !inside) ++ne;
  }
  s_e[tid + 1] = ne;
  s_h[tid + 1] = nh;
  __syncthreads();
  if (tid == 0) {
    s_e[0] = s_h[0] = 0;
    for (int i = 1; i <= kBrick; ++i) {
      s_e[i] += s_e[i - 1];
      s_h[i] += s_h[i - 1];
    }
  }
  __syncthreads();
  const int etot = s_e[kBrick], htot = s_h[kBrick];
  if (!FILL) {
    if (tid == 0) {
      const bool fits = htot <= kBrickHalo && brick_pool_bytes(etot, htot, nv) <= kBrickPool;
      info[b] = make_int4(fits ? etot : -etot - 1, htot, 0, 0);  // ragged sizes kept for tuning
      esize[b] = fits ? (etot + 1) & ~1 : 0;
      hsize[b] = fits ? (htot + 3) & ~3 : 0;
      if (!fits) atomicAdd(ragged_count, 1);
    }
    return;
  }
  const size_t eoff = (size_t)info[b].z, hoff = (size_t)info[b].w;
  int e = s_e[tid], h = s_h[tid];
  unsigned short* ri = idx + (size_t)b * 1536;
  unsigned short* fi = ri + 768;
  for (int t = 0; t < 6; ++t) {
    const int nb = s_nb[tid * 6 + t], ef = s_af[tid * 6 + t];
    const bool inside = nb >= lo && nb < lo + kBrick;
    unsigned short r = 0xffffu;
    if (nb >= 0) {
      if (inside) {
        r = (unsigned short)(nb - lo);
      } else {
        halo[hoff + h] = nb;
        r = (unsigned short)(kBrick + h);
        ++h;
      }
    }
    ri[tid * 6 + t] = r;
    int ent = -1;
    if (ef >= 0 || !inside) {
      const int f = ef >= 0 ? ef : ~ef;
      const double4 gq = geo[f];
      double* go = bgeo + (eoff + e) * 4;
      go[0] = gq.x;
      go[1] = gq.y;
      go[2] = gq.z;
      go[3] = gq.w;
      double* fo = bfcen + (eoff + e) * 3;
      fo[0] = fcen[3 * (size_t)f];
      fo[1] = fcen[3 * (size_t)f + 1];
      fo[2] = fcen[3 * (size_t)f + 2];
      ent = e++;
    }
    s_ent[tid * 6 + t] = ent;
  }
  __syncthreads();
  for (int t = 0; t < 6; ++t) {
    const int nb = s_nb[tid * 6 + t], ef = s_af[tid * 6 + t];
    int ent = s_ent[tid * 6 + t];
    if (ent < 0) {  // the right side of a face whose left cell is in the brick: that cell's entry
      const int f = ~ef, l = nb - lo;
      for (int q = 0; q < 6; ++q)
        if (s_af[l * 6 + q] == f) ent = s_ent[l * 6 + q];
    }
    fi[tid * 6 + t] = (unsigned short)(ent | (ef < 0 ? 0x8000 : 0));
  }
}
// Offsets (exclusive scans of the padded sizes) into info.z / .w.
__global__ void k_brick_offsets(int4* info, const int* eoff, const int* hoff, int nbricks) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nbricks; b += gridDim.x * blockDim.x) {
    info[b].z = eoff[b];
    info[b].w = hoff[b];
  }
}
// The cells the brick kernel leaves to k_grad_limit: ragged bricks and the tail.
__global__ void k_brick_ragged_cells(const int4* __restrict__ info, int nbricks, int n, int* list, int* n_out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const int b = c / kBrick;
    if (b >= nbricks || info[b].x < 0) list[atomicAdd(n_out, 1)] = c;
  }
}

// kernels.cpp:25-27 with the z term appended left to right; d = to - from.
template <int D>
__device__ __forceinline__ double extrapolate_d(double w, const double* g, const double* d) {
  double v = (w + g[0] * d[0]) + g[1] * d[1];
  if (D == 3) v = v + g[D - 1] * d[D - 1];
  return v;
}
template <int D>
__device__ __forceinline__ double extrapolate(double w, const double* g, const double* from,
                                              const double* to) {
  double v = (w + g[0] * (to[0] - from[0])) + g[1] * (to[1] - from[1]);
  if (D == 3) v = v + g[D - 1] * (to[D - 1] - from[D - 1]);
  return v;
}

// A cell's gradient row into registers (read-only in K2: only K1 writes it).
template <int NV>
__device__ __forceinline__ void load_grad(const StateDev& s, int x, double* g) {
  constexpr int GS = GradRow<NV>::S;
  const double* src = s.grad + (size_t)x * GS;
#pragma unroll
  for (int q = 0; q < GS; q += 4) {
    const double4 v = ld4a(src + q);
    g[q] = v.x;
    g[q + 1] = v.y;
    g[q + 2] = v.z;
    g[q + 3] = v.w;
  }
}

// ---- K2: window reset + reconstruction + Rusanov + predict/correct ---------
#ifndef TAFV_K2_MINB
#define TAFV_K2_MINB 7
#endif
// Items: list[i], or base + i (identity: every face of the range active).
template <class P, bool PRED>
__global__ void __launch_bounds__(128, TAFV_K2_MINB) k_face_flux(MeshDev m, StateDev s, PhysParams pp,
                                                   const int* __restrict__ list,
                                                   const int* __restrict__ n_dev, int base, int front,
                                                   const PlanDev* __restrict__ plan, int rev) {
  constexpr int NV = P::NV, D = P::DIM;
  const int n = *n_dev;
  const double dt = plan->dt_min;
  const int stride = gridDim.x * blockDim.x;
  for (int ii = blockIdx.x * blockDim.x + threadIdx.x; ii < n; ii += stride) {
    const int i = rev ? n - 1 - ii : ii;
    // shards: the pass over the interior faces (both sides deep owned: their
    // gradients come from the K1 over the deep cells) runs while the halo is
    // in flight; the border faces' pass after the join (two lists)
    const int f = list ? list[i] : base + i;
    const int2 lr = m.lr[f];
    const double4 gm = ld4(m.geo + f);
    const double nrm[3] = {gm.x, gm.y, gm.z};
    double wL[NV], wR[NV];
    int tl;
    {
      double we[NV];
      tl = stage_spec<NV, (TAFV_ROW128 >= 1)>(s, lr.x, front, PRED, we);
      double g[GradRow<NV>::S];
      load_grad<NV>(s, lr.x, g);
      if (m.fdx) {
        const double4 a = ld4(m.fdx + TAFV_FDX_L(f, m.n_faces));
        const double dl[3] = {a.x, a.y, a.z};
#pragma unroll
        for (int k = 0; k < NV; ++k) wL[k] = extrapolate_d<D>(we[k], g + 3 * k, dl);
      } else {
        const double fc[3] = {m.fcen[3 * (size_t)f], m.fcen[3 * (size_t)f + 1], m.fcen[3 * (size_t)f + 2]};
        const double cl[3] = {m.cen[3 * (size_t)lr.x], m.cen[3 * (size_t)lr.x + 1], m.cen[3 * (size_t)lr.x + 2]};
#pragma unroll
        for (int k = 0; k < NV; ++k) wL[k] = extrapolate<D>(we[k], g + 3 * k, cl, fc);
      }
      if (!P::admissible(pp, wL)) {
#pragma unroll
        for (int k = 0; k < NV; ++k) wL[k] = we[k];
      }
    }
    bool shared_start = (front & ((1 << tl) - 1)) == 0;
    bool eq = true;  // equal-level (or boundary) face
    if (lr.y >= 0) {
      double we[NV];
      const int tr = stage_spec<NV, (TAFV_ROW128 >= 1)>(s, lr.y, front, PRED, we);
      eq = tr == tl;
      shared_start = shared_start && (front & ((1 << tr) - 1)) == 0;
      double g[GradRow<NV>::S];
      load_grad<NV>(s, lr.y, g);
      if (m.fdx) {
        const double4 b = ld4(m.fdx + TAFV_FDX_R(f, m.n_faces));
        const double dr[3] = {b.x, b.y, b.z};
#pragma unroll
        for (int k = 0; k < NV; ++k) wR[k] = extrapolate_d<D>(we[k], g + 3 * k, dr);
      } else {
        const double cr[3] = {m.cen[3 * (size_t)lr.y], m.cen[3 * (size_t)lr.y + 1], m.cen[3 * (size_t)lr.y + 2]};
        const double* to = m.fcen + 3 * (size_t)(m.rcf ? m.rcf[f] : f);
        const double tc[3] = {to[0], to[1], to[2]};
#pragma unroll
        for (int k = 0; k < NV; ++k) wR[k] = extrapolate<D>(we[k], g + 3 * k, cr, tc);
      }
      if (!P::admissible(pp, wR)) {
#pragma unroll
        for (int k = 0; k < NV; ++k) wR[k] = we[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < NV; ++k) wR[k] = wL[k];
    }
    double r[NV];
    rusanov<P>(pp, wL, wR, nrm, r);
    constexpr int FS = FaceRow<NV>::S;
    double* phi = s.phi + (size_t)f * FS;
    double* iwin = s.iwin + (size_t)f * FS;
    if (PRED) {
      double row[FS];
#pragma unroll
      for (int k = 0; k < FS; ++k) row[k] = k < NV ? r[k] * gm.w : 0.0;
#pragma unroll
      for (int q = 0; q < FS; q += 2) st2(phi + q, row[q], row[q + 1]);
      if (shared_start && !(eq && s.ialias)) {
#pragma unroll
        for (int k = 0; k < NV; ++k) iwin[k] = 0.0;
      }
    } else {
      const double dt_sub = dt * (double)(1 << s.cad[f]);
      double* isub = s.isub + (size_t)f * FS;
      const bool skip = eq && s.ialias;
      double row[FS];
#pragma unroll
      for (int q = 0; q < FS; q += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(phi + q));
        row[q] = v.x;
        row[q + 1] = v.y;
      }
#pragma unroll
      for (int k = 0; k < FS; ++k) {
        if (k < NV) {
          const double phi_corr = r[k] * gm.w;
          row[k] = 0.5 * dt_sub * (row[k] + phi_corr);
          if (!skip) iwin[k] = iwin[k] + row[k];
        } else {
          row[k] = 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < FS; q += 2) st2(isub + q, row[q], row[q + 1]);
      if (s.ialias) s.ialias[f] = skip ? 1 : 0;
    }
  }
}

// ---- K3: flux gather + extensive/intensive update ---------------------------
// LAST (trailing corrector over every cell) additionally flags non-finite
// state (kernels.cpp:266-271) and leaves per-block compensated partial sums of
// W for the record (state.cpp:40-44; a deterministic fixed-shape reduction).
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, double b) {
  const double s = a.hi + b;
  const double bb = s - a.hi;
  const double e = (a.hi - (s - bb)) + (b - bb);
  DD r;
  r.hi = s;
  r.lo = a.lo + e;
  return r;
}
__device__ __forceinline__ DD dd_merge(DD a, DD b) {
  DD r = dd_add(a, b.hi);
  r.lo = r.lo + b.lo;
  const double s = r.hi + r.lo;
  r.lo = r.lo - (s - r.hi);
  r.hi = s;
  return r;
}

// Component-parallel like K1: lane k of a cell sums component k of the
// signed face fluxes over the CSR slots in order, then updates its own
// component. LAST (trailing corrector, identity list, all cells) also flags
// non-finite w/W and leaves per-block, per-component compensated partial sums
// of W (fixed shape => deterministic).
template <class P, bool PRED, bool LAST, int DEG>
__global__ void __launch_bounds__(128) k_gather_update(MeshDev m, StateDev s,
                                                       const int* __restrict__ list,
                                                       const int* __restrict__ n_dev,
                                                       PlanDev* plan, DD* partials, int rev) {
  constexpr int NV = P::NV, CPW = 32 / NV;
  const int n = *n_dev;
  const double dt = plan->dt_min;
  const int lane = threadIdx.x & 31;
  const int j = lane / NV, k = lane - j * NV;
  const bool lane_ok = j < CPW;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  DD acc{0.0, 0.0};
  bool bad = false;
  if (lane_ok) {
    for (int ii = warp * CPW + j; ii < n; ii += nwarps * CPW) {
      const int i = rev ? n - 1 - ii : ii;
      const int c = list ? list[i] : i;
      const int tc = __ldg(s.tau + c);
      double sum = 0.0;
      const int s0 = DEG ? DEG * c : m.adj_off[c];
      const int s1 = DEG ? s0 + DEG : m.adj_off[c + 1];
#pragma unroll
      for (int t = s0; t < s1; ++t) {
        const int e = m.adj_face[t];
        const int f = slot_face(e);
        const double* ph;
        if (PRED) ph = s.phi;
        else ph = tc > s.cad[f] ? s.iwin : s.isub;
        sum += slot_sign(e) * ph[(size_t)f * FaceRow<NV>::S + k];
      }
      const size_t ci = (size_t)c * NV + k;
      const double v = m.vol[c];
      if (PRED) {
        const double dtw = dt * (double)(1 << tc);
        s.wp[ci] = (s.W[ci] + dtw * (-sum)) / v;
      } else {
        const double Wn = s.W[ci] + (-sum);
        const double wn = Wn / v;
        s.W[ci] = Wn;
        s.w[ci] = wn;
        if (LAST) {
          bad = bad || !isfinite(Wn) || !isfinite(wn);
          acc = dd_add(acc, Wn);
        }
      }
    }
  }
  if (LAST) {
    if (__syncthreads_or(bad) && threadIdx.x == 0) plan->nonfinite = 1;
    // fixed-shape reduction: lane k of each warp merges its component's lanes
    // k + NV*j (j = 1 .. CPW-1) in order, then thread k merges the warps
    DD a = acc;
#pragma unroll
    for (int jj = 1; jj < CPW; ++jj) {
      DD o;
      o.hi = __shfl_sync(0xffffffffu, acc.hi, (lane + jj * NV) & 31);
      o.lo = __shfl_sync(0xffffffffu, acc.lo, (lane + jj * NV) & 31);
      if (lane < NV) a = dd_merge(a, o);
    }
    __shared__ DD wred[4][NV];
    if (lane < NV) wred[threadIdx.x >> 5][lane] = a;
    __syncthreads();
    if (threadIdx.x < NV) {
      DD b = wred[0][threadIdx.x];
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q) b = dd_merge(b, wred[q][threadIdx.x]);
      partials[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = b;
    }
  }
}

// Conservation ledger (new; the reference keeps none). A transmissive
// face's slot adds +int_substep to its left cell's residual sum
// (flux_sum_correct, kernels.cpp:204-216: tau_c == cadence_f on a boundary
// face, so the substep integral is the one read), i.e. takes it out of the
// domain. After each corrector's K2, on a side stream (off the critical
// path), every boundary face active at `level` (cadence <= level) adds its
// int_substep row to its running outflow bsum[b]; the trailing corrector's
// k_totals reduces and clears them. bface[b] = internal id of the b-th
// transmissive face touching an owned cell.
template <int NV>
__global__ void __launch_bounds__(256) k_ledger(const int* __restrict__ bface, int nb,
                                                const int8_t* __restrict__ cad, int level,
                                                const double* __restrict__ isub, int fs, double* bsum) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const int j = bface[b];
    if (cad[j] > level) continue;
#pragma unroll
    for (int k = 0; k < NV; ++k) bsum[(size_t)b * NV + k] += isub[(size_t)j * fs + k];
  }
}

// Fixed-order reduction of the per-block partials: block k reduces
// component k (deterministic tree over a fixed number of partials) of the
// state totals and, when the ledger runs, of its boundary outflows
// (k_ledger_reduce's partials) into plan->bflux[k].
__device__ __forceinline__ DD block_merge(const DD* part, int n, DD* red) {
  DD a{0.0, 0.0};
  for (int b = threadIdx.x; b < n; b += blockDim.x) a = dd_merge(a, part[b]);
  red[threadIdx.x] = a;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = dd_merge(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  const DD r = red[0];
  __syncthreads();
  return r;
}
// The ledger's per-face boundary outflows into per-block compensated
// partials: block g reduces faces [g*per, (g+1)*per) (fixed shape, so the
// sum is deterministic) component by component, clears them for the next
// iteration and leaves lpart[k][g]. Spread over the whole device: one block
// per component walking ~10^6 faces cost ~3 ms per iteration on config 4.
template <int NV>
__global__ void __launch_bounds__(256) k_ledger_reduce(double* bsum, int nb, DD* lpart) {
  __shared__ DD red[256];
  const int per = (nb + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, b1 = min(nb, b0 + per);
  DD o[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) o[k] = DD{0.0, 0.0};
  for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) {  // one pass over the rows
    double* p = bsum + (size_t)b * NV;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      o[k] = dd_add(o[k], p[k]);
      p[k] = 0.0;
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    red[threadIdx.x] = o[k];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) red[threadIdx.x] = dd_merge(red[threadIdx.x], red[threadIdx.x + w]);
      __syncthreads();
    }
    if (threadIdx.x == 0) lpart[(size_t)k * gridDim.x + blockIdx.x] = red[0];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_totals(const DD* partials, int nblocks, PlanDev* plan, const DD* lpart,
                                                int nl) {
  __shared__ DD red[256];
  const int k = blockIdx.x;
  const DD t = block_merge(partials + (size_t)k * nblocks, nblocks, red);
  if (threadIdx.x == 0) plan->totals[k] = t.hi + t.lo;
  const DD o = lpart ? block_merge(lpart + (size_t)k * nl, nl, red) : DD{0.0, 0.0};
  if (threadIdx.x == 0) plan->bflux[k] = o.hi + o.lo;
}

// ---- plan kernels ----------------------------------------------------------
// kernels.cpp:247-254: dt_max = speed > 0 ? min(dt_cap, cfl*h/speed) : dt_cap,
// and the order-free minimum of kernels.cpp:260-264 in the SAME launch: each
// block leaves its minimum, the last block to finish (fence + ticket) reduces
// them into plan->dt_min. With tau != null (synthetic level maps) the bound is
// dt_max / 2^tau. `reset` (plan_iteration): that block also clears the plan's
// error flag and counts for the counting kernels that follow.
template <class P>
__global__ void __launch_bounds__(256) k_dt_max(MeshDev m, StateDev s, PhysParams pp, double cfl,
                                                double dt_cap, double* dt_max, double* block_min,
                                                const int8_t* tau_scale, int n, unsigned* ticket,
                                                PlanDev* plan, int reset) {
  constexpr int NV = P::NV;
  constexpr double INF = __builtin_huge_val();
  double lowest = INF;
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += stride) {
    double w[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) w[k] = s.w[(size_t)c * NV + k];
    const double speed = P::speed(pp, w);
    const double d = speed > 0.0 ? smin(dt_cap, cfl * m.chl[c] / speed) : dt_cap;
    dt_max[c] = d;
    const double b = tau_scale ? d / (double)(1 << tau_scale[c]) : d;
    lowest = smin(lowest, b);
  }
  // warp-shuffle then per-warp minima (dt_max is never NaN: a NaN speed
  // takes dt_cap, so the order of the exact minimum does not matter)
  __shared__ double red[8];
  __shared__ bool last;
  auto block_reduce = [&](double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = smin(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = red[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) r = smin(r, red[q]);
    __syncthreads();
    return r;
  };
  const double bm = block_reduce(lowest);
  if (threadIdx.x == 0) {
    block_min[blockIdx.x] = bm;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  lowest = INF;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
    lowest = smin(lowest, *((volatile const double*)block_min + b));
  __syncthreads();
  const double dmin = block_reduce(lowest);
  if (threadIdx.x == 0) {
    plan->dt_min = dmin;
    *ticket = 0u;
    if (reset) plan->err = 0;
  }
  if (reset)
    for (int i = threadIdx.x; i < 3 * kMaxLevels; i += blockDim.x) (&plan->cell_count[0])[i] = 0;
  if (reset)
    for (int i = threadIdx.x; i < kMaxLevels; i += blockDim.x) plan->sweep_changed[i] = 0;
}

// levels.cpp:18-25: raw = ratio >= 1 ? ilogb(ratio) : 0, clamped.
// y = rcp_div(dt_min): the quotient is bitwise dt_max / dt_min (div_by).
__device__ __forceinline__ int classify_raw(double dt_max, double dt_min, double y, int theta_max) {
  const double ratio = div_by(dt_max, dt_min, y);
  int raw = 0;
  if (ratio >= 1.0) {
    const long long bits = __double_as_longlong(ratio);
    const int ex = (int)((bits >> 52) & 0x7ff);
    raw = ex == 0x7ff ? 0x7fffffff : ex - 1023;  // ratio >= 1 is normal or +inf
  }
  return raw < 0 ? 0 : (raw > theta_max ? theta_max : raw);
}

__global__ void k_classify(int n, const double* dt_max, const PlanDev* plan, int theta_max,
                           int8_t* raw) {
  const double dt_min = plan->dt_min;
  const bool ok = dt_min > 0.0 && isfinite(dt_min);
  const double y = rcp_div(dt_min);
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += stride)
    raw[c] = ok ? (int8_t)classify_raw(dt_max[c], dt_min, y, theta_max) : (int8_t)0;
}

// levels.cpp:33-46 one Jacobi sweep: out = min(in, 1 + min over neighbours).
__global__ void k_smooth(MeshDev m, const int8_t* in, int8_t* out, int n) {
  const int stride = gridDim.x * blockDim.x;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += stride) {
    int bound = in[c];
    const int s0 = m.adj_off[c], s1 = m.adj_off[c + 1];
    for (int t = s0; t < s1; ++t) {
      const int nb = m.adj_nb[t];
      if (nb >= 0) {
        const int v = in[nb] + 1;
        bound = v < bound ? v : bound;
      }
    }
    out[c] = (int8_t)bound;
  }
}

// Stable per-key compaction. Tile t covers items [t*kTile, (t+1)*kTile); the
// count and scatter passes use the same tiling, so the order inside each key
// bucket is ascending item id.
constexpr int kTile = 2048;
constexpr int kCompactThreads = 256;

// Single-domain plan: classification (levels.cpp:18-25) fused into the first
// Jacobi sweep (levels.cpp:33-46) -- a cell's and each neighbour's raw level
// are classified on the fly from dt_max (the same quotient and exponent every
// time), so no raw array is written -- and the per-tile level counts of the
// compaction fused into the last sweep. FIRST: classify the inputs; SMOOTH
// (theta_max > 0): apply the sweep, else the classification is the level;
// COUNT: block b covers tile b and leaves its counts. clear_flag: the fringe
// flags of the cells swept are cleared for k_face_cadence.
template <bool FIRST, bool COUNT>
__global__ void __launch_bounds__(kCompactThreads) k_level_sweep(MeshDev m, const int8_t* in,
                                                                 const double* dt_max, PlanDev* plan,
                                                                 int theta_max, int smooth, int8_t* out,
                                                                 int n, int nkeys, int* counts,
                                                                 uint8_t* clear_flag, int sweep, int deg,
                                                                 const uint8_t* tile_prev, uint8_t* tile_cur) {
  double dt_min = 0.0, y = 0.0;
  bool ok = false;
  if (FIRST) {
    dt_min = plan->dt_min;
    ok = dt_min > 0.0 && isfinite(dt_min);
    y = rcp_div(dt_min);
  }
  auto lev = [&](int x) -> int {
    if (FIRST) return ok ? classify_raw(dt_max[x], dt_min, y, theta_max) : 0;
    return in[x];
  };
  // Jacobi converged: the previous sweep changed no level, so this one would
  // not either -- copy its input (the fixpoint) instead of re-reading the
  // adjacency (sweeps after the fixpoint cost 2 bytes per cell, not ~30)
  const bool done = !FIRST && plan->sweep_changed[sweep - 1] == 0;
  __shared__ int cnt[kMaxLevels];
  if (COUNT) {
    if (threadIdx.x < kMaxLevels) cnt[threadIdx.x] = 0;
    __syncthreads();
  }
  bool changed = false;
  // tile_cur (block b covers tile b in every sweep): a cell whose level this
  // sweep lowers marks its own tile and its neighbours' tiles; a tile nobody
  // marked in the previous sweep holds only cells whose inputs -- their own
  // and their neighbours' levels -- that sweep left unchanged, so this sweep
  // would reproduce their levels: copied (1 byte per cell read instead of
  // ~30). Exact: the Jacobi iterates are the reference's (levels.cpp:33-46).
  const bool tiled = COUNT || tile_cur != nullptr;
  const bool idle = done || (!FIRST && tile_prev != nullptr && tile_prev[blockIdx.x] == 0);
  const int beg = tiled ? blockIdx.x * kTile + threadIdx.x : blockIdx.x * blockDim.x + threadIdx.x;
  const int end = tiled ? min(n, (int)(blockIdx.x + 1) * kTile) : n;
  const int step = tiled ? blockDim.x : gridDim.x * blockDim.x;
  for (int c = beg; c < end; c += step) {
    const int own = lev(c);
    int bound = own;
    if (smooth && !idle) {
      const int s0 = deg ? deg * c : m.adj_off[c], s1 = deg ? s0 + deg : m.adj_off[c + 1];  // hex: implicit offsets
      for (int t = s0; t < s1; ++t) {
        const int nb = m.adj_nb[t];
        if (nb >= 0) {
          const int v = lev(nb) + 1;
          bound = v < bound ? v : bound;
        }
      }
      if (tile_cur != nullptr && bound != own) {
        tile_cur[c / kTile] = 1;
        for (int t = s0; t < s1; ++t) {
          const int nb = m.adj_nb[t];
          if (nb >= 0 && nb < n) tile_cur[nb / kTile] = 1;
        }
      }
    }
    changed |= bound != own;
    out[c] = (int8_t)bound;
    if (clear_flag) clear_flag[c] = 0;
    if (COUNT) atomicAdd(&cnt[bound], 1);
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) atomicOr(&plan->sweep_changed[sweep], 1);
  if (COUNT) {
    __syncthreads();
    if (threadIdx.x < nkeys) counts[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = cnt[threadIdx.x];
  }
}

// levels.cpp:128-137 face cadence = min(tau_left, tau_right) (boundary: left),
// the fringe flag of levels.cpp:139-153 (the coarser side of a face whose
// sides differ; counted once per owned cell, by the face that sets it) and
// the |dtau| <= 1 invariant the staging relies on, fused with the per-tile
// cadence counts of the face compaction (faces [0, n_count)). Block b covers
// face tile b.
__global__ void __launch_bounds__(kCompactThreads) k_face_cadence(MeshDev m, const int8_t* tau, int8_t* cad,
                                                                  unsigned* fflag32, PlanDev* plan, int n_own,
                                                                  int n_count, int nkeys, int* counts,
                                                                  int ntiles_count) {
  __shared__ int cnt[kMaxLevels], fcnt[kMaxLevels];
  if (threadIdx.x < kMaxLevels) {
    cnt[threadIdx.x] = 0;
    fcnt[threadIdx.x] = 0;
  }
  __syncthreads();
  const int beg = blockIdx.x * kTile, end = min(m.n_faces, beg + kTile);
  for (int f = beg + threadIdx.x; f < end; f += blockDim.x) {
    const int2 lr = m.lr[f];
    const int tl = tau[lr.x];
    int c = tl;
    if (lr.y >= 0) {
      const int tr = tau[lr.y];
      c = tl < tr ? tl : tr;
      if (tl != tr) {
        const int x = tl > tr ? lr.x : lr.y;
        const int kx = tl > tr ? tl : tr;
        const unsigned bit = 1u << (8 * (x & 3));
        const unsigned old = atomicOr(&fflag32[x >> 2], bit);
        if (!(old & bit) && x < n_own) atomicAdd(&fcnt[kx - 1], 1);
        const int d = tl > tr ? tl - tr : tr - tl;
        if (d > 1) atomicOr(&plan->err, 1);
      }
    }
    cad[f] = (int8_t)c;
    if (f < n_count) atomicAdd(&cnt[c], 1);
  }
  __syncthreads();
  if (threadIdx.x < nkeys) {
    if ((int)blockIdx.x < ntiles_count)
      counts[(size_t)threadIdx.x * ntiles_count + blockIdx.x] = cnt[threadIdx.x];
    if (fcnt[threadIdx.x])
      atomicAdd(reinterpret_cast<unsigned long long*>(&plan->fringe_count[threadIdx.x]),
                (unsigned long long)fcnt[threadIdx.x]);
  }
}

// Per-tile counts of keys (cells of an injected map; shard K1 list).
__global__ void __launch_bounds__(kCompactThreads) k_tile_count(const int8_t* key, int n, int nkeys,
                                                                int* counts /*[nkeys][ntiles]*/) {
  __shared__ int cnt[kMaxLevels];
  if (threadIdx.x < kMaxLevels) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int base = blockIdx.x * kTile;
  for (int j = threadIdx.x; j < kTile; j += blockDim.x) {
    const int i = base + j;
    if (i < n) atomicAdd(&cnt[key[i]], 1);
  }
  __syncthreads();
  if (threadIdx.x < nkeys) counts[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = cnt[threadIdx.x];
}

// One compaction (keys, per-tile counts, list, per-key totals, prefix sums of
// the totals = active-set sizes of each level).
struct CompactJob {
  const int8_t* key;
  int n, ntiles;
  int* counts;       // [nkeys][ntiles]: counts in, exclusive offsets out
  int* list;         // item ids base + i (key points at item `base`)
  long long* totals; // [kMaxLevels]
  int* prefix;       // [kMaxLevels]
  int base;
  // or null: per-level CELL totals; the list entries of the top level theta
  // (the highest level with cells) are not written -- every consumer takes a
  // prefix "key <= l" with l < theta, the phases at level theta run over the
  // identity range (single domain only)
  const long long* top_of;
};
__device__ __forceinline__ int skipped_key(const CompactJob& jb, int nkeys) {
  int top = -1;
  if (jb.top_of)
    for (int k = 0; k < nkeys; ++k)
      if (jb.top_of[k] > 0) top = k;
  return top;
}
struct CompactJobs {
  CompactJob j[6 + 2 * kMaxPeers];
  int njobs;
};

// Exclusive scan of each job's counts in (key, tile) order, in place; block b
// scans job b, writes its per-key totals and their prefix sums. Block 0 (the
// K3 cell list) also publishes the record counts and, for a single domain,
// aliases the K1 list to it. Each warp scans a contiguous segment 32 entries
// at a time (coalesced, shuffle scan, running carry), then the warp offsets
// are added: ~10^6 counts (config 4's face tiles) in ~20 us instead of the
// 0.6 ms of per-thread sequential segments.
__global__ void __launch_bounds__(1024) k_tile_scan(CompactJobs jobs, int nkeys, PlanDev* plan,
                                                    int alias_k1) {
  const CompactJob jb = jobs.j[blockIdx.x];
  int* counts = jb.counts;
  const int ntiles = jb.ntiles;
  const int total = ntiles * nkeys;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int per = (total + nw - 1) / nw;
  const int b = min(total, warp * per), e = min(total, b + per);
  int carry = 0;
  for (int base = b; base < e; base += 32) {
    const int i = base + lane;
    const int v = i < e ? counts[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (i < e) counts[i] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  __shared__ int wofs[32];
  __shared__ int grand;
  if (lane == 0) wofs[warp] = carry;
  __syncthreads();
  if (warp == 0) {
    const int v = lane < nw ? wofs[lane] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wofs[lane] = x - v;
    if (lane == 31) grand = x;
  }
  __syncthreads();
  const int off = wofs[warp];
  if (off)
    for (int i = b + lane; i < e; i += 32) counts[i] += off;
  __syncthreads();
  // per-key totals: next key's first offset minus this key's first offset
  if (threadIdx.x < nkeys) {
    long long t = 0;
    if (ntiles > 0) {
      const int first = counts[(size_t)threadIdx.x * ntiles];
      const int next = threadIdx.x + 1 < nkeys ? counts[(size_t)(threadIdx.x + 1) * ntiles] : grand;
      t = next - first;
    }
    jb.totals[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int l = 0; l < kMaxLevels; ++l) {
      const long long t = l < nkeys ? jb.totals[l] : 0;
      acc += t;
      jb.prefix[l] = (int)acc;
      if (blockIdx.x == 0) {
        plan->gcell_count[l] = t;
        if (alias_k1) {
          plan->k1_count[l] = t;
          plan->nk1_prefix[l] = (int)acc;
        }
      }
    }
  }
}

// Scatter of every job in one launch: blocks [0, ntiles_0) job 0, then job 1, ...
__global__ void __launch_bounds__(kCompactThreads) k_tile_scatter(CompactJobs jobs, int nkeys) {
  __shared__ int wcount[kCompactThreads / 32][kMaxLevels];
  __shared__ int running[kMaxLevels];
  int tile = blockIdx.x, q = 0;
  while (q + 1 < jobs.njobs && tile >= jobs.j[q].ntiles) tile -= jobs.j[q++].ntiles;
  const CompactJob jb = jobs.j[q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < nkeys) running[threadIdx.x] = jb.counts[(size_t)threadIdx.x * jb.ntiles + tile];
  const int skip = skipped_key(jb, nkeys);
  const int base = tile * kTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kTile; r += blockDim.x) {
    const int i = base + r + threadIdx.x;
    const int k = i < jb.n ? jb.key[i] : -1;
    int rank = 0;
    for (int kk = 0; kk < nkeys; ++kk) {
      const unsigned mask = __ballot_sync(0xffffffffu, k == kk);
      if (k == kk) rank = __popc(mask & lt);
      if (lane == 0) wcount[warp][kk] = __popc(mask);
    }
    __syncthreads();
    if (k >= 0 && k != skip) {
      int pos = running[k] + rank;
      for (int w = 0; w < warp; ++w) pos += wcount[w][k];
      jb.list[pos] = jb.base + i;
    }
    __syncthreads();
    if (threadIdx.x < nkeys) {
      int tot = 0;
      for (int w = 0; w < kCompactThreads / 32; ++w) tot += wcount[w][threadIdx.x];
      running[threadIdx.x] += tot;
    }
    __syncthreads();
  }
}

// The same scatter for nkeys <= 5 with one block-wide scan per tile: each
// thread takes kTile / kCompactThreads consecutive items, packs its per-key
// counts into 12-bit fields of one 64-bit word (a tile holds <= 2048 items
// per key), and one exclusive scan of the packed words over the block gives
// every thread its stable offset within every key (2 barriers per tile
// instead of 3 per 256 items; 1.3 ms -> ~0.4 ms on config 4's lists).
__global__ void __launch_bounds__(kCompactThreads) k_tile_scatter_packed(CompactJobs jobs, int nkeys) {
  constexpr int IPT = kTile / kCompactThreads;
  __shared__ unsigned long long wsum[kCompactThreads / 32];
  int tile = blockIdx.x, q = 0;
  while (q + 1 < jobs.njobs && tile >= jobs.j[q].ntiles) tile -= jobs.j[q++].ntiles;
  const CompactJob jb = jobs.j[q];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int first = tile * kTile + threadIdx.x * IPT;
  const int skip = skipped_key(jb, nkeys);
  int key[IPT];
  unsigned long long mine = 0;
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int i = first + j;
    key[j] = i < jb.n ? jb.key[i] : -1;
    if (key[j] >= 0) mine += 1ull << (12 * key[j]);
  }
  unsigned long long x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  unsigned long long pre = x - mine;
  for (int w = 0; w < warp; ++w) pre += wsum[w];
#pragma unroll
  for (int j = 0; j < IPT; ++j) {
    const int k = key[j];
    if (k < 0) continue;
    const int pos = jb.counts[(size_t)k * jb.ntiles + tile] + (int)((pre >> (12 * k)) & 0xfff);
    pre += 1ull << (12 * k);
    if (k != skip) jb.list[pos] = jb.base + first + j;
  }
}

// The one-graph iteration's switch: theta of the plan just made (max level
// with cells), or past the last case (no sweep) when plan_iteration would
// have thrown (level error, non-finite or non-positive stable step).
__global__ void k_select_sweep(const PlanDev* plan, cudaGraphConditionalHandle h, int theta_max) {
  if (threadIdx.x != 0) return;
  int th = 0;
  for (int l = 0; l < kMaxLevels; ++l)
    if (plan->gcell_count[l] > 0) th = l;
  const double dt = plan->dt_min;
  const bool ok = plan->err == 0 && isfinite(dt) && dt > 0.0;
  cudaGraphSetConditional(h, ok ? (unsigned)th : (unsigned)theta_max + 1);
}

// Halo rows: pack owned rows for the peers, unpack received halo rows.
// The device plan into pinned host memory (mapped, written over the link by
// the SMs: no copy engine).
__global__ void k_store_plan(const PlanDev* __restrict__ src, PlanDev* dst) {
  static_assert(sizeof(PlanDev) % 8 == 0, "PlanDev is copied in 8-byte words");
  const unsigned long long* a = reinterpret_cast<const unsigned long long*>(src);
  unsigned long long* b = reinterpret_cast<unsigned long long*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(PlanDev) / 8); i += blockDim.x) b[i] = a[i];
}

// Shards: the levels of the listed cells (sort keys of the level-sorted
// exchange lists), and the lists in level order from the compaction.
__global__ void k_gather_keys(const int8_t* tau, const int* idx, int n, int8_t* key) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) key[i] = tau[idx[i]];
}
__global__ void k_permute_list(const int* idx, const int* pos, int n, int* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = idx[pos[i]];
}

__global__ void k_pack_rows(const double* src, const int* idx, int n, int width, double* dst) {
  const size_t total = (size_t)n * width;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    dst[i] = src[(size_t)idx[i / width] * width + i % width];
}
__global__ void k_unpack_rows(const double* src, const int* idx, int n, int width, double* dst) {
  const size_t total = (size_t)n * width;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    dst[(size_t)idx[i / width] * width + i % width] = src[i];
}
__global__ void k_pack_i8(const int8_t* src, const int* idx, int n, int8_t* dst) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[idx[i]];
}
__global__ void k_unpack_i8(const int8_t* src, const int* idx, int n, int8_t* dst) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[idx[i]] = src[i];
}

// ---- state movement (original <-> internal numbering) -----------------------
__global__ void k_gather_rows(const double* src, const int* perm, int n, int width, double* dst) {
  const size_t total = (size_t)n * width;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const size_t row = i / width, col = i % width;
    dst[i] = src[(size_t)perm[row] * width + col];
  }
}

// A state given as W alone, in original row order: W gathered into the
// internal order and w = W / V (intensive_correct, kernels.cpp:237-241), one
// pass (k_gather_rows + k_intensive fused).
__global__ void k_load_extensive(const double* src, const int* perm, const double* vol, int n, int width,
                                 double* W, double* w) {
  const size_t total = (size_t)n * width;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const size_t row = i / width, col = i % width;
    const double v = src[(size_t)perm[row] * width + col];
    W[i] = v;
    w[i] = v / vol[row];
  }
}

// One chunk of rows [r0, r0 + rows) in ORIGINAL order (tafv_gpu_iterate_host
// pipelines the link copies with these): W[inv[r]] = src[r - r0], w = W / V;
// and the reverse gather of a download chunk, dst[r - r0] = W[inv[r]].
__global__ void k_load_extensive_chunk(const double* src, const int* inv, const double* vol, long long r0,
                                       long long rows, int width, double* W, double* w) {
  const long long total = rows * width;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / width, col = i - r * width;
    const long long x = inv[r0 + r];
    const double v = src[i];
    W[x * width + col] = v;
    w[x * width + col] = v / vol[x];
  }
}
__global__ void k_gather_orig_chunk(const double* W, const int* inv, long long r0, long long rows, int width,
                                    double* dst) {
  const long long total = rows * width;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / width, col = i - r * width;
    dst[i] = W[(long long)inv[r0 + r] * width + col];
  }
}

// int_window with aliased (equal-level) faces materialised: isub + 0.0, the
// value the reference's reset-then-accumulate leaves (kernels.cpp:123-130,
// 183-185).
__global__ void k_window_rows(const double* iwin, const double* isub, const uint8_t* alias, int n,
                              int width, int stride, double* dst) {
  const long long total = (long long)n * width;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / width, j = row * stride + i % width;
    dst[i] = alias && alias[row] ? isub[j] + 0.0 : iwin[j];
  }
}

// iwin_alias switched off: faces still aliased get their window materialised
// (0.0 + int_substep, what K2 would have accumulated) and lose the alias.
__global__ void k_materialise_alias(double* iwin, const double* isub, uint8_t* alias, int n, int nv,
                                    int stride) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
    if (!alias[f]) continue;
    for (int k = 0; k < nv; ++k) iwin[(size_t)f * stride + k] = 0.0 + isub[(size_t)f * stride + k];
    alias[f] = 0;
  }
}

__global__ void k_scatter_rows(const double* src, const int* perm, int n, int width, double* dst) {
  const size_t total = (size_t)n * width;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const size_t row = i / width, col = i % width;
    dst[(size_t)perm[row] * width + col] = src[i];
  }
}

// W = w * V (sync_extensive, state.cpp:61-68) for set_state without W.
// w = W / V (intensive_correct, kernels.cpp:237-241)
__global__ void k_intensive(const double* W, const double* vol, int n, int nv, double* w) {
  const size_t total = (size_t)n * nv;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    w[i] = W[i] / vol[i / nv];
}

__global__ void k_sync_extensive(const double* w, const double* vol, int n, int nv, double* W) {
  const size_t total = (size_t)n * nv;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    W[i] = w[i] * vol[i / nv];
}

__global__ void k_gather_i8(const int32_t* src, const int* perm, int n, int8_t* dst, PlanDev* plan,
                            int max_level) {
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = src[perm[i]];
    if (v < 0 || v > max_level) atomicOr(&plan->err, 2);
    dst[i] = (int8_t)(v < 0 ? 0 : (v > max_level ? max_level : v));
  }
}

}  // namespace tafv
