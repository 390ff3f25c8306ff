// Device-side mesh preprocessing for tafv_gpu_create (one-time set-up, not
// the hot path): the caller's mesh arrays are uploaded raw and every derived
// array -- the Morton cell order, the face order, the CSR adjacency in the
// reference's slot order (ascending ORIGINAL face id per cell,
// mesh.cpp:241-271), the closure check (mesh.cpp:273-284), the permuted
// geometry and the hex fast path's per-slot streams -- is built here with
// the same IEEE expressions the host build used (bitwise the same arrays;
// the host build stays available, TAFV_HOST_UPLOAD=1). The three orderings
// are stable radix sorts (CUB), so ties resolve by original id exactly as
// the host's std::sort of (key, id) pairs did.
#pragma once

#include <cstdint>

namespace tafv {
namespace prep {

__device__ __forceinline__ uint64_t spread3_d(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffffull;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

// Range checks of the caller's face arrays (tafv_gpu_create's require()s):
// bit 0 left, bit 1 right, bit 2 partner out of range; bit 3 a periodic link.
__global__ void k_check_faces(const int* fl, const int* fr, const int* fp, int N, int F, int* flags) {
  int bad = 0;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    if (!(fl[f] >= 0 && fl[f] < N)) bad |= 1;
    if (!(fr[f] >= -1 && fr[f] < N)) bad |= 2;
    if (!(fp[f] >= -1 && fp[f] < F)) bad |= 4;
    if (fp[f] >= 0) bad |= 8;
  }
  if (bad) atomicOr(flags, bad);
}

// Per-block min / max of each centroid coordinate (NaN-free inputs; the
// std::min / std::max of the host loop are order-free on finite values).
__global__ void k_bbox_partial(const double* cen, int N, double* part) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x)
    for (int d = 0; d < 3; ++d) {
      const double v = cen[3 * (size_t)c + d];
      lo[d] = v < lo[d] ? v : lo[d];
      hi[d] = hi[d] < v ? v : hi[d];
    }
  __shared__ double s[6][256];
  for (int d = 0; d < 3; ++d) {
    s[d][threadIdx.x] = lo[d];
    s[3 + d][threadIdx.x] = hi[d];
  }
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int d = 0; d < 3; ++d) {
        const double a = s[d][threadIdx.x + w], b = s[3 + d][threadIdx.x + w];
        if (a < s[d][threadIdx.x]) s[d][threadIdx.x] = a;
        if (s[3 + d][threadIdx.x] < b) s[3 + d][threadIdx.x] = b;
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[(size_t)blockIdx.x * 6 + threadIdx.x] = s[threadIdx.x][0];
}
__global__ void k_bbox_final(const double* part, int nb, double* box) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int i = 0; i < nb; ++i)
    for (int d = 0; d < 3; ++d) {
      const double a = part[6 * (size_t)i + d], c = part[6 * (size_t)i + 3 + d];
      if (a < b[d]) b[d] = a;
      if (b[3 + d] < c) b[3 + d] = c;
    }
  for (int k = 0; k < 6; ++k) box[k] = b[k];
}

// 63-bit Morton key of each centroid (upload_mesh's expression, same IEEE
// operations) and the identity values for the stable sort.
__global__ void k_morton(const double* cen, const double* box, int N, uint64_t* key, int* val) {
  const double lo[3] = {box[0], box[1], box[2]}, hi[3] = {box[3], box[4], box[5]};
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < N; c += gridDim.x * blockDim.x) {
    uint64_t k = 0;
    for (int d = 0; d < 3; ++d) {
      const double span = hi[d] - lo[d];
      const double u = span > 0 ? (cen[3 * (size_t)c + d] - lo[d]) / span : 0.0;
      const double x = u * 2097151.0;
      const double q0 = x > 0.0 ? x : 0.0;  // std::max(0.0, x)
      const uint64_t q = (uint64_t)(2097151.0 < q0 ? 2097151.0 : q0);
      k |= spread3_d(q) << d;
    }
    key[c] = k;
    val[c] = c;
  }
}

// Second (stable) pass key: the shard class of the cell at each sorted slot.
__global__ void k_class_keys(const int* order, const uint8_t* cls4, int N, uint32_t* key, int* val) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    key[i] = cls4[order[i]];
    val[i] = order[i];
  }
}

__global__ void k_invert(const int* perm, int n, int* inv) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) inv[perm[i]] = i;
}

// Face order: (touching an owned cell -- shards: interior (both sides deep
// owned, or a boundary face of a deep cell) before border --, internal left
// cell), stable in original face id. cls4: 0 deep owned, 1 owned next to the
// halo, 2 ring 1, 3 ring 2 (null: single domain).
__global__ void k_face_keys(const int* fl, const int* fr, const int* fp, const int* cinv, const uint8_t* touch,
                            const uint8_t* cls4, int N, int F, uint32_t* key, int* val) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    int grp = 0;
    if (touch && !touch[f]) {
      grp = 2;
    } else if (cls4) {
      const int l = fl[f];
      const int r = fr[f] >= 0 ? fr[f] : fp[f] >= 0 ? fl[fp[f]] : -1;
      grp = cls4[l] == 0 && (r < 0 || cls4[r] == 0) ? 0 : 1;
    }
    key[f] = (uint32_t)grp * (uint32_t)N + (uint32_t)cinv[fl[f]];
    val[f] = f;
  }
}

// CSR slot entries: (internal cell, ORIGINAL face id) keys -- sorted, each
// cell's slots follow ascending original face id as mesh.cpp:241-271 builds
// them -- carrying the slot's adj_face value (internal face id, ~id on the
// face's right side). A face without a right cell leaves a sentinel that
// sorts last.
__global__ void k_slot_keys(const int* fl, const int* fr, const int* cinv, const int* finv, int F,
                            uint64_t* key, int* val, int* count) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x) {
    const int L = cinv[fl[f]];
    key[2 * (size_t)f] = ((uint64_t)(uint32_t)L << 32) | (uint32_t)f;
    val[2 * (size_t)f] = finv[f];
    atomicAdd(count + L, 1);
    if (fr[f] >= 0) {
      const int R = cinv[fr[f]];
      key[2 * (size_t)f + 1] = ((uint64_t)(uint32_t)R << 32) | (uint32_t)f;
      val[2 * (size_t)f + 1] = ~finv[f];
      atomicAdd(count + R, 1);
    } else {
      key[2 * (size_t)f + 1] = ~0ull;
      val[2 * (size_t)f + 1] = 0;
    }
  }
}

// Transmissive boundary faces (no right cell, no periodic partner) among
// the faces touching owned cells ([0, F_own) internally), flagged for the
// ledger's compaction (bface).
__global__ void k_boundary_flags(const int* fperm, const int* fr, const int* fp, int F, int F_own, int* flag) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x) {
    const int f = fperm[j];
    flag[j] = (j < F_own && fr[f] < 0 && fp[f] < 0) ? 1 : 0;
  }
}
__global__ void k_boundary_list(const int* flag, const int* idx, int F, int* bface) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x)
    if (flag[j]) bface[idx[j]] = j;
}

// Per internal face: lr, rcf, geo {n, area}, centroid (upload_mesh's loop
// over j).
__global__ void k_face_arrays(const int* fperm, const int* finv, const int* cinv, const int* fl, const int* fr,
                              const int* fp, const double* fn, const double* fa, const double* fc, int F,
                              int periodic, int2* lr, int* rcf, double4* geo, double* fcen) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x) {
    const int f = fperm[j];
    const int rr = fr[f] >= 0 ? fr[f] : fp[f] >= 0 ? fl[fp[f]] : -1;
    lr[j] = make_int2(cinv[fl[f]], rr >= 0 ? cinv[rr] : -1);
    if (periodic) rcf[j] = (fr[f] < 0 && fp[f] >= 0) ? finv[fp[f]] : j;
    geo[j] = make_double4(fn[3 * (size_t)f], fn[3 * (size_t)f + 1], fn[3 * (size_t)f + 2], fa[f]);
    for (int d = 0; d < 3; ++d) fcen[3 * (size_t)j + d] = fc[3 * (size_t)f + d];
  }
}

// Permuted cell arrays and 1 / V (the same IEEE quotient as the host's).
__global__ void k_cell_arrays(const int* cperm, const double* vol0, const double* chl0, const double* cen0, int N,
                              double* vol, double* ivol, double* chl, double* cen) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const int c = cperm[i];
    vol[i] = vol0[c];
    ivol[i] = 1.0 / vol0[c];
    chl[i] = chl0[c];
    for (int d = 0; d < 3; ++d) cen[3 * (size_t)i + d] = cen0[3 * (size_t)c + d];
  }
}

// Slot neighbours (adj_nb): the resolved right cell on the left side (-1
// across a transmissive face), the left cell on the right side.
__global__ void k_slot_nb(const int* adj_face, const int2* lr, int M, int* adj_nb) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < M; t += gridDim.x * blockDim.x) {
    const int e = adj_face[t];
    const int2 p = lr[e >= 0 ? e : ~e];
    adj_nb[t] = e >= 0 ? (p.y >= 0 ? p.y : -1) : p.x;
  }
}

// Geometric closure (mesh.cpp:273-284) on cells [0, n_check): sum over the
// slots, in slot order, of sign * normal * area (the host's expression);
// flags[0] |= 16 on a violation. Also counts cells whose slot count is not 6
// (the hex fast path test) among [0, n_check].
__global__ void k_closure(const int* off, const int* adj_face, const int* fperm, const double* fn, const double* fa,
                          int n_check, int* flags) {
  int bad = 0, not6 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n_check; i += gridDim.x * blockDim.x) {
    if (off[i] != 6 * i) not6 = 1;
    if (i == n_check) continue;
    double s[3] = {0.0, 0.0, 0.0};
    for (int t = off[i]; t < off[i + 1]; ++t) {
      const int e = adj_face[t];
      const int f = fperm[e >= 0 ? e : ~e];
      const double sg = e >= 0 ? 1.0 : -1.0;
      for (int d = 0; d < 3; ++d) s[d] += sg * fn[3 * (size_t)f + d] * fa[f];
    }
    if (fabs(s[0]) > 1e-12 || fabs(s[1]) > 1e-12 || fabs(s[2]) > 1e-12) bad = 1;
  }
  if (bad) atomicOr(flags, 16);
  if (not6) atomicOr(flags, 32);
}

// Hex fast path per-slot streams (cells [0, n_k1)): {n, sign * area} and the
// limiter offsets fc - cc.
__global__ void k_slot_geo(const int* adj_face, const double4* geo, const double* fcen, const double* cen, int n_k1,
                           double4* sgeo, double4* sdx) {
  const long long M6 = 6ll * n_k1;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < M6;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / 6);
    const int e = adj_face[t];
    const int j = e >= 0 ? e : ~e;
    const double4 g = geo[j];
    const double sg = e >= 0 ? 1.0 : -1.0;
    sgeo[t] = make_double4(g.x, g.y, g.z, sg * g.w);
    sdx[t] = make_double4(fcen[3 * (size_t)j] - cen[3 * (size_t)i], fcen[3 * (size_t)j + 1] - cen[3 * (size_t)i + 1],
                          fcen[3 * (size_t)j + 2] - cen[3 * (size_t)i + 2], 0.0);
  }
}

// K2 reconstruction offsets per face (MeshDev::fdx).
__global__ void k_face_dx(const int2* lr, const int* rcf, const double* fcen, const double* cen, int F,
                          int periodic, double4* fdx) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x) {
    const int l = lr[j].x, r = lr[j].y;
    double dl[3], dr[3] = {0.0, 0.0, 0.0};
    for (int d = 0; d < 3; ++d) dl[d] = fcen[3 * (size_t)j + d] - cen[3 * (size_t)l + d];
    if (r >= 0) {
      const int t = periodic ? rcf[j] : j;
      for (int d = 0; d < 3; ++d) dr[d] = fcen[3 * (size_t)t + d] - cen[3 * (size_t)r + d];
    }
    fdx[TAFV_FDX_L(j, F)] = make_double4(dl[0], dl[1], dl[2], 0.0);
    fdx[TAFV_FDX_R(j, F)] = make_double4(dr[0], dr[1], dr[2], 0.0);
  }
}

}  // namespace prep
}  // namespace tafv
