// 3D hexahedral mesh generator (host C++), exported as tafv_mesh_hex
// (include/tafv_gpu.h). New code: the reference generator is 1D/2D only
// (proj/core/src/mesh.cpp:302-317). Output is the reference Mesh layout
// (mesh.hpp:26-39) with Vec3 geometry, consumed unchanged by the GPU solver
// (tafv_gpu_create) and by the CPU oracle.
//
// Geometry decisions, fixed here once:
//   * face vector area S = 0.5 * (d1 x d2) of the quad diagonals; area = |S|,
//     normal = S / area, oriented low -> high index (outward on boundaries);
//   * face centroid = vertex average; cell centroid = vertex average;
//   * cell volume = (1/3) sum_f c_f . S_f (outward), the divergence theorem;
//   * char_length = V / max_f area (= h on a uniform cube).
// Interior nodes are jittered by +-jitter x the local spacing per axis with a
// counter-based SplitMix64 (portable, order-free); boundary nodes stay on the
// box. With `permute`, cell and face ids are Fisher-Yates shuffled from the
// seed ("connectivity randomly permuted from seed", BASELINE.json configs).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tafv_gpu.h"

namespace {

inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline double u01(uint64_t seed, uint64_t key) {
  return static_cast<double>(splitmix64(seed ^ (key * 0xD1B54A32D192ED03ull)) >> 11) * 0x1p-53;
}

struct V3 {
  double x, y, z;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

template <class F>
void parallel(int64_t n, F&& f) {
  const int T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 65536 || T == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
  for (auto& x : th) x.join();
}

std::vector<int32_t> shuffled(int64_t n, uint64_t seed) {
  std::vector<int32_t> p(n);
  for (int64_t i = 0; i < n; ++i) p[i] = static_cast<int32_t>(i);
  uint64_t state = seed;
  for (int64_t i = n - 1; i > 0; --i) {
    state = splitmix64(state);
    const uint64_t j = static_cast<uint64_t>((static_cast<unsigned __int128>(state) * (i + 1)) >> 64);
    std::swap(p[i], p[j]);
  }
  return p;
}

struct Quad {
  V3 S, c;
};

// Vector area and centroid of quad p0 p1 p2 p3 (loop order defines the side).
inline Quad quad(V3 p0, V3 p1, V3 p2, V3 p3) {
  const V3 d1 = sub(p2, p0), d2 = sub(p3, p1);
  const V3 x = cross(d1, d2);
  Quad q;
  q.S = {0.5 * x.x, 0.5 * x.y, 0.5 * x.z};
  q.c = {((p0.x + p1.x) + (p2.x + p3.x)) * 0.25, ((p0.y + p1.y) + (p2.y + p3.y)) * 0.25,
         ((p0.z + p1.z) + (p2.z + p3.z)) * 0.25};
  return q;
}

}  // namespace

// The cells [i0, i1) x [j0, j1) x [k0, k1) of the global nx x ny x nz
// lattice on nodes xs[nx+1], ys[ny+1], zs[nz+1]: node positions (jitter key,
// local spacing, "interior" = not on the GLOBAL box) are those of the full
// mesh, so a window's cells are bitwise the full mesh's cells there. Faces
// on the window's sides that are interior in the full mesh become boundary
// faces (transmissive) of the window mesh. The full mesh is the window
// [0, nx) x [0, ny) x [0, nz); only it may be permuted.
static int hex_window(int32_t nx, int32_t ny, int32_t nz, const double* xs, const double* ys, const double* zs,
               const int32_t* box, double jitter, uint64_t seed, int32_t permute, int32_t* n_cells,
               int32_t* n_faces, double* cell_volume, double* cell_centroid, double* cell_char_length,
               int32_t* face_left, int32_t* face_right, int32_t* face_partner, double* face_normal,
               double* face_area, double* face_centroid) {
  if (nx < 1 || ny < 1 || nz < 1) return TAFV_EINVAL;
  const int64_t i0 = box[0], j0 = box[2], k0 = box[4];
  const int64_t wx = int64_t(box[1]) - i0, wy = int64_t(box[3]) - j0, wz = int64_t(box[5]) - k0;
  if (i0 < 0 || j0 < 0 || k0 < 0 || wx < 1 || wy < 1 || wz < 1 || i0 + wx > nx || j0 + wy > ny ||
      k0 + wz > nz)
    return TAFV_EINVAL;
  if (permute && (wx != nx || wy != ny || wz != nz)) return TAFV_EINVAL;
  const int64_t N = wx * wy * wz;
  const int64_t Fx = (wx + 1) * wy * wz, Fy = wx * (wy + 1) * wz, Fz = wx * wy * (wz + 1);
  const int64_t F = Fx + Fy + Fz;
  if (N > INT32_MAX || F > INT32_MAX) return TAFV_EINVAL;
  if (n_cells) *n_cells = static_cast<int32_t>(N);
  if (n_faces) *n_faces = static_cast<int32_t>(F);
  if (!cell_volume) return TAFV_OK;
  for (int i = 0; i < nx; ++i)
    if (!(xs[i + 1] > xs[i])) return TAFV_EINVAL;
  for (int i = 0; i < ny; ++i)
    if (!(ys[i + 1] > ys[i])) return TAFV_EINVAL;
  for (int i = 0; i < nz; ++i)
    if (!(zs[i + 1] > zs[i])) return TAFV_EINVAL;

  // Node lattice of the window with the full mesh's jitter (global keys).
  const int64_t GX = nx + 1, GY = ny + 1;
  const int64_t NX = wx + 1, NY = wy + 1, NZ = wz + 1;
  std::vector<V3> node(NX * NY * NZ);
  auto nid = [&](int64_t i, int64_t j, int64_t k) { return (k * NY + j) * NX + i; };  // window-local
  auto local = [](const double* a, int64_t i) { return std::min(a[i] - a[i - 1], a[i + 1] - a[i]); };
  parallel(NZ, [&](int64_t a0, int64_t a1) {
    for (int64_t k = a0; k < a1; ++k)
      for (int64_t j = 0; j < NY; ++j)
        for (int64_t i = 0; i < NX; ++i) {
          const int64_t gi = i0 + i, gj = j0 + j, gk = k0 + k;
          V3 p{xs[gi], ys[gj], zs[gk]};
          const bool interior = gi > 0 && gi < nx && gj > 0 && gj < ny && gk > 0 && gk < nz;
          if (interior && jitter != 0.0) {
            const uint64_t key = static_cast<uint64_t>((gk * GY + gj) * GX + gi) * 3;
            p.x += jitter * local(xs, gi) * (2.0 * u01(seed, key) - 1.0);
            p.y += jitter * local(ys, gj) * (2.0 * u01(seed, key + 1) - 1.0);
            p.z += jitter * local(zs, gk) * (2.0 * u01(seed, key + 2) - 1.0);
          }
          node[nid(i, j, k)] = p;
        }
  });
  nx = static_cast<int32_t>(wx);  // from here on: the window's own lattice
  ny = static_cast<int32_t>(wy);
  nz = static_cast<int32_t>(wz);
  std::vector<int32_t> cperm, fperm;
  if (permute) {
    cperm = shuffled(N, splitmix64(seed ^ 0xC3115ull));
    fperm = shuffled(F, splitmix64(seed ^ 0xFACE5ull));
  }
  auto cell_id = [&](int64_t i, int64_t j, int64_t k) -> int32_t {
    const int64_t s = (k * ny + j) * nx + i;
    return permute ? cperm[s] : static_cast<int32_t>(s);
  };
  auto face_id = [&](int64_t s) -> int32_t { return permute ? fperm[s] : static_cast<int32_t>(s); };

  // Faces normal to an axis: Q(plane, a, b) in lexicographic order.
  auto xq = [&](int64_t i, int64_t j, int64_t k) {
    return quad(node[nid(i, j, k)], node[nid(i, j + 1, k)], node[nid(i, j + 1, k + 1)],
                node[nid(i, j, k + 1)]);
  };
  auto yq = [&](int64_t i, int64_t j, int64_t k) {
    return quad(node[nid(i, j, k)], node[nid(i, j, k + 1)], node[nid(i + 1, j, k + 1)],
                node[nid(i + 1, j, k)]);
  };
  auto zq = [&](int64_t i, int64_t j, int64_t k) {
    return quad(node[nid(i, j, k)], node[nid(i + 1, j, k)], node[nid(i + 1, j + 1, k)],
                node[nid(i, j + 1, k)]);
  };
  auto put_face = [&](int64_t s, const Quad& q, int32_t left, int32_t right, bool flip) {
    const int32_t f = face_id(s);
    V3 S = q.S;
    if (flip) S = {-S.x, -S.y, -S.z};
    const double a = std::sqrt(dot(S, S));
    face_left[f] = left;
    face_right[f] = right;
    face_partner[f] = -1;
    face_area[f] = a;
    face_normal[3 * f] = S.x / a;
    face_normal[3 * f + 1] = S.y / a;
    face_normal[3 * f + 2] = S.z / a;
    face_centroid[3 * f] = q.c.x;
    face_centroid[3 * f + 1] = q.c.y;
    face_centroid[3 * f + 2] = q.c.z;
  };
  parallel(nz, [&](int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i <= nx; ++i) {
          const int64_t s = (k * ny + j) * (nx + 1) + i;
          const Quad q = xq(i, j, k);
          if (i == 0) put_face(s, q, cell_id(0, j, k), -1, true);
          else if (i == nx) put_face(s, q, cell_id(nx - 1, j, k), -1, false);
          else put_face(s, q, cell_id(i - 1, j, k), cell_id(i, j, k), false);
        }
  });
  parallel(nz, [&](int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k)
      for (int64_t j = 0; j <= ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          const int64_t s = Fx + (k * (ny + 1) + j) * nx + i;
          const Quad q = yq(i, j, k);
          if (j == 0) put_face(s, q, cell_id(i, 0, k), -1, true);
          else if (j == ny) put_face(s, q, cell_id(i, ny - 1, k), -1, false);
          else put_face(s, q, cell_id(i, j - 1, k), cell_id(i, j, k), false);
        }
  });
  parallel(nz + 1, [&](int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          const int64_t s = Fx + Fy + (k * ny + j) * nx + i;
          const Quad q = zq(i, j, k);
          if (k == 0) put_face(s, q, cell_id(i, j, 0), -1, true);
          else if (k == nz) put_face(s, q, cell_id(i, j, nz - 1), -1, false);
          else put_face(s, q, cell_id(i, j, k - 1), cell_id(i, j, k), false);
        }
  });

  // Cells: volume by the divergence theorem over the 6 outward faces.
  parallel(nz, [&](int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k)
      for (int64_t j = 0; j < ny; ++j)
        for (int64_t i = 0; i < nx; ++i) {
          const int32_t c = cell_id(i, j, k);
          const Quad q[6] = {xq(i + 1, j, k), xq(i, j, k), yq(i, j + 1, k),
                             yq(i, j, k),     zq(i, j, k + 1), zq(i, j, k)};
          double v = 0.0, amax = 0.0;
          for (int t = 0; t < 6; ++t) {
            const double sgn = (t % 2 == 0) ? 1.0 : -1.0;
            v += sgn * dot(q[t].c, q[t].S);
            amax = std::max(amax, std::sqrt(dot(q[t].S, q[t].S)));
          }
          v = v / 3.0;
          V3 cc{0.0, 0.0, 0.0};
          for (int dk = 0; dk < 2; ++dk)
            for (int dj = 0; dj < 2; ++dj)
              for (int di = 0; di < 2; ++di) {
                const V3 p = node[nid(i + di, j + dj, k + dk)];
                cc.x += p.x;
                cc.y += p.y;
                cc.z += p.z;
              }
          cell_volume[c] = v;
          cell_centroid[3 * c] = cc.x * 0.125;
          cell_centroid[3 * c + 1] = cc.y * 0.125;
          cell_centroid[3 * c + 2] = cc.z * 0.125;
          cell_char_length[c] = v / amax;
        }
  });
  return TAFV_OK;
}

extern "C" int tafv_mesh_hex(int32_t nx, int32_t ny, int32_t nz, const double* xs,
                             const double* ys, const double* zs, double jitter, uint64_t seed,
                             int32_t permute, int32_t* n_cells, int32_t* n_faces,
                             double* cell_volume, double* cell_centroid, double* cell_char_length,
                             int32_t* face_left, int32_t* face_right, int32_t* face_partner,
                             double* face_normal, double* face_area, double* face_centroid) {
  const int32_t box[6] = {0, nx, 0, ny, 0, nz};
  return hex_window(nx, ny, nz, xs, ys, zs, box, jitter, seed, permute, n_cells, n_faces, cell_volume,
                    cell_centroid, cell_char_length, face_left, face_right, face_partner, face_normal,
                    face_area, face_centroid);
}

extern "C" int tafv_mesh_hex_window(int32_t nx, int32_t ny, int32_t nz, const double* xs, const double* ys,
                                    const double* zs, const int32_t* box6, double jitter, uint64_t seed,
                                    int32_t* n_cells, int32_t* n_faces, double* cell_volume,
                                    double* cell_centroid, double* cell_char_length, int32_t* face_left,
                                    int32_t* face_right, int32_t* face_partner, double* face_normal,
                                    double* face_area, double* face_centroid) {
  if (!box6) return TAFV_EINVAL;
  return hex_window(nx, ny, nz, xs, ys, zs, box6, jitter, seed, 0, n_cells, n_faces, cell_volume,
                    cell_centroid, cell_char_length, face_left, face_right, face_partner, face_normal,
                    face_area, face_centroid);
}
