// Domain decomposition for the multi-GPU path (host C++).
//
// Model (reference decomposition PAPER.md:366-370,
// ce.cpp:66-90, exchange.cpp:363-375): every cell is owned by one rank; a
// rank stores its owned cells O, ring 1 R1 (face neighbours of O outside O)
// and ring 2 R2 (face neighbours of R1 outside O u R1), and every face that
// touches O u R1, so O and R1 cells have their complete CSR adjacency. Faces
// between ranks are duplicated and evaluated bitwise-identically on both
// sides. Local ids are ascending GLOBAL ids (cells and faces), so every
// per-cell slot order is the reference's global order. Exchange lists pair
// (owned cells of r in q's halo) with (q's halo cells owned by r), both
// sorted by global id.
//
// Slab partition: contiguous slabs along an axis with cut positions
// balancing a per-cell weight (level cost 2^(theta - tau) when given,
// exchange.cpp:598-603), ties broken by global id.

#include "shard.h"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

namespace tafv {

void partition_slabs(const tafv_mesh_view& m, int nranks, int axis, const double* weight,
                     int32_t* rank_of_cell) {
  if (nranks < 1) throw std::invalid_argument("partition: nranks must be >= 1");
  if (axis < 0 || axis > 2) throw std::invalid_argument("partition: axis must be 0, 1 or 2");
  const int N = m.n_cells;
  std::vector<int> order(N);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return m.cell_centroid[3 * (size_t)a + axis] < m.cell_centroid[3 * (size_t)b + axis];
  });
  double total = 0.0;
  for (int c = 0; c < N; ++c) total += weight ? weight[c] : 1.0;
  double acc = 0.0;
  for (int i = 0; i < N; ++i) {
    const int c = order[i];
    const double w = weight ? weight[c] : 1.0;
    int r = (int)std::floor((acc + 0.5 * w) / total * nranks);
    rank_of_cell[c] = std::min(nranks - 1, std::max(0, r));
    acc += w;
  }
}

Shard build_shard(const tafv_mesh_view& m, const int32_t* rank_of_cell, int rank, int nranks) {
  const int N = m.n_cells, F = m.n_faces;
  // resolved right cell (kernels.cpp:15-20): the right cell, or across a
  // periodic boundary the partner face's left cell, or -1 (transmissive)
  auto rright = [&](int f) {
    if (m.face_right[f] >= 0) return m.face_right[f];
    return m.face_partner[f] >= 0 ? m.face_left[m.face_partner[f]] : -1;
  };
  for (int c = 0; c < N; ++c)
    if (rank_of_cell[c] < 0 || rank_of_cell[c] >= nranks)
      throw std::invalid_argument("shard: rank_of_cell out of range");
  // neighbour CSR (global)
  // (a periodic link appears once from each of its two boundary faces)
  std::vector<int> off(N + 1, 0);
  for (int f = 0; f < F; ++f) {
    if (m.face_right[f] >= 0) {
      ++off[m.face_left[f] + 1];
      ++off[m.face_right[f] + 1];
    } else if (m.face_partner[f] >= 0) {
      ++off[m.face_left[f] + 1];
    }
  }
  for (int c = 0; c < N; ++c) off[c + 1] += off[c];
  std::vector<int> nb(off[N]);
  {
    std::vector<int> cur(off.begin(), off.end() - 1);
    for (int f = 0; f < F; ++f)
      if (m.face_right[f] >= 0) {
        nb[cur[m.face_left[f]]++] = m.face_right[f];
        nb[cur[m.face_right[f]]++] = m.face_left[f];
      } else if (m.face_partner[f] >= 0) {
        nb[cur[m.face_left[f]]++] = rright(f);
      }
  }
  // ring classes per rank q: 0 owned, 1 ring 1, 2 ring 2, 3 absent
  auto classes = [&](int q) {
    std::vector<uint8_t> cls(N, 3);
    for (int c = 0; c < N; ++c)
      if (rank_of_cell[c] == q) cls[c] = 0;
    for (int ring = 1; ring <= 2; ++ring)
      for (int c = 0; c < N; ++c)
        if (cls[c] == ring - 1)
          for (int t = off[c]; t < off[c + 1]; ++t)
            if (cls[nb[t]] == 3) cls[nb[t]] = (uint8_t)ring;
    return cls;
  };
  Shard s;
  s.rank = rank;
  s.nranks = nranks;
  const std::vector<uint8_t> mine = classes(rank);
  std::vector<int> local(N, -1);
  for (int c = 0; c < N; ++c)
    if (mine[c] <= 2) {
      local[c] = (int)s.cells.size();
      s.cells.push_back(c);
      s.cls.push_back(mine[c]);
      if (mine[c] == 0) ++s.n_own;
      else if (mine[c] == 1) ++s.n_r1;
      else ++s.n_r2;
    }
  // faces with a side in owned or ring 1 (a kept periodic face's partner is
  // kept too: its sides are the same two cells)
  std::vector<int> lface(F, -1);
  for (int f = 0; f < F; ++f) {
    const int l = m.face_left[f], r = rright(f);
    const bool keep = mine[l] <= 1 || (r >= 0 && mine[r] <= 1);
    if (!keep) continue;
    lface[f] = (int)s.faces.size();
    s.faces.push_back(f);
    s.touch_own.push_back(mine[l] == 0 || (r >= 0 && mine[r] == 0) ? 1 : 0);
  }
  const int nc = (int)s.cells.size(), nf = (int)s.faces.size();
  s.vol.resize(nc);
  s.cen.resize(3 * (size_t)nc);
  s.chl.resize(nc);
  for (int i = 0; i < nc; ++i) {
    const int c = s.cells[i];
    s.vol[i] = m.cell_volume[c];
    s.chl[i] = m.cell_char_length[c];
    for (int d = 0; d < 3; ++d) s.cen[3 * (size_t)i + d] = m.cell_centroid[3 * (size_t)c + d];
  }
  s.fl.resize(nf);
  s.fr.resize(nf);
  s.fp.assign(nf, -1);
  s.fn.resize(3 * (size_t)nf);
  s.fa.resize(nf);
  s.fc.resize(3 * (size_t)nf);
  for (int j = 0; j < nf; ++j) {
    const int f = s.faces[j];
    s.fl[j] = local[m.face_left[f]];
    s.fr[j] = m.face_right[f] >= 0 ? local[m.face_right[f]] : -1;
    if (s.fl[j] < 0 || (m.face_right[f] >= 0 && s.fr[j] < 0))
      throw std::logic_error("shard: face side outside the local cell set");
    if (m.face_right[f] < 0 && m.face_partner[f] >= 0) {
      s.fp[j] = lface[m.face_partner[f]];
      if (s.fp[j] < 0 || local[rright(f)] < 0)
        throw std::logic_error("shard: periodic partner outside the local face set");
    }
    s.fa[j] = m.face_area[f];
    for (int d = 0; d < 3; ++d) {
      s.fn[3 * (size_t)j + d] = m.face_normal[3 * (size_t)f + d];
      s.fc[3 * (size_t)j + d] = m.face_centroid[3 * (size_t)f + d];
    }
  }
  // exchange lists with every peer that shares cells
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    const std::vector<uint8_t> theirs = classes(q);
    std::vector<int> send, recv;
    for (int c = 0; c < N; ++c) {
      if (mine[c] == 0 && (theirs[c] == 1 || theirs[c] == 2)) send.push_back(local[c]);
      if ((mine[c] == 1 || mine[c] == 2) && theirs[c] == 0) recv.push_back(local[c]);
    }
    if (send.empty() && recv.empty()) continue;
    s.peers.push_back(q);
    s.send.push_back(std::move(send));
    s.recv.push_back(std::move(recv));
  }
  return s;
}

tafv_mesh_view Shard::view(int dim) const {
  return tafv_mesh_view{dim, (int32_t)cells.size(), (int32_t)faces.size(), vol.data(), cen.data(),
                        chl.data(), fl.data(), fr.data(), fp.data(), fn.data(), fa.data(), fc.data()};
}

}  // namespace tafv

// ---- C ABI (host only: usable without a GPU) --------------------------------
namespace {
thread_local std::string g_shard_err;
}

extern "C" int tafv_partition_slabs(const tafv_mesh_view* m, int32_t nranks, int32_t axis,
                                    const double* weight, int32_t* rank_of_cell) {
  try {
    tafv::partition_slabs(*m, nranks, axis, weight, rank_of_cell);
    return TAFV_OK;
  } catch (const std::invalid_argument& e) {
    g_shard_err = e.what();
    return TAFV_EINVAL;
  }
}

extern "C" int tafv_shard_describe(const tafv_mesh_view* m, const int32_t* rank_of_cell, int32_t rank,
                                   int32_t nranks, int32_t* counts, int32_t* cells, int32_t* faces,
                                   int32_t* peers, int32_t* send_counts, int32_t* recv_counts,
                                   int32_t* send_flat, int32_t* recv_flat) {
  try {
    const tafv::Shard s = tafv::build_shard(*m, rank_of_cell, rank, nranks);
    // counts: n_own, n_r1, n_r2, n_faces, n_faces_touching_owned, n_peers, send total, recv total
    int fo = 0;
    for (uint8_t t : s.touch_own) fo += t;
    size_t st = 0, rt = 0;
    for (auto& v : s.send) st += v.size();
    for (auto& v : s.recv) rt += v.size();
    const int32_t cnt[8] = {s.n_own, s.n_r1, s.n_r2, (int32_t)s.faces.size(), fo,
                            (int32_t)s.peers.size(), (int32_t)st, (int32_t)rt};
    if (counts) std::copy(cnt, cnt + 8, counts);
    if (cells) std::copy(s.cells.begin(), s.cells.end(), cells);
    if (faces) std::copy(s.faces.begin(), s.faces.end(), faces);
    if (peers) std::copy(s.peers.begin(), s.peers.end(), peers);
    size_t so = 0, ro = 0;
    for (size_t p = 0; p < s.peers.size(); ++p) {
      if (send_counts) send_counts[p] = (int32_t)s.send[p].size();
      if (recv_counts) recv_counts[p] = (int32_t)s.recv[p].size();
      if (send_flat) std::copy(s.send[p].begin(), s.send[p].end(), send_flat + so);
      if (recv_flat) std::copy(s.recv[p].begin(), s.recv[p].end(), recv_flat + ro);
      so += s.send[p].size();
      ro += s.recv[p].size();
    }
    return TAFV_OK;
  } catch (const std::invalid_argument& e) {
    g_shard_err = e.what();
    return TAFV_EINVAL;
  } catch (const std::exception& e) {
    g_shard_err = e.what();
    return TAFV_ELOGIC;
  }
}

// smooth_sweep / smooth_to_fixpoint (levels.cpp:33-51) on the host: Jacobi
// tau <- min(tau, 1 + min over face neighbours) until no change (resolved
// right across periodic links). Used for the slab cut weights of a
// decomposed run (the initial plan's levels, before any device exists) and
// for synthetic level maps.
extern "C" int tafv_level_smooth(const tafv_mesh_view* m, int32_t* tau) {
  try {
    if (!m || !tau) throw std::invalid_argument("level_smooth: null argument");
    const int N = m->n_cells, F = m->n_faces;
    std::vector<int32_t> next(tau, tau + N);
    for (;;) {
      for (int f = 0; f < F; ++f) {
        const int l = m->face_left[f];
        const int r = m->face_right[f] >= 0 ? m->face_right[f]
                      : m->face_partner[f] >= 0 ? m->face_left[m->face_partner[f]] : -1;
        if (r < 0) continue;
        next[l] = std::min(next[l], tau[r] + 1);
        next[r] = std::min(next[r], tau[l] + 1);
      }
      bool changed = false;
      for (int c = 0; c < N; ++c)
        if (next[c] != tau[c]) {
          changed = true;
          tau[c] = next[c];
        }
      if (!changed) return TAFV_OK;
    }
  } catch (const std::exception& e) {
    g_shard_err = e.what();
    return TAFV_EINVAL;
  }
}

extern "C" const char* tafv_shard_last_error() { return g_shard_err.c_str(); }
