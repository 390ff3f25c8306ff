// Domain decomposition for the multi-GPU path (see shard.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tafv_gpu.h"

namespace tafv {

struct Shard {
  int rank = 0, nranks = 1;
  int n_own = 0, n_r1 = 0, n_r2 = 0;
  std::vector<int> cells;         // local -> global cell id (ascending)
  std::vector<uint8_t> cls;       // 0 owned, 1 ring 1, 2 ring 2
  std::vector<int> faces;         // local -> global face id (ascending)
  std::vector<uint8_t> touch_own; // face has an owned side
  std::vector<int> peers;         // ranks sharing cells with this one
  std::vector<std::vector<int>> send, recv;  // local cell ids per peer, ascending global id
  // local mesh arrays (reference layout)
  std::vector<double> vol, cen, chl, fn, fa, fc;
  std::vector<int32_t> fl, fr, fp;
  tafv_mesh_view view(int dim) const;
};

void partition_slabs(const tafv_mesh_view& m, int nranks, int axis, const double* weight,
                     int32_t* rank_of_cell);
Shard build_shard(const tafv_mesh_view& m, const int32_t* rank_of_cell, int rank, int nranks);

}  // namespace tafv
