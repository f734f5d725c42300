// tma_host.h -- host-side tensor-map construction shared by the TMA kernels
// (k_tma.cu, k_qft13.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <vector>

namespace qs {

// Build the 5-D tensor map of one side of a tile pass over a shard of 2^nl
// amplitudes at base: pos_of_tile[b] = the position of box bit b; fixed
// position p carries tile-id bit fid[p] (-1 for box positions).  first[d] /
// len[d] give, per tensor dim d, the tile-id bit run it addresses (len 0: a
// box dim); rank[b] = index bit of box bit b in the box layout (by position).
// False if the geometry needs more than 5 dims, position 0 is not a box
// position, or a fixed run is not a consecutive tile-id range.
bool build_side(const double2 *base, int nl, const std::vector<int> &pos_of_tile, const std::vector<int> &fid,
                CUtensorMap &map, int (&first)[5], int (&len)[5], int *rank);

}  // namespace qs
