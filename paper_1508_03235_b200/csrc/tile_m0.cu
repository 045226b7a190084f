// tile_m0.cu -- instantiations of the TILED kernel for traffic mode 0
// (uniform random); the kernel is tile_kernel.cuh, the host side tile_engine.cu.
#define NOC_LEAN 1   // node_logic.cuh: no L1 / migration / memory-node code
#include "tile_kernel.cuh"

namespace noc {
#define NOC_TILED_INST(D, F) \
    template __global__ void k_tiled<0, D, F>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);
NOC_TILED_INST(false, 0) NOC_TILED_INST(true, 0) NOC_TILED_INST(false, 1) NOC_TILED_INST(true, 1)
NOC_TILED_INST(false, 2) NOC_TILED_INST(true, 2) NOC_TILED_INST(false, 3) NOC_TILED_INST(true, 3)
NOC_TILED_INST(false, 4) NOC_TILED_INST(true, 4) NOC_TILED_INST(false, 5) NOC_TILED_INST(true, 5)
NOC_TILED_INST(false, 6) NOC_TILED_INST(true, 6) NOC_TILED_INST(false, 7) NOC_TILED_INST(true, 7)
NOC_TILED_INST(false, 8) NOC_TILED_INST(true, 8)   // cluster exchange
#undef NOC_TILED_INST
}  // namespace noc
