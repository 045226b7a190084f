// persist_lean.cu -- the lean PERSIST kernels (UR, plain LSPD): NOC_LEAN
// compiles the private-L1, migration and memory-node paths out of the node
// step; the full LSPD kernel is instantiated in kernels.cu.
#define NOC_LEAN 1
#include "persist_kernel.cuh"

namespace noc {
const void *persist_fn_lean(uint32_t mode)
{
    return mode == 1u ? (const void *)k_persist<1> : (const void *)k_persist<0>;
}
}  // namespace noc
