// kernels.h -- launch wrappers of kernels.cu, used by runtime.cu.
#pragma once
#include "common.cuh"

namespace noc {

constexpr uint32_t PERSIST_BLOCK = 256;
constexpr uint32_t TILE_BLOCK_MAX = 512;                  // nodes (= threads) per CTA
constexpr uint32_t TILE_MIN_BLOCKS = 1;                   // co-resident CTAs per SM

// TILED engine (tile_engine.cu): configure picks the tiling (sets S.TX, S.TY)
cudaError_t tiled_configure(Dev &S, int device, uint32_t *grid, uint32_t *tpad, uint32_t *smem_hist);
cudaError_t launch_tiled(const Dev &S, uint64_t t0, uint32_t ncyc, uint32_t grid, uint32_t tpad, uint32_t smem_hist,
                         uint32_t *activity, cudaStream_t st);
cudaError_t launch_ll_reset(const Dev &S, uint64_t t, cudaStream_t st);

cudaError_t launch_step(const Dev &S, uint64_t t, uint32_t *activity, cudaStream_t st);
cudaError_t persist_configure(const Dev &S, int device, uint32_t *grid, uint32_t *nodes_per_cta,
                              uint32_t *smem_hist);
cudaError_t launch_persist(const Dev &S, uint64_t t0, uint32_t ncyc, uint32_t *progress, uint32_t pbase,
                           uint32_t grid, uint32_t nodes_per_cta, uint32_t smem_hist, uint32_t *activity,
                           cudaStream_t st);
cudaError_t launch_busy_count(const Dev &S, uint64_t t, uint32_t *out, cudaStream_t st);
cudaError_t launch_hash(const Dev &S, uint64_t t, unsigned long long *out, cudaStream_t st);

}  // namespace noc
