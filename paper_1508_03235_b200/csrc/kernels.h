// kernels.h -- launch wrappers of kernels.cu, used by runtime.cu.
#pragma once
#include "common.cuh"

namespace noc {

#ifndef NOC_PERSIST_BLOCK
#define NOC_PERSIST_BLOCK 256   // A/B builds: -DNOC_PERSIST_BLOCK=N
#endif
constexpr uint32_t PERSIST_BLOCK = NOC_PERSIST_BLOCK;
// 3 co-resident PERSIST CTAs per SM (<= 80 registers): large meshes are DRAM-latency
// bound and need the warps (A/B at C5: 24 vs 16 warps per SM, -18% per cycle)
#ifndef NOC_PERSIST_MIN_BLOCKS
#define NOC_PERSIST_MIN_BLOCKS 3   // A/B builds: -DNOC_PERSIST_MIN_BLOCKS=N
#endif
constexpr uint32_t PERSIST_MIN_BLOCKS = NOC_PERSIST_MIN_BLOCKS;
constexpr uint32_t TILE_BLOCK_MAX = 320;                  // nodes per CTA: C3 tiles are 300 (the 320 cap beat 512 by 2.7 % in round 1)
constexpr uint32_t TILE_MIN_BLOCKS = 1;                   // co-resident CTAs per SM
// boundary-ring nodes per ring warp at most (tile_kernel.cuh ring_map); below
// 32 the block gets extra ring warps, up to TILE_THREADS_MAX threads
#ifndef NOC_RING_CAP
#define NOC_RING_CAP 4
#endif
constexpr uint32_t TILE_RING_CAP = NOC_RING_CAP;
#ifndef NOC_TILE_THREADS
#define NOC_TILE_THREADS (NOC_RING_CAP >= 32 ? 320 : 384)
#endif
constexpr uint32_t TILE_THREADS_MAX = NOC_TILE_THREADS;   // launch bound (384: <= 170 registers, 157 used)
// (A/B, profiles/r02_ab_split_barrier.txt: a 384-thread CTA gives C3's 76 ring nodes 5 warps of <= 16,
// C3 -3 %; C2's 30-node tiles get an interior warp and 5 ring warps of <= 4, C2 -27 % (cap 8: -25 %); 416 threads
// squeeze the kernel to 128 registers and are slower)

// Row bands handled by one process (virtual bands on one GPU, or the single
// band of a rank); every band's tiles run in one cooperative launch.
constexpr uint32_t MAX_BANDS = 8;
struct DevSet {
    Dev d[MAX_BANDS];
    uint32_t nbands;
    uint32_t tile0[MAX_BANDS + 1];   // first CTA of each band
    uint32_t general;                // several bands or ranks: band lookup and system-scope band-edge links
    uint32_t cluster;                // TILED cluster exchange: the tiles form one cluster (FEAT bit 3)
};

// TILED engine (tile_engine.cu): tiled_plan picks the tiling of one band
// (sets S.TX, S.TY) within tiles_budget CTAs; tiled_prepare sets the launch
// attributes for all bands' tiles in one cooperative launch
bool tiled_plan(Dev &S, uint32_t tiles_budget, uint32_t *tiles, uint32_t *np);
// TILED kernel variant for a band: 0 UR, 1 lean LSPD, 2 full LSPD (tile_engine.cu)
uint32_t tiled_kernel_mode(const Dev &D);
// streamed scripts (NEXT-f3, R57): per-node counts and the merge of pushed events
cudaError_t launch_script_count(const Dev &S, const uint32_t *add_off, uint32_t *cnt, cudaStream_t st);
cudaError_t launch_script_merge(const Dev &S, const uint32_t *add_off, const uint4 *add_ev, const uint32_t *new_off,
                                uint4 *new_ev, uint32_t *new_base, cudaStream_t st);
// the cluster exchange: one band of <= TILE_CLUSTER_MAX tiles as one cluster
constexpr uint32_t TILE_CLUSTER_MAX = 16;
cudaError_t tiled_prepare_cluster(uint32_t mode, uint32_t nb, uint32_t np, uint32_t tiles, uint32_t *smem_hist);
cudaError_t tiled_prepare(uint32_t mode, uint32_t route, uint32_t nb, uint32_t np, uint32_t total_tiles, int device,
                          uint32_t *smem_hist);
cudaError_t launch_tiled(const DevSet &P, uint64_t t0, uint32_t ncyc, uint32_t tpad, uint32_t smem_hist,
                         uint32_t *activity, cudaStream_t st);
cudaError_t launch_ll_refresh(const Dev &S, uint64_t t0, cudaStream_t st);

// TILED4 engine (tile4_engine.cu): 4 lanes per node, <= 160 nodes per CTA,
// 2 CTAs per SM
constexpr uint32_t TILE4_BLOCK_MAX = 640;
constexpr uint32_t TILE4_MIN_BLOCKS = 2;
bool tiled4_plan(Dev &S, uint32_t tiles_budget, uint32_t *tiles, uint32_t *np);
cudaError_t tiled4_prepare(uint32_t mode, uint32_t nb, uint32_t np, uint32_t total_tiles, int device,
                           uint32_t *smem_hist);
cudaError_t launch_tiled4(const DevSet &P, uint64_t t0, uint32_t ncyc, uint32_t np, uint32_t smem_hist,
                          uint32_t *activity, cudaStream_t st);
cudaError_t launch_ll_reset(const Dev &S, uint64_t t, cudaStream_t st);

// lean PERSIST kernel (persist_lean.cu) for traffic mode 0 / 1
const void *persist_fn_lean(uint32_t mode);
cudaError_t launch_step(const Dev &S, uint64_t t, uint32_t *activity, cudaStream_t st);
cudaError_t persist_configure(const Dev &S, int device, uint32_t nbands, uint32_t *grid, uint32_t *nodes_per_cta,
                              uint32_t *smem_hist);
cudaError_t launch_persist(const DevSet &P, uint64_t t0, uint32_t ncyc, uint32_t pbase, uint32_t smem_hist,
                           uint32_t *activity, cudaStream_t st);
cudaError_t launch_busy_count(const Dev &S, uint64_t t, uint32_t *out, cudaStream_t st);
cudaError_t launch_hash(const Dev &S, uint64_t t, unsigned long long *out, cudaStream_t st);

}  // namespace noc
