// tile_engine.cu -- host side of the TILED engine:
// tiling plan, launch attributes, launches, LL-slot refresh / reset kernels.
// The node-step kernel k_tiled (tile_kernel.cuh) is instantiated in
// tile_m0.cu / tile_m1.cu / tile_m2.cu.
#include "node_logic.cuh"
#include "kernels.h"
#include <cstdio>
#include <cstdlib>

namespace noc {

template <uint32_t MODE, bool DRAIN, uint32_t FEAT>
__global__ void k_tiled(const __grid_constant__ DevSet P, uint64_t t0, uint32_t ncyc, uint32_t smem_hist, uint32_t *activity);
#define NOC_TILED_EXTERN(M)                                                                                   \
    extern template __global__ void k_tiled<M, false, 0>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 0>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 1>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 1>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 2>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 2>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 3>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 3>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 4>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 4>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 5>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 5>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 6>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 6>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 7>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 7>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);  \
    extern template __global__ void k_tiled<M, false, 8>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *); \
    extern template __global__ void k_tiled<M, true, 8>(const __grid_constant__ DevSet, uint64_t, uint32_t, uint32_t, uint32_t *);
NOC_TILED_EXTERN(0)
NOC_TILED_EXTERN(1)
NOC_TILED_EXTERN(2)
#undef NOC_TILED_EXTERN

__device__ __forceinline__ unsigned long long llw(uint32_t stamp, uint32_t data)
{
    return ((unsigned long long)data << 32) | stamp;
}

// Before each launch at t0: every LL word that does not carry a live flit of
// cycle t0 gets stamp t0-1, which no poll of the next 2^32-1 cycles can
// mistake for its own (ABA guard for slots that stayed idle for long).
__global__ void k_ll_refresh(Dev S, uint64_t t0)
{
    const size_t total = (size_t)8u * S.nloc;    // (parity, slot, node)
    const uint32_t st0 = (uint32_t)t0, old = (uint32_t)(t0 - 1);
    const uint32_t b0 = (uint32_t)t0 & 1u;
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (size_t)gridDim.x * blockDim.x) {
        unsigned long long *w = S.ll + k * 4u;
        const uint32_t b = (uint32_t)(k / (4u * (size_t)S.nloc));
        const unsigned long long w0 = w[0];
        const bool live = b == b0 && (uint32_t)w0 == st0 && (uint32_t)(w0 >> 32) != LL_EMPTY;
        if (live) continue;
        if (b != b0 && (uint32_t)w0 != old) w[0] = llw(old, (uint32_t)(w0 >> 32));
        for (int j = 1; j < 4; ++j) w[j] = llw(old, (uint32_t)(w[j] >> 32));
    }
}

// Quiescent reset at cycle t (no flit anywhere): every LL slot of parity t&1
// holds EMPTY stamped t; used at create (t=0) and after a drain rewind.
__global__ void k_ll_reset(Dev S, uint64_t t)
{
    const size_t total = (size_t)4u * S.nloc;
    const uint32_t b = (uint32_t)t & 1u;
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (size_t)gridDim.x * blockDim.x) {
        unsigned long long *w = S.ll + ((size_t)b * 4u * S.nloc + k) * 4u;
        w[0] = llw((uint32_t)t, LL_EMPTY);
        for (int j = 1; j < 4; ++j) w[j] = llw((uint32_t)(t - 1), 0u);
    }
}

// ------------------------------------------------------------------ host side
size_t tiled_smem_bytes(const Dev &S, uint32_t np, bool with_hist)
{
    return (size_t)np * (8u * 16u + 6u * 4u) + 4u * NCOUNTERS + (with_hist ? 12u * (size_t)S.nb : 0u);
}

// Pick TX x TY tiles for one band (<= tiles_budget CTAs, <= TILE_BLOCK_MAX
// nodes each) minimising the largest tile, then its perimeter.  Host only.
bool tiled_plan(Dev &S, uint32_t tiles_budget, uint32_t *tiles, uint32_t *np)
{
    uint64_t best_tn = ~0ull, best_per = ~0ull;
    uint32_t bx = 0, by = 0;
    // a band that fits one CTA runs as ONE tile: no cross-tile exchange at all,
    // the cycle barrier is the only synchronisation (measured: a cycle with an
    // exchange costs 4-6x one without, whatever the tile size, DESIGN 6.4)
    const bool one = (uint64_t)S.W * S.rows <= TILE_BLOCK_MAX && !getenv("NOCSIM_TILING");
    if (one) { bx = by = 1; best_tn = (uint64_t)S.W * S.rows; }
    for (uint32_t tx = 1; !one && tx <= S.W && tx <= tiles_budget; ++tx) {
        for (uint32_t ty = 1; ty <= S.rows && (uint64_t)tx * ty <= tiles_budget; ++ty) {
            uint64_t tw = (S.W + tx - 1) / tx, th = (S.rows + ty - 1) / ty;
            uint64_t tn = tw * th, per = tw + th;
            if (tn < best_tn || (tn == best_tn && per < best_per)) { best_tn = tn; best_per = per; bx = tx; by = ty; }
        }
    }
    // experiment hook: NOCSIM_TILING=TXxTY forces the tiling when it fits
    if (const char *e = getenv("NOCSIM_TILING")) {
        unsigned ex = 0, ey = 0;
        if (sscanf(e, "%ux%u", &ex, &ey) == 2 && ex >= 1 && ey >= 1 && ex <= S.W && ey <= S.rows &&
            (uint64_t)ex * ey <= tiles_budget) {
            bx = ex;
            by = ey;
            best_tn = (uint64_t)((S.W + bx - 1) / bx) * ((S.rows + by - 1) / by);
        }
    }
    if (bx == 0 || best_tn > TILE_BLOCK_MAX) return false;
    S.TX = bx;
    S.TY = by;
    *tiles = bx * by;
    *np = (uint32_t)((best_tn + 31u) / 32u * 32u);
    // room for the ring warps of the largest tile (tile_kernel.cuh ring_map)
    const uint32_t tw = (S.W + bx - 1) / bx, th = (S.rows + by - 1) / by;
    // (one tile: only meshes of <= 64 nodes -- a 4x4 mesh in 4 warps instead of
    // one is 8 % faster, a 16x16 mesh in more warps slower)
    if (TILE_RING_CAP < 32u && (bx * by > 1u || tw * th <= 64u) && tw >= 3 && th >= 3) {
        const uint32_t ic = (tw - 2) * (th - 2), ring = tw * th - ic;
        const uint32_t npr = (ic + 31u) / 32u * 32u + 32u * ((ring + TILE_RING_CAP - 1u) / TILE_RING_CAP);
        if (npr > *np) *np = npr <= TILE_THREADS_MAX ? npr : TILE_THREADS_MAX / 32u * 32u;
    }
    return true;
}

// Shared-memory attribute and co-residency check for one launch of
// total_tiles CTAs of np threads.
// kernel mode: 0 UR, 1 LSPD (lean: NOC_LEAN), 2 LSPD with the private L1,
// migration, memory nodes or hub FIFOs (full); feat: FEAT bits
uint32_t tiled_kernel_mode(const Dev &D)
{
    if (D.mode != 1u) return D.mode;
    return (D.l1_sets || D.mig_hist || D.mem_mode || D.hub_cap) ? 2u : 1u;
}
static const void *tiled_fn(uint32_t mode, bool drain, uint32_t feat)
{
#define NOC_TD(M, F) (drain ? (const void *)k_tiled<M, true, F> : (const void *)k_tiled<M, false, F>)
#define NOC_TF4(M, B) (feat == 3u + B ? NOC_TD(M, 3 + B) : feat == 2u + B ? NOC_TD(M, 2 + B) : \
                       feat == 1u + B ? NOC_TD(M, 1 + B) : NOC_TD(M, 0 + B))
#define NOC_TF(M) (feat == 8u ? NOC_TD(M, 8) : feat >= 4u ? NOC_TF4(M, 4) : NOC_TF4(M, 0))
    return mode == 2u ? NOC_TF(2) : mode == 1u ? NOC_TF(1) : NOC_TF(0);
#undef NOC_TF
#undef NOC_TF4
#undef NOC_TD
}

cudaError_t tiled_prepare(uint32_t mode, uint32_t route, uint32_t nb, uint32_t np, uint32_t total_tiles, int device,
                          uint32_t *smem_hist)
{
    int sms = 0, optin = 0, smem_sm = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    if (e != cudaSuccess) return e;
    Dev tmp;
    tmp.nb = nb;
    bool with_hist = true;
    size_t smem = tiled_smem_bytes(tmp, np, true);
    if ((smem + 1024) * TILE_MIN_BLOCKS > (size_t)smem_sm || smem > (size_t)optin) {
        with_hist = false;
        smem = tiled_smem_bytes(tmp, np, false);
    }
    const void *fns[2] = {tiled_fn(mode, false, route), tiled_fn(mode, true, route)};
    for (const void *fn : fns) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)np, smem);
        if (e != cudaSuccess) return e;
        if ((uint64_t)per_sm * sms < total_tiles) return cudaErrorCooperativeLaunchTooLarge;
    }
    *smem_hist = with_hist ? 1u : 0u;
    return cudaSuccess;
}

// Cluster exchange (FEAT 8): one band of tiles <= TILE_CLUSTER_MAX launched as
// a single thread-block cluster (co-resident by construction)
cudaError_t tiled_prepare_cluster(uint32_t mode, uint32_t nb, uint32_t np, uint32_t tiles, uint32_t *smem_hist)
{
    if (tiles < 2 || tiles > TILE_CLUSTER_MAX) return cudaErrorInvalidConfiguration;
    Dev tmp;
    tmp.nb = nb;
    size_t smem = tiled_smem_bytes(tmp, np, true);
    *smem_hist = 1u;
    for (int drain = 0; drain < 2; ++drain) {
        const void *fn = tiled_fn(mode, drain != 0, 8u);
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = tiles;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(tiles);
        cfg.blockDim = dim3(np);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
        if (e != cudaSuccess) return e;
        if (nclusters < 1) return cudaErrorCooperativeLaunchTooLarge;
    }
    return cudaSuccess;
}

cudaError_t launch_ll_refresh(const Dev &S, uint64_t t0, cudaStream_t st)
{
    k_ll_refresh<<<256, 256, 0, st>>>(S, t0);
    return cudaGetLastError();
}

cudaError_t launch_tiled(const DevSet &P, uint64_t t0, uint32_t ncyc, uint32_t tpad, uint32_t smem_hist,
                         uint32_t *activity, cudaStream_t st)
{
    size_t smem = tiled_smem_bytes(P.d[0], tpad, smem_hist != 0);
    void *args[] = {(void *)&P, (void *)&t0, (void *)&ncyc, (void *)&smem_hist, (void *)&activity};
    const bool dr = activity != nullptr;
    const void *fn = tiled_fn(tiled_kernel_mode(P.d[0]), dr,
                              P.cluster ? 8u : P.d[0].route | (P.d[0].inject_mode ? 2u : 0u) | (P.general ? 4u : 0u));
    // the dynamic shared-memory limit is a per-function (process-wide)
    // attribute: another handle of a different size may have lowered it
    {
        const cudaError_t ea = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return ea;
    }
    if (P.cluster) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = P.cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(P.cluster);
        cfg.blockDim = dim3(tpad);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelExC(&cfg, fn, args);
    }
    return cudaLaunchCooperativeKernel(fn, dim3(P.tile0[P.nbands]), dim3(tpad), args, smem, st);
}

cudaError_t launch_ll_reset(const Dev &S, uint64_t t, cudaStream_t st)
{
    k_ll_reset<<<256, 256, 0, st>>>(S, t);
    return cudaGetLastError();
}

}  // namespace noc
