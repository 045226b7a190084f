// persist_kernel.cuh -- the PERSIST engine's kernel,
// instantiated in kernels.cu (full LSPD: MODE 2, with the private L1,
// migration, memory nodes and hub FIFOs) and in persist_lean.cu (UR and plain
// LSPD: MODE 0 / 1, compiled with NOC_LEAN, so those paths are compiled out of
// the node step -- as for the lean TILED kernels, tile_m0.cu / tile_m1.cu).
#pragma once
#include "node_logic.cuh"
#include "kernels.h"

namespace noc {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Flush per-thread register accumulators: warp reduce, then one atomic per warp.
__device__ __forceinline__ void flush_acc(const Dev &S, const Acc &a, unsigned int *scnt)
{
    uint32_t v[4] = {a.injected, a.ejected, a.hops, a.defl};
    const uint32_t idx[4] = {C_INJECTED, C_EJECTED, C_HOPS, C_DEFL};
    unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t s = __reduce_add_sync(0xFFFFFFFFu, v[i]);
        if (lane == 0 && s) {
            if (scnt) atomicAdd(&scnt[idx[i]], s);
            else atomicAdd(&S.cnt[idx[i]], (unsigned long long)s);
        }
    }
}

// ------------------------------------------------------------------ PERSIST engine
// One cooperative launch for all row bands of this process (DevSet; band k
// owns CTAs [tile0[k], tile0[k+1])).  Each CTA owns S.npc consecutive nodes of
// its band and, before each cycle, waits for the CTAs whose nodes lie within
// one row of its own: in its band (from the second cycle of the launch on) and,
// at a band edge, in the neighbouring band (from the first cycle on, since
// that band may still be finishing its previous launch; system scope, since it
// may be another GPU).  Progress counters count completed cycles (pbase + c + 1).
// Dynamic shared memory: NCOUNTERS u32 counters, then (optionally) 3*nb u32 bins.
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <uint32_t MODE>
__global__ void __launch_bounds__(PERSIST_BLOCK, PERSIST_MIN_BLOCKS) k_persist(const __grid_constant__ DevSet P, uint64_t t0, uint32_t ncyc,
                                                         uint32_t pbase, uint32_t smem_hist, uint32_t *activity)
{
    uint32_t band = 0;
    while (band + 1 < P.nbands && blockIdx.x >= P.tile0[band + 1]) ++band;
    __shared__ Dev sD;   // this band's parameters (read every cycle; see tile_engine.cu)
    for (uint32_t k = threadIdx.x; k < sizeof(Dev) / 4; k += blockDim.x)
        reinterpret_cast<uint32_t *>(&sD)[k] = reinterpret_cast<const uint32_t *>(&P.d[band])[k];
    extern __shared__ unsigned int sm[];
    unsigned int *scnt = sm;
    unsigned int *shist = smem_hist ? sm + NCOUNTERS : nullptr;
    __syncthreads();
    const Dev &S = sD;
    const uint32_t nsm = NCOUNTERS + (smem_hist ? 3u * S.nb : 0u);
    for (uint32_t i = threadIdx.x; i < nsm; i += blockDim.x) sm[i] = 0u;

    const uint32_t G = P.tile0[band + 1] - P.tile0[band], b = blockIdx.x - P.tile0[band];
    const uint32_t npc = S.npc;
    uint32_t *const progress = S.progress;
    const uint32_t lo_node = b * npc;
    const uint32_t hi_node = min(S.nloc, lo_node + npc);
    // CTAs of this band owning nodes within one row (W) of ours: they feed our input links
    const uint32_t first = lo_node >= S.W ? (lo_node - S.W) / npc : 0u;
    const uint32_t lastn = min(S.nloc - 1u, hi_node - 1u + S.W);
    const uint32_t last = min(G - 1u, lastn / npc);
    // neighbour bands: the CTAs owning the north band's last row / the south band's first row
    const bool north = lo_node < S.W && S.prog_nb[0] != nullptr;
    const bool south = hi_node + S.W > S.nloc && S.prog_nb[1] != nullptr;
    const uint32_t n_first = north ? (S.nloc_nb[0] - S.W) / S.npc_nb[0] : 0u;
    const uint32_t n_last = north ? (S.nloc_nb[0] - 1u) / S.npc_nb[0] : 0u;
    const uint32_t s_last = south ? (S.W - 1u) / S.npc_nb[1] : 0u;
    Sink K{scnt, shist, true};
    Acc acc = {0, 0, 0, 0};
    __shared__ int s_abort;
    __shared__ uint32_t s_busy[2];
    if (threadIdx.x == 0) { s_abort = 0; s_busy[0] = s_busy[1] = 0u; }
    __syncthreads();

    auto wait_for = [&](const uint32_t *prog, uint32_t j, uint32_t target, bool sys) {
        uint32_t spins = 0;
        while ((int32_t)((sys ? ld_acquire_sys_u32(&prog[j]) : ld_acquire_u32(&prog[j])) - target) < 0) {
            if (++spins > (1u << 24)) {   // a hung neighbour: abort the launch, report
                atomicOr(S.err, 0x80000000u);
                s_abort = 1;
                break;
            }
            __nanosleep(64);   // leave the issue slots to the co-resident CTAs that compute (C5: -1.2 %)
        }
    };
    for (uint32_t c = 0; c < ncyc; ++c) {
        const uint64_t t = t0 + c;
        const uint32_t target = pbase + c;
        // wait until every neighbouring CTA completed cycle t-1
        if (c > 0)
            for (uint32_t j = first + threadIdx.x; j <= last; j += blockDim.x)
                if (j != b) wait_for(progress, j, target, false);
        if (north)
            for (uint32_t j = n_first + threadIdx.x; j <= n_last; j += blockDim.x) wait_for(S.prog_nb[0], j, target, true);
        if (south)
            for (uint32_t j = threadIdx.x; j <= s_last; j += blockDim.x) wait_for(S.prog_nb[1], j, target, true);
        __syncthreads();
        if (s_abort) break;
        bool busy = false;
        // the words every node step reads first (occupancy, FIFO control, core
        // state) are prefetched one node ahead: each thread walks several
        // nodes per cycle, and at 1M nodes they come from DRAM
        for (uint32_t l = lo_node + threadIdx.x; l < hi_node; l += blockDim.x) {
#ifndef NOC_NO_PERSIST_PREFETCH
            const uint32_t ln = l + blockDim.x;
#if defined(NOC_AB_PF4) || defined(NOC_AB_PF2)
            if (ln < hi_node) {
                const uint32_t pb = (uint32_t)t & 1u;
#pragma unroll
                for (uint32_t d = 0; d < 4; ++d) prefetch_l1(&S.flit[pb][flit_at(S.nloc, d, ln)]);
            }
#endif
#ifdef NOC_AB_PF2
            const uint32_t ln2 = ln + blockDim.x;
            if (ln2 < hi_node) {
                prefetch_l1(&S.flag[(uint32_t)t & 1u][ln2]);
                prefetch_l1(&S.fifo_ctl[ln2]);
                if (MODE != 0u) prefetch_l1(&S.core_hot[ln2]);
            }
            if (l == lo_node + threadIdx.x && ln < hi_node) {
                prefetch_l1(&S.flag[(uint32_t)t & 1u][ln]);
                prefetch_l1(&S.fifo_ctl[ln]);
                if (MODE != 0u) prefetch_l1(&S.core_hot[ln]);
            }
#else
            if (ln < hi_node) {
                prefetch_l1(&S.flag[(uint32_t)t & 1u][ln]);
                prefetch_l1(&S.fifo_ctl[ln]);
                if (MODE != 0u) prefetch_l1(&S.core_hot[ln]);
            }
#endif
#endif
            busy |= node_step_global<(MODE == 2u ? 1u : MODE)>(S, K, l, t, acc);
        }
        // full BAR.SYNC (see tile_engine.cu); busy nodes stamp a per-parity word
        if (activity && busy) s_busy[c & 1u] = c + 1u;
        __syncthreads();
        if (threadIdx.x == 0) {
            if (activity && s_busy[c & 1u] == c + 1u) atomicAdd(&activity[c], 1u);
            if (north || south) {   // links written into another band (GPU): system scope
                __threadfence_system();
                st_release_sys_u32(&progress[b], pbase + c + 1u);
            } else {
                __threadfence();
                st_release_u32(&progress[b], pbase + c + 1u);
            }
        }
    }
    flush_acc(S, acc, scnt);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < NCOUNTERS; i += blockDim.x)
        if (scnt[i]) atomicAdd(&S.cnt[i], (unsigned long long)scnt[i]);
    if (smem_hist)
        for (uint32_t i = threadIdx.x; i < 3u * S.nb; i += blockDim.x)
            if (shist[i]) atomicAdd(&S.hist[i], (unsigned long long)shist[i]);
}

}  // namespace noc
