// kernels.cu -- the CUDA kernels of libnocsim.so (sm_100a) and their launch
// wrappers.  DESIGN.md section 6 describes the engines:
//   STEP    : one fused node-step launch per simulated cycle (all three phases
//             of the paper's loop, in ONE kernel);
//   PERSIST : one cooperative launch advances many cycles; each CTA owns a
//             contiguous range of nodes and, between cycles, waits only for the
//             CTAs whose nodes neighbour its own (neighbour-progress flags,
//             no grid-wide barrier, no host round trip).
#include "node_logic.cuh"
#include "kernels.h"

#include <cooperative_groups.h>

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

// ------------------------------------------------------------------ STEP engine
template <uint32_t MODE>
__global__ void __launch_bounds__(256) k_step(Dev S, uint64_t t, uint32_t *activity)
{
    uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    Acc acc = {0, 0, 0, 0};
    Sink K{nullptr, nullptr, true};
    bool busy = false;
    if (l < S.nloc) busy = node_step_global<MODE>(S, K, l, t, acc);
    flush_acc(S, acc, nullptr);
    if (activity) {
        if (__syncthreads_or(busy) && threadIdx.x == 0) atomicAdd(activity, 1u);
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
                if (MODE == 1u) prefetch_l1(&S.core_hot[ln2]);
            }
            if (l == lo_node + threadIdx.x && ln < hi_node) {
                prefetch_l1(&S.flag[(uint32_t)t & 1u][ln]);
                prefetch_l1(&S.fifo_ctl[ln]);
                if (MODE == 1u) prefetch_l1(&S.core_hot[ln]);
            }
#else
            if (ln < hi_node) {
                prefetch_l1(&S.flag[(uint32_t)t & 1u][ln]);
                prefetch_l1(&S.fifo_ctl[ln]);
                if (MODE == 1u) prefetch_l1(&S.core_hot[ln]);
            }
#endif
#endif
            busy |= node_step_global<MODE>(S, K, l, t, acc);
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

// ------------------------------------------------------------------ link state between launches
// Input slot d of local node l at the boundary before cycle t: a flit, or none.
// Tile-crossing links of the TILED engine live in LL slots, all others in the
// flag/flit arrays.
__device__ bool read_slot(const Dev &S, uint32_t l, uint32_t d, uint64_t t, Flit &f)
{
    const uint32_t n = S.n0 + l, y = n / S.W, x = n - y * S.W;
    const uint32_t b = (uint32_t)t & 1u;
    if (slot_external(S, x, y, d)) {
        unsigned long long w0 = S.ll[ll_index(S, b, d, l, 0)];
        if ((uint32_t)w0 != (uint32_t)t || (uint32_t)(w0 >> 32) == LL_EMPTY) return false;
        f.x = (uint32_t)(w0 >> 32);
        f.y = (uint32_t)(S.ll[ll_index(S, b, d, l, 1)] >> 32);
        f.z = (uint32_t)(S.ll[ll_index(S, b, d, l, 2)] >> 32);
        f.w = (uint32_t)(S.ll[ll_index(S, b, d, l, 3)] >> 32);
        return true;
    }
    uint32_t fl = S.flag[b][l];
    if (((fl >> (8u * d)) & 0xFFu) != stamp_of(t)) return false;
    uint4 v = S.flit[b][flit_at(S.nloc, d, l)];
    f = Flit{v.x, v.y, v.z, v.w};
    return true;
}

// ------------------------------------------------------------------ streamed scripts (R57)
// Per node: events still to come = the old queue minus the consumed ones,
// then the pushed ones (add_off / add_ev: this band's pushed events by node).
__global__ void k_script_count(Dev S, const uint32_t *add_off, uint32_t *cnt)
{
    const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= S.nloc) return;
    const uint32_t base = S.script_base ? S.script_base[l] : 0u;
    const uint32_t rem = S.script_off[l + 1] - S.script_off[l] - (S.script_pos[l] - base);
    cnt[l] = rem + add_off[l + 1] - add_off[l];
}

__global__ void k_script_merge(Dev S, const uint32_t *add_off, const uint4 *add_ev, const uint32_t *new_off,
                               uint4 *new_ev, uint32_t *new_base)
{
    const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= S.nloc) return;
    const uint32_t pos = S.script_pos[l], base = S.script_base ? S.script_base[l] : 0u;
    uint32_t k = new_off[l];
    for (uint32_t i = S.script_off[l] + pos - base; i < S.script_off[l + 1]; ++i) new_ev[k++] = S.script[i];
    for (uint32_t i = add_off[l]; i < add_off[l + 1]; ++i) new_ev[k++] = add_ev[i];
    new_base[l] = pos;
}

cudaError_t launch_script_count(const Dev &S, const uint32_t *add_off, uint32_t *cnt, cudaStream_t st)
{
    k_script_count<<<(S.nloc + 255) / 256, 256, 0, st>>>(S, add_off, cnt);
    return cudaGetLastError();
}

cudaError_t launch_script_merge(const Dev &S, const uint32_t *add_off, const uint4 *add_ev, const uint32_t *new_off,
                                uint4 *new_ev, uint32_t *new_base, cudaStream_t st)
{
    k_script_merge<<<(S.nloc + 255) / 256, 256, 0, st>>>(S, add_off, add_ev, new_off, new_ev, new_base);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ drain helper
__global__ void k_busy_count(Dev S, uint64_t t, uint32_t *out)
{
    uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    bool busy = false;
    if (l < S.nloc) {
        Flit f;
        for (uint32_t d = 0; d < 4; ++d) busy |= read_slot(S, l, d, t, f);
        busy |= q_count(S.fifo_ctl[l]) > 0;
        if (S.mode == 1u) busy |= core_mode(S.core_hot[l]) != MIDLE;
    }
    if (__syncthreads_or(busy) && threadIdx.x == 0) atomicAdd(out, 1u);
}

// ------------------------------------------------------------------ state hash
// Node-owned terms (LINK, FIFO, FIFONEXT, CORE, L2, SCRIPT) of DESIGN 3.7.
__global__ void k_hash_nodes(Dev S, uint64_t t, unsigned long long *out)
{
    uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t H = 0;
    if (l < S.nloc) {
        const uint64_t n = S.n0 + l;
        for (uint32_t d = 0; d < 4; ++d) {
            Flit f;
            if (!read_slot(S, l, d, t, f)) continue;
            uint64_t life = (uint32_t)((uint32_t)t - f.z);
            uint64_t inj = t - life;
            TupleHash th(7);
            th.add(f_dst(f)).add(f_src(f)).add(f_kind(f)).add(f_fid(f)).add(f.w).add(f_age(f)).add(inj);
            H += hterm(D_LINK, n * 4 + d, th.h);
        }
        uint32_t q = S.fifo_ctl[l];
        for (uint32_t k = 0; k < q_count(q); ++k) {
            const FifoRef F = fifo_of(S, l);
            uint2 p = F.p[(q_head(q) + k) & (F.cap - 1u)];
            TupleHash th(4);
            th.add((p.x >> 21) & 7u).add(p.x & NODE_MASK).add(p.y).add((p.x >> 24) & 15u);
            H += hterm(D_FIFO, (n << 16) + k, th.h);
        }
        if (q_next(q)) H += hterm(D_FIFONEXT, n, TupleHash(1).add(q_next(q)).h);
        if (S.mode == 1u) {
            uint32_t hot = S.core_hot[l];
            uint32_t mode = core_mode(hot);
            if (mode != MIDLE) {
                uint4 cold = S.core_cold[l];
                uint64_t ready = 0, tag = 0, inst = 0, rx = 0;
                uint64_t start = ((uint64_t)cold.y << 32) | cold.x;
                uint64_t r29 = t + (uint64_t)((hot - (uint32_t)t) & 0x1FFFFFFFu);
                switch (mode) {
                case ML2WAIT: ready = r29; break;
                case ML1WAIT: ready = r29; tag = cold.z; break;
                case MWAITDIR: tag = cold.z; break;
                case MWAITDATA: tag = cold.z; rx = cold.w >> 2; break;
                case MMEMFETCH: tag = cold.z; inst = cold.w & 3u; rx = cold.w >> 2; break;
                default: ready = r29; tag = cold.z; inst = cold.w & 3u; break;
                }
                TupleHash th(6);
                th.add(mode).add(ready).add(tag).add(inst).add(start).add(rx);
                H += hterm(D_CORE, n, th.h);
            }
            const uint4 *L = S.l2 + (size_t)l * S.sets * S.ways;
            for (uint32_t i = 0; i < S.sets * S.ways; ++i) {
                uint4 v = L[i];
                if (S.mig_hist) {
                    // NEXT-f2: (state, tag, target, history count, history oldest first)
                    const uint32_t st = lw_state(v.w), cnt = lw_count(v.w);
                    if (st != MS_NORMAL || (line_valid(v) && cnt)) {
                        const size_t li = (size_t)l * S.sets * S.ways + i;
                        const uint32_t N = S.mig_hist, head = lw_head(v.w);
                        TupleHash th(4 + (int)cnt);
                        th.add(st).add(v.x ? v.x - 1u : 0u).add(lw_target(v.w)).add(cnt);
                        for (uint32_t k = 0; k < cnt; ++k) th.add(S.l2h[li * N + (head + k) % N]);
                        H += hterm(D_L2MIG, (n * S.sets) * S.ways + i, th.h);
                    }
                }
                if (!line_valid(v)) continue;
                uint64_t stamp = ((uint64_t)v.z << 32) | v.y;
                H += hterm(D_L2, (n * S.sets) * S.ways + i, TupleHash(2).add(v.x - 1u).add(stamp).h);
            }
            if (S.mig_hist)
                for (uint32_t k = 0; k < 4u; ++k) {
                    const uint2 x = S.migrx[(size_t)l * 4u + k];
                    if (x.y) H += hterm(D_MIGRX, (n << 2) + k, TupleHash(2).add(x.x).add(x.y).h);
                }
            if (S.l1_sets) {   // NEXT-f1 L1 lines: (tag, stamp, owner)
                const uint4 *M = S.l1 + (size_t)l * S.l1_sets * S.l1_ways;
                for (uint32_t i = 0; i < S.l1_sets * S.l1_ways; ++i) {
                    uint4 v = M[i];
                    if (v.x == 0u) continue;
                    uint64_t stamp = ((uint64_t)v.z << 32) | v.y;
                    H += hterm(D_L1, (n * S.l1_sets) * S.l1_ways + i, TupleHash(3).add(v.x - 1u).add(stamp).add(v.w).h);
                }
            }
        }
        if (S.has_script) {
            uint32_t pos = S.script_pos[l];
            if (pos) H += hterm(D_SCRIPT, n, TupleHash(1).add(pos).h);
        }
    }
    // block reduction of a u64 sum (mod 2^64)
    __shared__ unsigned long long red[32];
    unsigned long long v = H;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (threadIdx.x == 0) atomicAdd(out, v);
    }
}

// LOC terms: entries loc[q][lh] != 0, tag T = q*N + n0 + lh.
__global__ void k_hash_loc(Dev S, unsigned long long *out)
{
    uint64_t H = 0;
    const uint64_t total = S.loc_n;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t e = S.loc[i];
        const uint32_t m = S.mig_hist ? S.loc_mig[i] : 0u;
        if (!e && !m) continue;
        uint64_t T = i;   // centralized: the entry index is the tag
        if (!S.dir_mode) {
            const uint64_t q = i / S.nloc, lh = i - q * S.nloc;
            T = q * S.N + S.n0 + lh;
        }
        if (m) H += hterm(D_LOCMIG, T, TupleHash(2).add(m & 1u).add((m >> 1) & 1u).h);   // NEXT-f2
        if (e) H += hterm(D_LOC, T, TupleHash(2).add(e & HOLDER_MASK).add(e >> HOLDER_BITS).h);
    }
    __shared__ unsigned long long red[32];
    unsigned long long v = H;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (threadIdx.x == 0) atomicAdd(out, v);
    }
}

// ------------------------------------------------------------------ launch wrappers
cudaError_t launch_step(const Dev &S, uint64_t t, uint32_t *activity, cudaStream_t st)
{
    uint32_t grid = (S.nloc + 255u) / 256u;
    if (S.mode == 1u) k_step<1><<<grid, 256, 0, st>>>(S, t, activity);
    else k_step<0><<<grid, 256, 0, st>>>(S, t, activity);
    return cudaGetLastError();
}

size_t persist_smem_bytes(const Dev &S, bool with_hist)
{
    return sizeof(unsigned int) * (NCOUNTERS + (with_hist ? 3u * S.nb : 0u));
}

// Nodes per CTA and grid for one band with at most max_ctas co-resident CTAs
// (the whole device divided among the process's bands).
cudaError_t persist_configure(const Dev &S, int device, uint32_t nbands, uint32_t *grid, uint32_t *nodes_per_cta,
                              uint32_t *smem_hist)
{
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    bool with_hist = 3u * S.nb * 4u <= 64u * 1024u;
    size_t smem = persist_smem_bytes(S, with_hist);
    const void *fn = S.mode == 1u ? (const void *)k_persist<1> : (const void *)k_persist<0>;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, PERSIST_BLOCK, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    uint64_t max_ctas = (uint64_t)sms * (uint64_t)per_sm / (nbands ? nbands : 1u);
    if (max_ctas < 1) return cudaErrorInvalidConfiguration;
    uint32_t npc = PERSIST_BLOCK;                     // one node per thread when possible
    uint64_t g = (S.nloc + npc - 1u) / npc;
    if (g > max_ctas) {
        npc = (uint32_t)((S.nloc + max_ctas - 1u) / max_ctas);
        g = (S.nloc + npc - 1u) / npc;
    }
    *grid = (uint32_t)g;
    *nodes_per_cta = npc;
    *smem_hist = with_hist ? 1u : 0u;
    return cudaSuccess;
}

cudaError_t launch_persist(const DevSet &P, uint64_t t0, uint32_t ncyc, uint32_t pbase, uint32_t smem_hist,
                           uint32_t *activity, cudaStream_t st)
{
    size_t smem = persist_smem_bytes(P.d[0], smem_hist != 0);
    void *args[] = {(void *)&P, (void *)&t0, (void *)&ncyc, (void *)&pbase, (void *)&smem_hist, (void *)&activity};
    const void *fn = P.d[0].mode == 1u ? (const void *)k_persist<1> : (const void *)k_persist<0>;
    // the dynamic shared-memory limit is a per-function (process-wide)
    // attribute: another handle of a different size may have lowered it
    {
        const cudaError_t ea = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return ea;
    }
    return cudaLaunchCooperativeKernel(fn, dim3(P.tile0[P.nbands]), dim3(PERSIST_BLOCK), args, smem, st);
}

cudaError_t launch_busy_count(const Dev &S, uint64_t t, uint32_t *out, cudaStream_t st)
{
    uint32_t grid = (S.nloc + 255u) / 256u;
    k_busy_count<<<grid, 256, 0, st>>>(S, t, out);
    return cudaGetLastError();
}

cudaError_t launch_hash(const Dev &S, uint64_t t, unsigned long long *out, cudaStream_t st)
{
    uint32_t grid = (S.nloc + 255u) / 256u;
    k_hash_nodes<<<grid, 256, 0, st>>>(S, t, out);
    if (S.mode == 1u) k_hash_loc<<<1024, 256, 0, st>>>(S, out);
    return cudaGetLastError();
}

}  // namespace noc
