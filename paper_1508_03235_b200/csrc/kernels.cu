// kernels.cu -- the CUDA kernels of libnocsim.so (sm_100a) and their launch
// wrappers.  DESIGN.md section 6 describes the engines:
//   STEP    : one fused node-step launch per simulated cycle (all three phases
//             of the paper's loop, in ONE kernel);
//   PERSIST : one cooperative launch advances many cycles; each CTA owns a
//             contiguous range of nodes and, between cycles, waits only for the
//             CTAs whose nodes neighbour its own (neighbour-progress flags,
//             no grid-wide barrier, no host round trip).
#include "persist_kernel.cuh"

#include <cooperative_groups.h>

namespace noc {

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

// PERSIST kernel of a band: the full LSPD kernel (MODE 2) when the private L1,
// migration, memory nodes or hub FIFOs are on, else the lean UR / LSPD kernel
static const void *persist_fn(const Dev &S)
{
    if (S.mode == 1u && (S.l1_sets || S.mig_hist || S.mem_mode || S.hub_cap)) return (const void *)k_persist<2>;
    return persist_fn_lean(S.mode);
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
    const void *fn = persist_fn(S);
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
    const void *fn = persist_fn(P.d[0]);
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
