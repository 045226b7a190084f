// tile_engine.cu -- the TILED engine.
//
// One persistent CTA per rectangular tile of the mesh (one CTA per SM), one
// thread per node, many cycles per launch:
//   * every node's core / FIFO-control / script state lives in REGISTERS of
//     its thread for the whole launch (no per-cycle HBM/L2 round trip);
//   * links between nodes of the same tile live in SHARED memory, double
//     buffered by cycle parity, occupancy bytes cleared on read;
//   * links that cross a tile boundary are "LL" slots in global memory: the
//     sender writes 64-bit words that carry (cycle stamp, 32 data bits), so the
//     receiver polls the data itself -- no fence, no flag, no grid barrier.
//     Every boundary output port is written every cycle (a flit or EMPTY), and
//     each cross-tile link pairs with its reverse link, so a receiver can never
//     be overrun by more than one cycle (DESIGN 6.3 proof sketch);
//   * the per-node service of an ejected flit (directory / L2 lookups, Fig. 4
//     P:L219) is deferred to the start of the next cycle, after the tile
//     barrier, so its global-memory latency overlaps the boundary exchange;
//     it still precedes the node's next Phase 1 and injection, so the order of
//     DESIGN 3.3 (R27) is unchanged.
// The model is exactly node_logic.cuh's (bit-identical to every other engine).
#include "node_logic.cuh"
#include "kernels.h"

namespace noc {

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long llw(uint32_t stamp, uint32_t data)
{
    return ((unsigned long long)data << 32) | stamp;
}

// a[p] for a runtime p without indexing a local array (keeps a[] in registers)
__device__ __forceinline__ uint32_t pick4(const uint32_t (&a)[4], uint32_t p)
{
    return p == 0u ? a[0] : p == 1u ? a[1] : p == 2u ? a[2] : a[3];
}

struct TileShape {
    uint32_t x0, y0, tw, th, tn;
};

__device__ __forceinline__ TileShape tile_shape(const Dev &S, uint32_t b)
{
    const uint32_t tx = b % S.TX, ty = b / S.TX;
    TileShape T;
    T.x0 = (uint32_t)((uint64_t)tx * S.W / S.TX);
    const uint32_t x1 = (uint32_t)((uint64_t)(tx + 1) * S.W / S.TX);
    const uint32_t ly0 = (uint32_t)((uint64_t)ty * S.rows / S.TY);
    const uint32_t ly1 = (uint32_t)((uint64_t)(ty + 1) * S.rows / S.TY);
    T.y0 = S.row0 + ly0;
    T.tw = x1 - T.x0;
    T.th = ly1 - ly0;
    T.tn = T.tw * T.th;
    return T;
}

// Dynamic shared memory layout (tpad = threads per CTA):
//   uint4    sflit[2][4][tpad]
//   uint32_t sflag[2][tpad]
//   uint32_t scnt[NCOUNTERS]
//   uint32_t shist[3][nb]        (optional)
template <uint32_t MODE>
__global__ void __launch_bounds__(TILE_MAX_THREADS, 1)
k_tiled(Dev S, uint64_t t0, uint32_t ncyc, uint32_t smem_hist, uint32_t *activity)
{
    extern __shared__ uint4 smem4[];
    const uint32_t tpad = blockDim.x;
    uint4 *sflit = smem4;                                        // [2][4][tpad]
    uint32_t *sflag = reinterpret_cast<uint32_t *>(sflit + 8u * tpad);  // [2][tpad]
    unsigned int *scnt = sflag + 2u * tpad;
    unsigned int *shist = smem_hist ? scnt + NCOUNTERS : nullptr;
    __shared__ int s_abort;
    __shared__ uint32_t s_busy[2];

    const uint32_t i = threadIdx.x;
    const TileShape T = tile_shape(S, blockIdx.x);
    const bool active = i < T.tn;

    {
        const uint32_t nsm = NCOUNTERS + (smem_hist ? 3u * S.nb : 0u);
        for (uint32_t k = i; k < nsm; k += blockDim.x) scnt[k] = 0u;
        if (i == 0) { s_abort = 0; s_busy[0] = s_busy[1] = 0u; }
    }

    // ---- node registers (persist for the whole launch)
    NodeCtx c;
    const uint32_t lx = active ? i % T.tw : 0u, lyy = active ? i / T.tw : 0u;
    c.x = T.x0 + lx;
    c.y = T.y0 + lyy;
    c.n = c.y * S.W + c.x;
    c.l = c.n - S.n0;
    c.head_ok = false;
    c.cold_loaded = true;
    c.q_dirty = c.hot_dirty = c.cold_dirty = false;
    c.busy_flit = false;
    uint32_t ext = 0;      // bit d: input/output port d crosses the tile boundary
    uint32_t exist = 0;    // bit d: port d exists
    if (active) {
        c.qctl = S.fifo_ctl[c.l];
        if (MODE == 1u) {
            c.hot = S.core_hot[c.l];
            c.cold = S.core_cold[c.l];
        } else {
            c.hot = 0u;
            c.cold = make_uint4(0, 0, 0, 0);
        }
        if (q_count(c.qctl)) { c.head = S.fifo_pkt[(size_t)c.l * S.qcap + q_head(c.qctl)]; c.head_ok = true; }
        exist = (c.y > 0 ? 1u : 0u) | (c.y + 1 < S.H ? 2u : 0u) | (c.x + 1 < S.W ? 4u : 0u) | (c.x > 0 ? 8u : 0u);
        ext = (lyy == 0 ? 1u : 0u) | (lyy + 1 == T.th ? 2u : 0u) | (lx + 1 == T.tw ? 4u : 0u) | (lx == 0 ? 8u : 0u);
        ext &= exist;
        // internal inputs of cycle t0 (spilled by the previous launch)
        const uint32_t b0 = (uint32_t)t0 & 1u;
        uint32_t fl = S.flag[b0][c.l];
        uint32_t sfl = 0;
        const uint8_t st0 = stamp_of(t0);
        for (uint32_t d = 0; d < 4; ++d) {
            if (!((ext >> d) & 1u) && ((fl >> (8u * d)) & 0xFFu) == st0) {
                sflit[(b0 * 4u + d) * tpad + i] = S.flit[b0][(size_t)d * S.nloc + c.l];
                sfl |= (uint32_t)st0 << (8u * d);
            }
        }
        sflag[b0 * tpad + i] = sfl;
        sflag[(b0 ^ 1u) * tpad + i] = 0u;
    }
    __syncthreads();

    // LL word offsets (parity 0) of this node's boundary input slots and of the
    // neighbours' slots its boundary output ports feed; parity 1 adds pstride
    const uint32_t pstride = 16u * S.nloc;
    uint32_t inw[4], outw[4], outi[4];
#pragma unroll
    for (uint32_t d = 0; d < 4; ++d) {
        inw[d] = (uint32_t)ll_index(S, 0, d, c.l, 0);
        uint32_t m = c.l, mi = i;
        switch (d) {
        case PN: m = c.l - S.W; mi = i - T.tw; break;
        case PS: m = c.l + S.W; mi = i + T.tw; break;
        case PE: m = c.l + 1u; mi = i + 1u; break;
        default: m = c.l - 1u; mi = i - 1u; break;
        }
        outw[d] = ((ext >> d) & 1u) ? (uint32_t)ll_index(S, 0, d ^ 1u, m, 0) : 0u;
        outi[d] = mi;
    }

    Sink K{scnt, shist};
    Acc acc = {0, 0, 0, 0};
    Flit pend;
    bool has_pend = false;

    for (uint32_t cc = 0; cc < ncyc; ++cc) {
        const uint64_t t = t0 + cc;
        const uint32_t pb = (uint32_t)t & 1u, nb1 = pb ^ 1u;
        const uint32_t st32 = (uint32_t)t, st32n = (uint32_t)(t + 1);
        bool busy = false;
        if (active) {
            // issue the boundary polls first: their latency overlaps the
            // deferred service and Phase 1
            unsigned long long xw[4] = {0, 0, 0, 0};
            unsigned long long *const llp = S.ll + (size_t)pb * pstride;     // this cycle's inputs
            unsigned long long *const lln = S.ll + (size_t)nb1 * pstride;    // next cycle's inputs
#pragma unroll
            for (uint32_t d = 0; d < 4; ++d)
                if ((ext >> d) & 1u) xw[d] = ld_relaxed_u64(llp + inw[d]);

            // deferred Phase 3 of cycle t-1
            if (has_pend) { phase3(S, K, c, pend, t - 1, acc); has_pend = false; }

            // Phase 1
            if (MODE == 0u) phase1_ur(S, K, c, t);
            else phase1_lspd(S, K, c, t);

            // Phase 2: latch internal inputs from shared memory ...
            Inputs in;
            in.present = 0;
            const uint32_t fl = sflag[pb * tpad + i];
            if (fl) sflag[pb * tpad + i] = 0u;
            const uint8_t st = stamp_of(t);
#pragma unroll
            for (uint32_t d = 0; d < 4; ++d) {
                if (((fl >> (8u * d)) & 0xFFu) == st) {
                    uint4 v = sflit[(pb * 4u + d) * tpad + i];
                    in.f[d] = Flit{v.x, v.y, v.z, v.w};
                    in.present |= 1u << d;
                }
            }
            // ... and boundary inputs from the LL slots (spin on the stamp)
#pragma unroll
            for (uint32_t d = 0; d < 4; ++d) {
                if (!((ext >> d) & 1u)) continue;
                const unsigned long long *slot = llp + inw[d];
                uint32_t spins = 0;
                unsigned long long w = xw[d];
                while ((uint32_t)w != st32) {
                    if (++spins > (1u << 22)) { atomicOr(S.err, 0x80000000u); s_abort = 1; break; }
                    w = ld_relaxed_u64(slot);
                }
                const uint32_t x = (uint32_t)(w >> 32);
                if ((uint32_t)w == st32 && x != LL_EMPTY) {
                    unsigned long long w1 = ld_relaxed_u64(slot + 1), w2 = ld_relaxed_u64(slot + 2),
                                       w3 = ld_relaxed_u64(slot + 3);
                    while (((uint32_t)w1 != st32 || (uint32_t)w2 != st32 || (uint32_t)w3 != st32) && !s_abort) {
                        if (++spins > (1u << 22)) { atomicOr(S.err, 0x80000000u); s_abort = 1; break; }
                        if ((uint32_t)w1 != st32) w1 = ld_relaxed_u64(slot + 1);
                        if ((uint32_t)w2 != st32) w2 = ld_relaxed_u64(slot + 2);
                        if ((uint32_t)w3 != st32) w3 = ld_relaxed_u64(slot + 3);
                    }
                    in.f[d] = Flit{x, (uint32_t)(w1 >> 32), (uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32)};
                    in.present |= 1u << d;
                }
            }

            inject(S, c, in, t, acc);
            Flit ej;
            bool has_ej = false;
            uint32_t used = 0;
            if (in.present) {
                const uint8_t st1 = stamp_of(t + 1);
                used = route(S, c, in, t, acc, ej, has_ej, [&](uint32_t p, const Flit &f) {
                    const uint32_t slot = p ^ 1u;   // opp(p): N<->S (0,1), E<->W (2,3)
                    if ((ext >> p) & 1u) {
                        unsigned long long *o = lln + pick4(outw, p);
                        st_relaxed_u64(o + 1, llw(st32n, f.y));
                        st_relaxed_u64(o + 2, llw(st32n, f.z));
                        st_relaxed_u64(o + 3, llw(st32n, f.w));
                        st_relaxed_u64(o, llw(st32n, f.x));
                    } else {
                        const uint32_t mi = pick4(outi, p);
                        sflit[(nb1 * 4u + slot) * tpad + mi] = make_uint4(f.x, f.y, f.z, f.w);
                        reinterpret_cast<uint8_t *>(sflag + nb1 * tpad + mi)[slot] = st1;
                    }
                });
            }
            // boundary ports without a flit carry an explicit EMPTY every cycle
            const uint32_t idle_ext = ext & ~used;
#pragma unroll
            for (uint32_t p = 0; p < 4; ++p)
                if ((idle_ext >> p) & 1u) st_relaxed_u64(lln + outw[p], llw(st32n, LL_EMPTY));
            if (has_ej) {
                // while draining, quiescence is judged at the end of each cycle,
                // so the service is not deferred there
                if (activity) phase3(S, K, c, ej, t, acc);
                else { pend = ej; has_pend = true; }
            }
            busy = used != 0u || has_pend || q_count(c.qctl) > 0u || core_mode(c.hot) != MIDLE;
        }
        // The cycle barrier must be a full BAR.SYNC: it orders the shared-memory
        // link stores of this cycle before next cycle's loads.  (A reducing
        // barrier, __syncthreads_or, measurably did not on sm_100a.)  Busy
        // nodes instead stamp a per-parity shared word with the cycle index.
        if (activity && busy) s_busy[cc & 1u] = cc + 1u;
        __syncthreads();
        if (activity && i == 0 && s_busy[cc & 1u] == cc + 1u) atomicAdd(&activity[cc], 1u);
        if (s_abort) break;
    }

    // ---- epilogue: finish the last deferred service, spill state
    const uint64_t tend = t0 + ncyc;
    if (active) {
        if (has_pend) phase3(S, K, c, pend, tend - 1, acc);
        S.fifo_ctl[c.l] = c.qctl;
        if (MODE == 1u) {
            S.core_hot[c.l] = c.hot;
            S.core_cold[c.l] = c.cold;
        }
        const uint32_t be = (uint32_t)tend & 1u;
        const uint32_t fl = sflag[be * tpad + i];
        const uint8_t ste = stamp_of(tend);
        uint32_t gfl = 0;
        for (uint32_t d = 0; d < 4; ++d) {
            if (((fl >> (8u * d)) & 0xFFu) == ste) {
                S.flit[be][(size_t)d * S.nloc + c.l] = sflit[(be * 4u + d) * tpad + i];
                gfl |= (uint32_t)ste << (8u * d);
            }
        }
        S.flag[be][c.l] = gfl;
        S.flag[be ^ 1u][c.l] = 0u;
    }
    // statistics
    {
        uint32_t v[4] = {acc.injected, acc.ejected, acc.hops, acc.defl};
        const uint32_t idx[4] = {C_INJECTED, C_EJECTED, C_HOPS, C_DEFL};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t s = __reduce_add_sync(0xFFFFFFFFu, v[k]);
            if ((i & 31u) == 0 && s) atomicAdd(&scnt[idx[k]], s);
        }
    }
    __syncthreads();
    for (uint32_t k = i; k < NCOUNTERS; k += blockDim.x)
        if (scnt[k]) atomicAdd(&S.cnt[k], (unsigned long long)scnt[k]);
    if (smem_hist)
        for (uint32_t k = i; k < 3u * S.nb; k += blockDim.x)
            if (shist[k]) atomicAdd(&S.hist[k], (unsigned long long)shist[k]);
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
size_t tiled_smem_bytes(const Dev &S, uint32_t tpad, bool with_hist)
{
    return (size_t)tpad * (8u * 16u + 2u * 4u) + 4u * NCOUNTERS + (with_hist ? 12u * (size_t)S.nb : 0u);
}

// Pick TX x TY <= SMs tiles minimising the largest tile, then its perimeter.
cudaError_t tiled_configure(Dev &S, int device, uint32_t *grid, uint32_t *tpad, uint32_t *smem_hist)
{
    int sms = 0, optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    uint64_t best_tn = ~0ull, best_per = ~0ull;
    uint32_t bx = 0, by = 0;
    for (uint32_t tx = 1; tx <= S.W && tx <= (uint32_t)sms; ++tx) {
        for (uint32_t ty = 1; ty <= S.rows && tx * ty <= (uint32_t)sms; ++ty) {
            uint64_t tw = (S.W + tx - 1) / tx, th = (S.rows + ty - 1) / ty;
            uint64_t tn = tw * th, per = tw + th;
            if (tn < best_tn || (tn == best_tn && per < best_per)) { best_tn = tn; best_per = per; bx = tx; by = ty; }
        }
    }
    if (best_tn > TILE_MAX_THREADS) return cudaErrorInvalidConfiguration;
    S.TX = bx;
    S.TY = by;
    uint32_t tp = (uint32_t)((best_tn + 31u) / 32u * 32u);
    bool with_hist = true;
    size_t smem = tiled_smem_bytes(S, tp, true);
    if (smem > (size_t)optin) {
        with_hist = false;
        smem = tiled_smem_bytes(S, tp, false);
        if (smem > (size_t)optin) return cudaErrorInvalidConfiguration;
    }
    const void *fn = S.mode == 1u ? (const void *)k_tiled<1> : (const void *)k_tiled<0>;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)tp, smem);
    if (e != cudaSuccess) return e;
    if ((uint64_t)per_sm * sms < (uint64_t)bx * by) return cudaErrorCooperativeLaunchTooLarge;
    *grid = bx * by;
    *tpad = tp;
    *smem_hist = with_hist ? 1u : 0u;
    return cudaSuccess;
}

cudaError_t launch_tiled(const Dev &S, uint64_t t0, uint32_t ncyc, uint32_t grid, uint32_t tpad, uint32_t smem_hist,
                         uint32_t *activity, cudaStream_t st)
{
    k_ll_refresh<<<256, 256, 0, st>>>(S, t0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t smem = tiled_smem_bytes(S, tpad, smem_hist != 0);
    Dev Sc = S;
    void *args[] = {(void *)&Sc, (void *)&t0, (void *)&ncyc, (void *)&smem_hist, (void *)&activity};
    const void *fn = S.mode == 1u ? (const void *)k_tiled<1> : (const void *)k_tiled<0>;
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(tpad), args, smem, st);
}

cudaError_t launch_ll_reset(const Dev &S, uint64_t t, cudaStream_t st)
{
    k_ll_reset<<<256, 256, 0, st>>>(S, t);
    return cudaGetLastError();
}

}  // namespace noc
