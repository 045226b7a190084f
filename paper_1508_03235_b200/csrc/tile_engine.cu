// tile_engine.cu -- the TILED engine.
//
// Persistent CTAs, each owning a rectangular tile of the mesh, many cycles per
// launch.  FOUR LANES PER NODE: lane g of a node's 4-lane group owns the
// node's input slot g and output port g (N, S, E, W).
//   * the node's core / FIFO-control state is REPLICATED in the 4 lanes'
//     registers: Phase 1 and the Phase-3 service run converged on all 4 lanes
//     (identical, idempotent global stores; only the lead lane counts), so
//     there is no per-cycle state round trip and no broadcast;
//   * Phase 2 is lane-parallel: each lane latches its own slot, computes its
//     flit's 64-bit priority key and routing preference; ranks come from
//     group shuffles; every lane then replays the same greedy port assignment
//     (serial dictatorship over <= 4 flits) and stores its own flit;
//   * links inside a tile live in SHARED memory (flit + 32-bit cycle stamp,
//     double buffered by parity); links that cross a tile boundary are "LL"
//     slots in global memory whose 64-bit words carry (stamp, 32 data bits), so
//     a receiver polls the data itself -- no fence, flag or grid barrier.
//     Every boundary output port is written every cycle (a flit or EMPTY), and
//     each cross-tile link pairs with its reverse link, so a sender can never
//     overwrite a slot its receiver has not consumed (DESIGN 6.3);
//   * the service of an ejected flit (directory / L2 lookups, Fig. 4)
//     is deferred to the start of the next cycle, so its global-memory latency
//     overlaps the tile barrier and the boundary exchange; it still precedes
//     the node's next Phase 1 and injection (DESIGN 3.3 order, R27).
// The model is node_logic.cuh's; results are bit-identical to every engine.
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

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr uint32_t NOPORT = 8u;

// Dynamic shared memory layout (np = node slots per CTA = blockDim/4):
//   uint4    sflit[2][4][np]     link flits (input slot d of node i, by parity)
//   uint32_t sst[2][4][np]       stamp = the cycle the slot is an input of
//   uint32_t scnt[NCOUNTERS]
//   uint32_t shist[3][nb]        (optional)
template <uint32_t MODE>
__global__ void __launch_bounds__(TILE_BLOCK_MAX, TILE_MIN_BLOCKS)
k_tiled(Dev S, uint64_t t0, uint32_t ncyc, uint32_t smem_hist, uint32_t *activity)
{
    extern __shared__ uint4 smem4[];
    const uint32_t np = blockDim.x >> 2;
    uint4 *sflit = smem4;
    uint32_t *sst = reinterpret_cast<uint32_t *>(sflit + 8u * np);
    unsigned int *scnt = sst + 8u * np;
    unsigned int *shist = smem_hist ? scnt + NCOUNTERS : nullptr;
    __shared__ int s_abort;
    __shared__ uint32_t s_busy[2];

    const uint32_t tid = threadIdx.x, g = tid & 3u, i = tid >> 2;
    const uint32_t gb = tid & 28u;               // first lane of this node's group in the warp
    const TileShape T = tile_shape(S, blockIdx.x);
    const bool active = i < T.tn;

    {
        const uint32_t nsm = NCOUNTERS + (smem_hist ? 3u * S.nb : 0u);
        for (uint32_t k = tid; k < nsm; k += blockDim.x) scnt[k] = 0u;
        if (tid == 0) { s_abort = 0; s_busy[0] = s_busy[1] = 0u; }
    }

    // ---- node registers (replicated in the 4 lanes, kept for the whole launch)
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
    c.qctl = 0u;
    c.hot = 0u;
    c.cold = make_uint4(0, 0, 0, 0);
    uint32_t exist = 0, ext = 0;                 // bit d: port d exists / crosses the tile boundary
    uint32_t inw = 0, outw = 0, nbi = 0;         // LL word offsets (parity 0) / neighbour node slot
    const uint32_t pstride = 16u * S.nloc;
    const uint32_t b0 = (uint32_t)t0 & 1u;
    if (active) {
        c.qctl = S.fifo_ctl[c.l];
        if (MODE == 1u) {
            c.hot = S.core_hot[c.l];
            c.cold = S.core_cold[c.l];
        }
        if (q_count(c.qctl)) { c.head = S.fifo_pkt[(size_t)c.l * S.qcap + q_head(c.qctl)]; c.head_ok = true; }
        exist = (c.y > 0 ? 1u : 0u) | (c.y + 1 < S.H ? 2u : 0u) | (c.x + 1 < S.W ? 4u : 0u) | (c.x > 0 ? 8u : 0u);
        ext = ((lyy == 0 ? 1u : 0u) | (lyy + 1 == T.th ? 2u : 0u) | (lx + 1 == T.tw ? 4u : 0u) |
               (lx == 0 ? 8u : 0u)) & exist;
        if ((exist >> g) & 1u) {
            uint32_t m, mi;
            switch (g) {
            case PN: m = c.l - S.W; mi = i - T.tw; break;
            case PS: m = c.l + S.W; mi = i + T.tw; break;
            case PE: m = c.l + 1u; mi = i + 1u; break;
            default: m = c.l - 1u; mi = i - 1u; break;
            }
            if ((ext >> g) & 1u) {
                inw = (uint32_t)ll_index(S, 0, g, c.l, 0);
                outw = (uint32_t)ll_index(S, 0, g ^ 1u, m, 0);
            }
            nbi = mi;
        }
        // this lane's internal input slot of cycle t0 (spilled by the previous launch)
        bool has = false;
        if ((exist >> g) & 1u && !((ext >> g) & 1u)) {
            const uint32_t fb = (S.flag[b0][c.l] >> (8u * g)) & 0xFFu;
            if (fb == stamp_of(t0)) {
                sflit[(b0 * 4u + g) * np + i] = S.flit[b0][(size_t)g * S.nloc + c.l];
                has = true;
            }
        }
        sst[(b0 * 4u + g) * np + i] = has ? (uint32_t)t0 : (uint32_t)t0 - 1u;
        sst[((b0 ^ 1u) * 4u + g) * np + i] = (uint32_t)t0 - 1u;
    }
    const bool my_ext = (ext >> g) & 1u;
    const bool my_int = ((exist & ~ext) >> g) & 1u;
    __syncthreads();

    Sink K{scnt, shist, g == 0u};
    Acc acc = {0, 0, 0, 0};
    Flit pend = {0, 0, 0, 0};
    bool has_pend = false;

    for (uint32_t cc = 0; cc < ncyc; ++cc) {
        const uint64_t t = t0 + cc;
        const uint32_t pb = (uint32_t)t & 1u, nb1 = pb ^ 1u;
        const uint32_t st = (uint32_t)t, stn = st + 1u;
        unsigned long long *const llp = S.ll + (size_t)pb * pstride;   // this cycle's boundary inputs
        unsigned long long *const lln = S.ll + (size_t)nb1 * pstride;  // next cycle's
        bool pres = false;
        Flit f = {0, 0, 0, 0};
        if (active) {
            // issue the boundary poll first: its latency overlaps the deferred
            // service and Phase 1
            unsigned long long w = my_ext ? ld_relaxed_u64(llp + inw) : 0ull;

            // deferred Phase 3 of cycle t-1
            if (has_pend) { phase3(S, K, c, pend, t - 1, acc); has_pend = false; }

            // Phase 1
            if (MODE == 0u) phase1_ur(S, K, c, t);
            else phase1_lspd(S, K, c, t);

            // Phase 2: latch this lane's input slot
            if (my_int) {
                const uint32_t si = (pb * 4u + g) * np + i;
                if (sst[si] == st) {
                    const uint4 v = sflit[si];
                    f = Flit{v.x, v.y, v.z, v.w};
                    pres = true;
                }
            } else if (my_ext) {
                const unsigned long long *slot = llp + inw;
                uint32_t spins = 0;
                while ((uint32_t)w != st) {
                    if (++spins > (1u << 22)) { atomicOr(S.err, 0x80000000u); s_abort = 1; break; }
                    w = ld_relaxed_u64(slot);
                }
                const uint32_t x = (uint32_t)(w >> 32);
                if ((uint32_t)w == st && x != LL_EMPTY) {
                    unsigned long long w1 = ld_relaxed_u64(slot + 1), w2 = ld_relaxed_u64(slot + 2),
                                       w3 = ld_relaxed_u64(slot + 3);
                    while ((uint32_t)w1 != st || (uint32_t)w2 != st || (uint32_t)w3 != st) {
                        if (++spins > (1u << 22)) { atomicOr(S.err, 0x80000000u); s_abort = 1; break; }
                        if ((uint32_t)w1 != st) w1 = ld_relaxed_u64(slot + 1);
                        if ((uint32_t)w2 != st) w2 = ld_relaxed_u64(slot + 2);
                        if ((uint32_t)w3 != st) w3 = ld_relaxed_u64(slot + 3);
                    }
                    f = Flit{x, (uint32_t)(w1 >> 32), (uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32)};
                    pres = true;
                }
            }
        }

        // ---- injection (R7, R8): one flit of the head packet
        // into the first empty lane, if fewer flits than ports arrived
        uint32_t gp = (__ballot_sync(FULL, pres) >> gb) & 0xFu;
        if (active) {
            const uint32_t qn = q_count(c.qctl);
            if (qn > 0u && (uint32_t)__popc(gp) < (uint32_t)__popc(exist)) {
                const uint32_t slot = __ffs(~gp & 0xFu) - 1u;
                const uint32_t h = q_head(c.qctl);
                uint32_t nx = q_next(c.qctl);
                if (!c.head_ok) { c.head = S.fifo_pkt[(size_t)c.l * S.qcap + h]; c.head_ok = true; }
                const uint2 p = c.head;
                if (g == slot) {
                    f = f_make(p.x & NODE_MASK, (p.x >> 21) & 7u, nx, c.n, st, p.y);
                    pres = true;
                }
                gp |= 1u << slot;
                if (g == 0u) ++acc.injected;
                ++nx;
                if (nx == ((p.x >> 24) & 15u)) {
                    const uint32_t h1 = (h + 1u) & (S.qcap - 1u);
                    c.qctl = q_make(h1, qn - 1u, 0u);
                    c.head_ok = qn > 1u;
                    if (c.head_ok) c.head = S.fifo_pkt[(size_t)c.l * S.qcap + h1];
                } else {
                    c.qctl = q_make(h, qn, nx);
                }
            }
        }

        // ---- priority key (R1, R2) and routing preference of this lane's flit
        uint64_t key = 0ull;
        uint32_t pref = 0u;   // bit0 present, bit1 at destination, bit2 has x-port, [3:5) x-port,
                              // bit5 has y-port, [6:8) y-port
        if (pres) {
            key = prio_key(S, f, st);
            const uint32_t dst = f_dst(f);
            pref = 1u;
            if (dst == c.n) {
                pref |= 2u;
            } else {
                const uint32_t dy = row_of(S, dst), dx = dst - dy * S.W;
                if (dx != c.x) pref |= 4u | ((dx > c.x ? PE : PW) << 3);
                if (dy != c.y) pref |= 32u | ((dy > c.y ? PS : PN) << 6);
            }
        }
        // rank = number of group flits with a larger key ("Priority Sort")
        uint32_t rank = 0;
#pragma unroll
        for (uint32_t j = 1; j < 4; ++j) {
            const uint32_t src = gb + ((g + j) & 3u);
            const uint32_t lo = __shfl_sync(FULL, (uint32_t)key, src);
            const uint32_t hi = __shfl_sync(FULL, (uint32_t)(key >> 32), src);
            rank += (((uint64_t)hi << 32) | lo) > key;
        }
        const uint32_t word = pref | (rank << 8);
        uint32_t w4[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) w4[k] = __shfl_sync(FULL, word, gb + k);

        // ---- port assignment in rank order (PMDR x then y, P:L116;
        // deflection to the first free existing port in N,S,E,W, R4-R6);
        // replayed identically by the 4 lanes of the group
        uint32_t used = 0, ports = 0, dmask = 0, ejl = NOPORT;
#pragma unroll
        for (uint32_t r = 0; r < 4; ++r) {
            uint32_t sel = 0, lk = 0;
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k)
                if ((w4[k] & 1u) && (w4[k] >> 8) == r) { sel = w4[k]; lk = k; }
            if (sel & 1u) {
                uint32_t p = NOPORT;
                if ((sel & 2u) && ejl == NOPORT) {
                    ejl = lk;
                    p = PX;
                } else {
                    if (!(sel & 2u)) {
                        const uint32_t xp = (sel >> 3) & 3u, yp = (sel >> 6) & 3u;
                        if ((sel & 4u) && !((used >> xp) & 1u)) p = xp;
                        else if ((sel & 32u) && !((used >> yp) & 1u)) p = yp;
                    }
                    if (p == NOPORT) {
                        p = __ffs(exist & ~used) - 1u;
                        dmask |= 1u << lk;
                    }
                    used |= 1u << p;
                }
                ports |= p << (4u * lk);
            }
        }

        // ---- store this lane's routed flit into its next-cycle slot
        const uint32_t myport = pres ? ((ports >> (4u * g)) & 0xFu) : 0u;
        const uint32_t sl = gb + (myport & 3u);
        const uint32_t o_ll = __shfl_sync(FULL, outw, sl);     // LL offset of port myport
        const uint32_t o_ni = __shfl_sync(FULL, nbi, sl);      // neighbour slot of port myport
        if (pres && myport != PX) {
            if ((dmask >> g) & 1u) {
                uint32_t a = f_age(f) + 1u;                      // P:L116 age increment
                if (a > AGE_MAX) { atomicOr(S.err, ERR_AGE); a = AGE_MAX; }
                f_set_age(f, a);
                ++acc.defl;
            }
            ++acc.hops;
            const uint32_t slot = myport ^ 1u;                   // opp(port)
            if ((ext >> myport) & 1u) {
                unsigned long long *o = lln + o_ll;
                st_relaxed_u64(o + 1, llw(stn, f.y));
                st_relaxed_u64(o + 2, llw(stn, f.z));
                st_relaxed_u64(o + 3, llw(stn, f.w));
                st_relaxed_u64(o, llw(stn, f.x));
            } else {
                const uint32_t so = (nb1 * 4u + slot) * np + o_ni;
                sflit[so] = make_uint4(f.x, f.y, f.z, f.w);
                sst[so] = stn;
            }
        }
        // a boundary port without a flit carries an explicit EMPTY every cycle
        if (my_ext && !((used >> g) & 1u)) st_relaxed_u64(lln + outw, llw(stn, LL_EMPTY));

        // ---- ejection: hand the flit to the whole group (Phase 3 runs replicated)
        if (__any_sync(FULL, ejl != NOPORT)) {
            const uint32_t es = gb + (ejl & 3u);
            Flit e;
            e.x = __shfl_sync(FULL, f.x, es);
            e.y = __shfl_sync(FULL, f.y, es);
            e.z = __shfl_sync(FULL, f.z, es);
            e.w = __shfl_sync(FULL, f.w, es);
            if (active && ejl != NOPORT) {
                // while draining, quiescence is judged at the end of each cycle,
                // so the service is not deferred there
                if (activity) phase3(S, K, c, e, t, acc);
                else { pend = e; has_pend = true; }
            }
        }
        const bool busy = active && (used != 0u || has_pend || q_count(c.qctl) > 0u || core_mode(c.hot) != MIDLE);
        // The cycle barrier is a full BAR.SYNC: it orders this cycle's shared-
        // memory link stores before the next cycle's loads (a reducing barrier,
        // __syncthreads_or, measurably did not on sm_100a).
        if (activity && busy) s_busy[cc & 1u] = cc + 1u;
        __syncthreads();
        if (activity && tid == 0 && s_busy[cc & 1u] == cc + 1u) atomicAdd(&activity[cc], 1u);
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
        const uint32_t si = (be * 4u + g) * np + i;
        uint8_t fb = 0;
        if (my_int && sst[si] == (uint32_t)tend) {
            S.flit[be][(size_t)g * S.nloc + c.l] = sflit[si];
            fb = stamp_of(tend);
        }
        reinterpret_cast<uint8_t *>(&S.flag[be][c.l])[g] = fb;
        reinterpret_cast<uint8_t *>(&S.flag[be ^ 1u][c.l])[g] = 0;
    }
    // statistics
    {
        uint32_t v[4] = {acc.injected, acc.ejected, acc.hops, acc.defl};
        const uint32_t idx[4] = {C_INJECTED, C_EJECTED, C_HOPS, C_DEFL};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t s = __reduce_add_sync(FULL, v[k]);
            if ((tid & 31u) == 0 && s) atomicAdd(&scnt[idx[k]], s);
        }
    }
    __syncthreads();
    for (uint32_t k = tid; k < NCOUNTERS; k += blockDim.x)
        if (scnt[k]) atomicAdd(&S.cnt[k], (unsigned long long)scnt[k]);
    if (smem_hist)
        for (uint32_t k = tid; k < 3u * S.nb; k += blockDim.x)
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
size_t tiled_smem_bytes(const Dev &S, uint32_t np, bool with_hist)
{
    return (size_t)np * (8u * 16u + 8u * 4u) + 4u * NCOUNTERS + (with_hist ? 12u * (size_t)S.nb : 0u);
}

// Pick TX x TY tiles (<= TILE_MIN_BLOCKS CTAs per SM, <= TILE_MAX_NODES nodes
// each) minimising the largest tile, then its perimeter.
cudaError_t tiled_configure(Dev &S, int device, uint32_t *grid, uint32_t *tpad, uint32_t *smem_hist)
{
    int sms = 0, optin = 0, smem_sm = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    if (e != cudaSuccess) return e;
    const uint64_t max_ctas = (uint64_t)sms * TILE_MIN_BLOCKS;
    uint64_t best_tn = ~0ull, best_per = ~0ull;
    uint32_t bx = 0, by = 0;
    for (uint32_t tx = 1; tx <= S.W && tx <= max_ctas; ++tx) {
        for (uint32_t ty = 1; ty <= S.rows && (uint64_t)tx * ty <= max_ctas; ++ty) {
            uint64_t tw = (S.W + tx - 1) / tx, th = (S.rows + ty - 1) / ty;
            uint64_t tn = tw * th, per = tw + th;
            if (tn < best_tn || (tn == best_tn && per < best_per)) { best_tn = tn; best_per = per; bx = tx; by = ty; }
        }
    }
    if (best_tn > TILE_MAX_NODES) return cudaErrorInvalidConfiguration;
    S.TX = bx;
    S.TY = by;
    const uint32_t np = (uint32_t)((best_tn + 7u) / 8u * 8u);
    const uint32_t threads = 4u * np;
    const void *fn = S.mode == 1u ? (const void *)k_tiled<1> : (const void *)k_tiled<0>;
    bool with_hist = true;
    size_t smem = tiled_smem_bytes(S, np, true);
    if (smem * TILE_MIN_BLOCKS + 2048 > (size_t)smem_sm || smem > (size_t)optin) {
        with_hist = false;
        smem = tiled_smem_bytes(S, np, false);
    }
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)threads, smem);
    if (e != cudaSuccess) return e;
    if ((uint64_t)per_sm * sms < (uint64_t)bx * by) return cudaErrorCooperativeLaunchTooLarge;
    *grid = bx * by;
    *tpad = threads;
    *smem_hist = with_hist ? 1u : 0u;
    return cudaSuccess;
}

cudaError_t launch_tiled(const Dev &S, uint64_t t0, uint32_t ncyc, uint32_t grid, uint32_t tpad, uint32_t smem_hist,
                         uint32_t *activity, cudaStream_t st)
{
    k_ll_refresh<<<256, 256, 0, st>>>(S, t0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    size_t smem = tiled_smem_bytes(S, tpad / 4u, smem_hist != 0);
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
