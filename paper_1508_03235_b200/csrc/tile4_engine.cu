// tile4_engine.cu -- the TILED4 engine: the tiled,
// persistent, shared-memory/LL design of tile_engine.cu with FOUR LANES PER
// NODE.  Lane g of a node's group owns input slot g and output port g (N, S,
// E, W):
//   * every lane latches its own slot (shared memory, or an LL poll for a
//     boundary slot) and, holding at most one flit, computes that flit's first
//     choice (eject / x-port / y-port);
//   * two xor-shuffles tell the group whether two flits want the same port;
//     if not, every flit takes its first choice (the greedy of P:L131 without
//     contention) and each lane stores its own flit -- the common case costs a
//     handful of instructions per lane instead of a serial loop per node;
//   * on a conflict the group ranks its flits by 64-bit priority keys (R1, R2;
//     shuffles) and every lane replays the same greedy over <= 4 flits;
//   * the node's core / FIFO state lives in the LEAD lane (g = 0) only: Phase 1
//     (P:L257), the injection decision (R7), and the deferred Phase-3 service
//     (Fig. 4) run there; an injected flit is handed to the first empty
//     lane and an ejected flit back to the lead by shuffles.
// Splitting a node over 4 lanes quarters the length of each warp's per-cycle
// instruction chain (the limiter of the one-thread-per-node kernel, which is
// latency-bound) at the same total work.  Model code is node_logic.cuh's; the
// results are bit-identical to every engine.
#include "node_logic.cuh"
#include "kernels.h"

namespace noc {
namespace t4 {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr uint32_t NOPORT = 8u;

__device__ __forceinline__ void ld2(bool sys, const unsigned long long *p, unsigned long long &a, unsigned long long &b)
{
    if (sys) asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st2(bool sys, unsigned long long *p, unsigned long long a, unsigned long long b)
{
    if (sys) asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
    else asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st1(bool sys, unsigned long long *p, unsigned long long a)
{
    if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ unsigned long long llw(uint32_t stamp, uint32_t data)
{
    return ((unsigned long long)data << 32) | stamp;
}

struct Shape {
    uint32_t x0, y0, tw, th, tn;
};

__device__ __forceinline__ Shape tile_shape(const Dev &S, uint32_t b)
{
    const uint32_t tx = b % S.TX, ty = b / S.TX;
    Shape T;
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

// node slot <-> tile coordinates: interior nodes first, then the boundary ring
__device__ __forceinline__ void pos(const Shape &T, uint32_t i, uint32_t &lx, uint32_t &ly)
{
    if (T.tw < 3 || T.th < 3) { lx = i % T.tw; ly = i / T.tw; return; }
    const uint32_t iw = T.tw - 2, ic = iw * (T.th - 2);
    if (i < ic) { lx = 1 + i % iw; ly = 1 + i / iw; return; }
    uint32_t j = i - ic;
    if (j < T.tw) { lx = j; ly = 0; return; }
    j -= T.tw;
    if (j < T.tw) { lx = j; ly = T.th - 1; return; }
    j -= T.tw;
    if (j < T.th - 2) { lx = 0; ly = 1 + j; return; }
    j -= T.th - 2;
    lx = T.tw - 1; ly = 1 + j;
}

__device__ __forceinline__ uint32_t slot_of(const Shape &T, uint32_t lx, uint32_t ly)
{
    if (T.tw < 3 || T.th < 3) return ly * T.tw + lx;
    const uint32_t iw = T.tw - 2, ic = iw * (T.th - 2);
    if (lx >= 1 && lx + 1 < T.tw && ly >= 1 && ly + 1 < T.th) return (ly - 1) * iw + (lx - 1);
    if (ly == 0) return ic + lx;
    if (ly + 1 == T.th) return ic + T.tw + lx;
    if (lx == 0) return ic + 2 * T.tw + (ly - 1);
    return ic + 2 * T.tw + (T.th - 2) + (ly - 1);
}

// Dynamic shared memory (np = node slots = blockDim/4):
//   uint4    sflit[2][4][np]     internal link flits, by parity
//   uint32_t sst[2][4][np]       stamp = the cycle the slot is an input of
//   uint32_t snb[4][np]          neighbour node slot of port p (internal ports)
//   uint32_t sllw[4][np]         LL word offset (parity 0) of port p's receiver (boundary ports)
//   uint32_t scnt[NCOUNTERS], shist[3][nb] (optional)
template <uint32_t MODE, bool DRAIN>
__global__ void __launch_bounds__(TILE4_BLOCK_MAX, TILE4_MIN_BLOCKS)
k_tiled4(const __grid_constant__ DevSet P, uint64_t t0, uint32_t ncyc, uint32_t smem_hist, uint32_t *activity)
{
    uint32_t band = 0;
    while (band + 1 < P.nbands && blockIdx.x >= P.tile0[band + 1]) ++band;
    const Dev &S = P.d[band];
    extern __shared__ uint4 smem4[];
    const uint32_t np = blockDim.x >> 2;
    uint4 *sflit = smem4;
    uint32_t *sst = reinterpret_cast<uint32_t *>(sflit + 8u * np);
    uint32_t *snb = sst + 8u * np;
    uint32_t *sllw = snb + 4u * np;
    unsigned int *scnt = sllw + 4u * np;
    unsigned int *shist = smem_hist ? scnt + NCOUNTERS : nullptr;
    __shared__ int s_abort;
    __shared__ uint32_t s_busy[2];

    const uint32_t tid = threadIdx.x, g = tid & 3u, i = tid >> 2;
    const uint32_t gb = tid & 28u;                 // first lane of this group in the warp
    const bool lead = g == 0u;
    const Shape T = tile_shape(S, blockIdx.x - P.tile0[band]);
    const bool active = i < T.tn;
    {
        const uint32_t nsm = NCOUNTERS + (smem_hist ? 3u * S.nb : 0u);
        for (uint32_t k = tid; k < nsm; k += blockDim.x) scnt[k] = 0u;
        if (tid == 0) { s_abort = 0; s_busy[0] = s_busy[1] = 0u; }
    }

    // ---- per-node constants (all lanes) and node state (lead lane)
    NodeCtx c;
    uint32_t lx = 0, lyy = 0;
    if (active) pos(T, i, lx, lyy);
    c.x = T.x0 + lx;
    c.y = T.y0 + lyy;
    c.n = c.y * S.W + c.x;
    c.l = c.n - S.n0;
    c.head_ok = false;
    c.nd_ok = false;
    c.cold_loaded = true;
    c.q_dirty = c.hot_dirty = c.cold_dirty = false;
    c.busy_flit = false;
    c.qctl = 0u;
    c.hot = 0u;
    c.cold = make_uint4(0, 0, 0, 0);
    const uint32_t exist = active ? ((c.y > 0 ? 1u : 0u) | (c.y + 1 < S.H ? 2u : 0u) | (c.x + 1 < S.W ? 4u : 0u) |
                                     (c.x > 0 ? 8u : 0u))
                                  : 0u;
    const uint32_t ext = ((lyy == 0 ? 1u : 0u) | (lyy + 1 == T.th ? 2u : 0u) | (lx + 1 == T.tw ? 4u : 0u) |
                          (lx == 0 ? 8u : 0u)) & exist;
    const uint32_t bedge = active ? (((c.y == S.row0 && c.y > 0) ? 1u : 0u) |
                                     ((c.y + 1 == S.row0 + S.rows && c.y + 1 < S.H) ? 2u : 0u))
                                  : 0u;
    c.deg = __popc(exist);
    const bool my_exist = (exist >> g) & 1u, my_ext = (ext >> g) & 1u, my_int = my_exist && !my_ext;
    const bool my_sys = (bedge >> g) & 1u;
    uint32_t inw = 0;
    const uint32_t b0 = (uint32_t)t0 & 1u;
    if (active) {
        if (lead) {
            c.qctl = S.fifo_ctl[c.l];
            if (MODE == 1u) {
                c.hot = S.core_hot[c.l];
                c.cold = S.core_cold[c.l];
            }
            if (q_count(c.qctl)) { c.head = fifo_of(S, c.l).p[q_head(c.qctl)]; c.head_ok = true; }
        }
        // port g's neighbour: slot in this tile, or LL receiver slot
        uint32_t m = c.l, mi = 0, w = 0;
        if (my_exist) {
            switch (g) {
            case PN: m = c.l - S.W; if (my_int) mi = slot_of(T, lx, lyy - 1); break;
            case PS: m = c.l + S.W; if (my_int) mi = slot_of(T, lx, lyy + 1); break;
            case PE: m = c.l + 1u; if (my_int) mi = slot_of(T, lx + 1, lyy); break;
            default: m = c.l - 1u; if (my_int) mi = slot_of(T, lx - 1, lyy); break;
            }
            if (my_ext) {
                inw = (uint32_t)ll_index(S, 0, g, c.l, 0);
                if (my_sys) {
                    const uint32_t nr = S.nloc_nb[g];
                    const uint32_t lr = g == PN ? c.l - S.W + nr : c.l + S.W - S.nloc;
                    w = (uint32_t)(((size_t)(g ^ 1u) * nr + lr) * 4u);
                } else {
                    w = (uint32_t)ll_index(S, 0, g ^ 1u, m, 0);
                }
            }
        }
        snb[g * np + i] = mi;
        sllw[g * np + i] = w;
        // this lane's internal input slot of cycle t0 (spilled by the previous launch)
        bool has = false;
        const uint32_t si = (b0 * 4u + g) * np + i;
        if (my_int && ((S.flag[b0][c.l] >> (8u * g)) & 0xFFu) == stamp_of(t0)) {
            sflit[si] = S.flit[b0][flit_at(S.nloc, g, c.l)];
            has = true;
        }
        sst[si] = has ? (uint32_t)t0 : (uint32_t)t0 - 1u;
        sst[((b0 ^ 1u) * 4u + g) * np + i] = (uint32_t)t0 - 1u;
    }
    __syncthreads();

    const uint32_t pstride = 16u * S.nloc;
    Sink K{scnt, shist, true};
    Acc acc = {0, 0, 0, 0};
    Flit pend = {0, 0, 0, 0};
    bool has_pend = false;
    uint32_t errf = 0;

    for (uint32_t cc = 0; cc < ncyc; ++cc) {
        const uint64_t t = t0 + cc;
        const uint32_t pb = (uint32_t)t & 1u, nb1 = pb ^ 1u;
        const uint32_t st = (uint32_t)t, stn = st + 1u;
        // (0) boundary poll issued first
        unsigned long long w0 = 0, w1 = 0, w2 = 0, w3 = 0;
        const unsigned long long *slot = S.ll + (size_t)pb * pstride + inw;
        if (my_ext) {
            ld2(my_sys, slot, w0, w1);
            ld2(my_sys, slot + 2, w2, w3);
        }
        // (1) lead: deferred Phase 3 of cycle t-1, then Phase 1 of cycle t
        if (active && lead) {
            if (has_pend) { phase3(S, K, c, pend, t - 1, acc); has_pend = false; }
            if (MODE == 0u) phase1_ur(S, K, c, t);
            else phase1_lspd(S, K, c, t);
        }
        // (2) latch this lane's slot
        bool pres = false;
        Flit f = {0, 0, 0, 0};
        if (my_int) {
            const uint32_t si = (pb * 4u + g) * np + i;
            if (sst[si] == st) {
                const uint4 v = sflit[si];
                f = Flit{v.x, v.y, v.z, v.w};
                pres = true;
            }
        } else if (my_ext) {
            uint32_t spins = 0;
            while ((uint32_t)w0 != st ||
                   ((uint32_t)(w0 >> 32) != LL_EMPTY &&
                    ((uint32_t)w1 != st || (uint32_t)w2 != st || (uint32_t)w3 != st))) {
                if (++spins > (1u << 22)) { atomicOr(S.err, 0x80000000u); s_abort = 1; break; }
                ld2(my_sys, slot, w0, w1);
                ld2(my_sys, slot + 2, w2, w3);
            }
            const uint32_t x = (uint32_t)(w0 >> 32);
            if ((uint32_t)w0 == st && x != LL_EMPTY) {
                f = Flit{x, (uint32_t)(w1 >> 32), (uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32)};
                pres = true;
            }
        }
        // (3) injection (R7, R8): the lead decides; the flit goes
        // to the first lane without an input flit
        uint32_t gp = (__ballot_sync(FULL, pres) >> gb) & 0xFu;
        uint32_t inj_lane = NOPORT;
        Flit fi = {0, 0, 0, 0};
        if (active && lead && inject_flit(S, c, (uint32_t)__popc(gp), t, acc, fi)) inj_lane = __ffs(~gp & 0xFu) - 1u;
        if (__any_sync(FULL, inj_lane != NOPORT)) {
            const uint32_t il = __shfl_sync(FULL, inj_lane, gb);
            const uint32_t ix = __shfl_sync(FULL, fi.x, gb), iy = __shfl_sync(FULL, fi.y, gb);
            const uint32_t iz = __shfl_sync(FULL, fi.z, gb), iw = __shfl_sync(FULL, fi.w, gb);
            if (il == g) { f = Flit{ix, iy, iz, iw}; pres = true; }
            if (il != NOPORT) gp |= 1u << il;
        }

        // (4) first choice and the group's conflict check
        uint32_t fc = NOPORT;
        if (pres) fc = first_choice(S, c, f, st, errf);
        const uint32_t mbit = pres ? (1u << fc) : 0u;
        const uint32_t m1 = __shfl_xor_sync(FULL, mbit, 1);
        uint32_t conf = (mbit & m1) ? 1u : 0u;
        const uint32_t pair = mbit | m1;
        const uint32_t m2 = __shfl_xor_sync(FULL, pair, 2);
        conf |= (pair & m2) ? 1u : 0u;
        conf |= __shfl_xor_sync(FULL, conf, 2);
        uint32_t used = (pair | m2) & 15u;           // ports taken if no conflict
        uint32_t port = fc;
        bool defl = false;
        if (__any_sync(FULL, conf)) {
            // (5) conflict: rank the group's flits ("Priority Sort") and
            // replay the greedy (R3-R6) in every lane
            const uint64_t key = pres ? prio_key(S, f, st) : 0ull;
            uint32_t rank = 0;
#pragma unroll
            for (uint32_t j = 1; j < 4; ++j) {
                const uint32_t src = gb + ((g + j) & 3u);
                const uint32_t lo = __shfl_sync(FULL, (uint32_t)key, src);
                const uint32_t hi = __shfl_sync(FULL, (uint32_t)(key >> 32), src);
                rank += (((uint64_t)hi << 32) | lo) > key;
            }
            // preference word: bit0 present, bit1 at destination, bit2 has x-port,
            // [3:5) x-port, bit5 has y-port, [6:8) y-port, [8:11) rank
            uint32_t pref = 0;
            if (pres) {
                const uint32_t dst = f_dst(f);
                pref = 1u;
                if (dst == c.n) {
                    pref |= 2u;
                } else {
                    const uint32_t dy = row_of(S, dst), dx = dst - dy * S.W;
                    if (dx != c.x) pref |= 4u | ((dx > c.x ? PE : PW) << 3);
                    if (dy != c.y && (S.route == 0u || dx == c.x)) pref |= 32u | ((dy > c.y ? PS : PN) << 6);
                }
            }
            const uint32_t word = pref | (rank << 8);
            uint32_t w4[4];
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) w4[k] = __shfl_sync(FULL, word, gb + k);
            uint32_t u = 0, ports = 0, dmask = 0, ejl = NOPORT;
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
                            if ((sel & 4u) && !((u >> xp) & 1u)) p = xp;
                            else if ((sel & 32u) && !((u >> yp) & 1u)) p = yp;
                        }
                        if (p == NOPORT) {
                            p = defl_port(exist & ~u, S.route);   // first free existing port, N,S,E,W (R5) / N,E,S,W (XY)
                            dmask |= 1u << lk;
                        }
                        u |= 1u << p;
                    }
                    ports |= p << (4u * lk);
                }
            }
            if (conf) {
                used = u;
                port = (ports >> (4u * g)) & 15u;
                defl = (dmask >> g) & 1u;
            }
        }

        // (6) store this lane's routed flit into its next-cycle slot
        const uint32_t pp = pres ? port : PX;
        if (pp < 4u) {
            if (defl) {
                uint32_t a = f_age(f) + 1u;                       // P:L116 age increment
                if (a > AGE_MAX) { errf |= ERR_AGE; a = AGE_MAX; }
                f_set_age(f, a);
                ++acc.defl;
            }
            ++acc.hops;
            if ((ext >> pp) & 1u) {
                const bool sys = (bedge >> pp) & 1u;
                unsigned long long *base = S.ll + (size_t)nb1 * pstride;
                if (sys) {
                    const uint32_t side = pp == PN ? 0u : 1u;
                    base = S.ll_nb[side] + (size_t)nb1 * 16u * S.nloc_nb[side];
                }
                unsigned long long *o = base + sllw[pp * np + i];
                st2(sys, o + 2, llw(stn, f.z), llw(stn, f.w));
                st2(sys, o, llw(stn, f.x), llw(stn, f.y));
            } else {
                const uint32_t so = (nb1 * 4u + (pp ^ 1u)) * np + snb[pp * np + i];
                sflit[so] = make_uint4(f.x, f.y, f.z, f.w);
                sst[so] = stn;
            }
        }
        // a boundary port without a flit carries an explicit EMPTY every cycle
        if (my_ext && !((used >> g) & 1u)) {
            unsigned long long *base = S.ll + (size_t)nb1 * pstride;
            if (my_sys) {
                const uint32_t side = g == PN ? 0u : 1u;
                base = S.ll_nb[side] + (size_t)nb1 * 16u * S.nloc_nb[side];
            }
            st1(my_sys, base + sllw[g * np + i], llw(stn, LL_EMPTY));
        }
        // (7) ejection: the flit goes to the lead (Phase 3 there)
        const bool ej = pres && pp == PX;
        const uint32_t ejm = (__ballot_sync(FULL, ej) >> gb) & 0xFu;
        if (__any_sync(FULL, ejm != 0u)) {
            const uint32_t es = gb + (ejm ? __ffs(ejm) - 1u : 0u);
            Flit e;
            e.x = __shfl_sync(FULL, f.x, es);
            e.y = __shfl_sync(FULL, f.y, es);
            e.z = __shfl_sync(FULL, f.z, es);
            e.w = __shfl_sync(FULL, f.w, es);
            if (active && lead && ejm) {
                if (DRAIN) phase3(S, K, c, e, t, acc);
                else { pend = e; has_pend = true; if (MODE == 1u) prefetch_service(S, c, e); }
            }
        }
        bool busy = false;
        if (active && lead) {
            if (DRAIN) busy = used != 0u || has_pend || q_count(c.qctl) > 0u || core_mode(c.hot) != MIDLE;
            predraw(S, c, t + 1);
        }
        if (DRAIN && busy) s_busy[cc & 1u] = cc + 1u;
        __syncthreads();
        if (DRAIN && tid == 0 && s_busy[cc & 1u] == cc + 1u) atomicAdd(&activity[cc], 1u);
        if (s_abort) break;
    }

    // ---- epilogue
    const uint64_t tend = t0 + ncyc;
    if (active) {
        if (lead) {
            if (has_pend) phase3(S, K, c, pend, tend - 1, acc);
            S.fifo_ctl[c.l] = c.qctl;
            if (MODE == 1u) {
                S.core_hot[c.l] = c.hot;
                S.core_cold[c.l] = c.cold;
            }
        }
        if (errf) atomicOr(S.err, errf);
        const uint32_t be = (uint32_t)tend & 1u;
        const uint32_t si = (be * 4u + g) * np + i;
        uint8_t fb = 0;
        if (my_int && sst[si] == (uint32_t)tend) {
            S.flit[be][flit_at(S.nloc, g, c.l)] = sflit[si];
            fb = stamp_of(tend);
        }
        reinterpret_cast<uint8_t *>(&S.flag[be][c.l])[g] = fb;
        reinterpret_cast<uint8_t *>(&S.flag[be ^ 1u][c.l])[g] = 0;
    }
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

}  // namespace t4

size_t tiled4_smem_bytes(uint32_t nb, uint32_t np, bool with_hist)
{
    return (size_t)np * (8u * 16u + 16u * 4u) + 4u * NCOUNTERS + (with_hist ? 12u * (size_t)nb : 0u);
}

bool tiled4_plan(Dev &S, uint32_t tiles_budget, uint32_t *tiles, uint32_t *np)
{
    uint64_t best_tn = ~0ull, best_per = ~0ull;
    uint32_t bx = 0, by = 0;
    for (uint32_t tx = 1; tx <= S.W && tx <= tiles_budget; ++tx) {
        for (uint32_t ty = 1; ty <= S.rows && (uint64_t)tx * ty <= tiles_budget; ++ty) {
            uint64_t tw = (S.W + tx - 1) / tx, th = (S.rows + ty - 1) / ty;
            uint64_t tn = tw * th, per = tw + th;
            if (tn < best_tn || (tn == best_tn && per < best_per)) { best_tn = tn; best_per = per; bx = tx; by = ty; }
        }
    }
    if (bx == 0 || 4u * ((best_tn + 7u) / 8u * 8u) > TILE4_BLOCK_MAX) return false;
    S.TX = bx;
    S.TY = by;
    *tiles = bx * by;
    *np = (uint32_t)((best_tn + 7u) / 8u * 8u);
    return true;
}

cudaError_t tiled4_prepare(uint32_t mode, uint32_t nb, uint32_t np, uint32_t total_tiles, int device,
                           uint32_t *smem_hist)
{
    int sms = 0, optin = 0, smem_sm = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
    if (e != cudaSuccess) return e;
    const uint32_t ctas_per_sm = (total_tiles + sms - 1) / sms;
    bool with_hist = true;
    size_t smem = tiled4_smem_bytes(nb, np, true);
    if ((smem + 1024) * ctas_per_sm > (size_t)smem_sm || smem > (size_t)optin) {
        with_hist = false;
        smem = tiled4_smem_bytes(nb, np, false);
    }
    const void *fns[2] = {mode == 1u ? (const void *)t4::k_tiled4<1, false> : (const void *)t4::k_tiled4<0, false>,
                          mode == 1u ? (const void *)t4::k_tiled4<1, true> : (const void *)t4::k_tiled4<0, true>};
    for (const void *fn : fns) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)(4u * np), smem);
        if (e != cudaSuccess) return e;
        if ((uint64_t)per_sm * sms < total_tiles) return cudaErrorCooperativeLaunchTooLarge;
    }
    *smem_hist = with_hist ? 1u : 0u;
    return cudaSuccess;
}

cudaError_t launch_tiled4(const DevSet &P, uint64_t t0, uint32_t ncyc, uint32_t np, uint32_t smem_hist,
                          uint32_t *activity, cudaStream_t st)
{
    size_t smem = tiled4_smem_bytes(P.d[0].nb, np, smem_hist != 0);
    void *args[] = {(void *)&P, (void *)&t0, (void *)&ncyc, (void *)&smem_hist, (void *)&activity};
    const bool dr = activity != nullptr;
    const void *fn = P.d[0].mode == 1u
                         ? (dr ? (const void *)t4::k_tiled4<1, true> : (const void *)t4::k_tiled4<1, false>)
                         : (dr ? (const void *)t4::k_tiled4<0, true> : (const void *)t4::k_tiled4<0, false>);
    // the dynamic shared-memory limit is a per-function (process-wide)
    // attribute: another handle of a different size may have lowered it
    {
        const cudaError_t ea = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return ea;
    }
    return cudaLaunchCooperativeKernel(fn, dim3(P.tile0[P.nbands]), dim3(4u * np), args, smem, st);
}

}  // namespace noc
