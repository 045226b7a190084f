// tile_engine.cu -- the TILED engine.
//
// One persistent CTA per rectangular tile of the mesh (<= 1 CTA per SM), one
// thread per node, many cycles per launch:
//   * every node's core / FIFO-control state lives in REGISTERS of its thread
//     for the whole launch (no per-cycle state round trip);
//   * links between nodes of the same tile live in SHARED memory: a flit and a
//     32-bit stamp (the cycle the slot is an input of) per slot, double
//     buffered by cycle parity -- nothing to clear, no ABA within a launch;
//   * links that cross a tile boundary are "LL" slots in global memory: the
//     sender writes 64-bit words carrying (cycle stamp, 32 data bits), so the
//     receiver polls the data itself -- no fence, flag or grid barrier.  Every
//     boundary output port is written every cycle (a flit or EMPTY), and each
//     cross-tile link pairs with its reverse link, so a sender never overwrites
//     a slot its receiver has not consumed (DESIGN 6.3);
//   * the boundary polls are issued first, so their latency overlaps the
//     node's other work;
//   * the service of an ejected flit (directory / L2 lookups, Fig. 4)
//     is deferred to the start of the next cycle (after the tile barrier) so
//     its global-memory latency overlaps the exchange; it still precedes the
//     node's next Phase 1 and injection, so the order of DESIGN 3.3 (R27) holds.
// The per-node model code is node_logic.cuh's (bit-identical to every engine).
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

// 16-byte relaxed accesses (two LL words).  Each 64-bit word carries its own
// stamp, so the receiver validates every word; no 128-bit atomicity is assumed.
__device__ __forceinline__ void ld_relaxed_x2(const unsigned long long *p, unsigned long long &a,
                                              unsigned long long &b)
{
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

__device__ __forceinline__ void st_relaxed_x2(unsigned long long *p, unsigned long long a, unsigned long long b)
{
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
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

// Thread <-> node mapping inside a tile: the interior nodes (no boundary port)
// take the first threads/warps, the boundary ring the last ones, so the warps
// of interior nodes never execute (or wait in) the boundary-exchange code.
__device__ __forceinline__ void tile_pos(const TileShape &T, uint32_t i, uint32_t &lx, uint32_t &ly)
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

__device__ __forceinline__ uint32_t tile_slot(const TileShape &T, uint32_t lx, uint32_t ly)
{
    if (T.tw < 3 || T.th < 3) return ly * T.tw + lx;
    const uint32_t iw = T.tw - 2, ic = iw * (T.th - 2);
    if (lx >= 1 && lx + 1 < T.tw && ly >= 1 && ly + 1 < T.th) return (ly - 1) * iw + (lx - 1);
    if (ly == 0) return ic + lx;
    if (ly + 1 == T.th) return ic + T.tw + lx;
    if (lx == 0) return ic + 2 * T.tw + (ly - 1);
    return ic + 2 * T.tw + (T.th - 2) + (ly - 1);
}

// Dynamic shared memory layout (np = blockDim.x node slots):
//   uint4    sflit[2][4][np]   link flits (input slot d of node slot i, by parity)
//   uint32_t sst[2][4][np]     stamp = the cycle the slot is an input of
//   uint4    sinj[np]          the flit injected this cycle
//   uint32_t scnt[NCOUNTERS]
//   uint32_t shist[3][nb]      (optional)
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void ld_relaxed_sys_x2(const unsigned long long *p, unsigned long long &a,
                                                  unsigned long long &b)
{
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys_x2(unsigned long long *p, unsigned long long a, unsigned long long b)
{
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// LL accesses: links inside the band use gpu scope, links across a band edge
// (possibly another GPU) system scope
__device__ __forceinline__ void ll_load2(bool sys, const unsigned long long *p, unsigned long long &a,
                                         unsigned long long &b)
{
    if (sys) ld_relaxed_sys_x2(p, a, b);
    else ld_relaxed_x2(p, a, b);
}
__device__ __forceinline__ void ll_store2(bool sys, unsigned long long *p, unsigned long long a, unsigned long long b)
{
    if (sys) st_relaxed_sys_x2(p, a, b);
    else st_relaxed_x2(p, a, b);
}
__device__ __forceinline__ void ll_store1(bool sys, unsigned long long *p, unsigned long long a)
{
    if (sys) st_relaxed_sys_u64(p, a);
    else st_relaxed_u64(p, a);
}

// Base of the LL array (parity nb) that output port p writes into: this band's
// own array, or the north / south neighbour band's across a band edge.
__device__ __forceinline__ unsigned long long *ll_out(const Dev &S, bool band_edge, uint32_t p, uint32_t nb,
                                                     uint32_t pstride)
{
    if (!band_edge) return S.ll + (size_t)nb * pstride;
    const uint32_t side = p == PN ? 0u : 1u;
    return S.ll_nb[side] + (size_t)nb * 16u * S.nloc_nb[side];
}

template <uint32_t MODE, bool DRAIN>
__global__ void __launch_bounds__(TILE_BLOCK_MAX, TILE_MIN_BLOCKS)
k_tiled(const __grid_constant__ DevSet P, uint64_t t0, uint32_t ncyc, uint32_t smem_hist, uint32_t *activity)
{
    // this CTA's band and tile
    uint32_t band = 0;
    while (band + 1 < P.nbands && blockIdx.x >= P.tile0[band + 1]) ++band;
    const Dev &S = P.d[band];
    const uint32_t tile = blockIdx.x - P.tile0[band];
    extern __shared__ uint4 smem4[];
    const uint32_t np = blockDim.x;
    uint4 *sflit = smem4;
    uint4 *sinj = sflit + 8u * np;
    uint32_t *sst = reinterpret_cast<uint32_t *>(sinj + np);
    uint32_t *snb = sst + 8u * np;                 // [4][np] neighbour node slot per port
    unsigned int *scnt = snb + 4u * np;
    unsigned int *shist = smem_hist ? scnt + NCOUNTERS : nullptr;
    __shared__ int s_abort;
    __shared__ uint32_t s_busy[2];

    const uint32_t i = threadIdx.x;
    const TileShape T = tile_shape(S, tile);
    const bool active = i < T.tn;

    {
        const uint32_t nsm = NCOUNTERS + (smem_hist ? 3u * S.nb : 0u);
        for (uint32_t k = i; k < nsm; k += blockDim.x) scnt[k] = 0u;
        if (i == 0) { s_abort = 0; s_busy[0] = s_busy[1] = 0u; }
    }

    // ---- node registers (persist for the whole launch)
    NodeCtx c;
    uint32_t lx = 0, lyy = 0;
    if (active) tile_pos(T, i, lx, lyy);
    c.x = T.x0 + lx;
    c.y = T.y0 + lyy;
    c.n = c.y * S.W + c.x;
    c.l = c.n - S.n0;
    c.head_ok = false;
    c.nd_ok = false;
    c.cold_loaded = true;
    c.q_dirty = c.hot_dirty = c.cold_dirty = false;
    c.busy_flit = false;
    uint32_t errf = 0;     // overflow flags seen by this thread (R32), reported once
    c.qctl = 0u;
    c.hot = 0u;
    c.cold = make_uint4(0, 0, 0, 0);
    uint32_t ext = 0;      // bit d: port d crosses the tile boundary
    uint32_t intl = 0;     // bit d: port d exists inside the tile
    uint32_t bedge = 0;    // bit d: port d crosses the band edge (N: 0, S: 1)
    uint32_t inw[4] = {0, 0, 0, 0}, outw[4] = {0, 0, 0, 0};
    c.deg = 0;
    const uint32_t b0 = (uint32_t)t0 & 1u;
    if (active) {
        c.qctl = S.fifo_ctl[c.l];
        if (MODE == 1u) {
            c.hot = S.core_hot[c.l];
            c.cold = S.core_cold[c.l];
        }
        if (q_count(c.qctl)) { c.head = S.fifo_pkt[(size_t)c.l * S.qcap + q_head(c.qctl)]; c.head_ok = true; }
        const uint32_t exist = (c.y > 0 ? 1u : 0u) | (c.y + 1 < S.H ? 2u : 0u) | (c.x + 1 < S.W ? 4u : 0u) |
                               (c.x > 0 ? 8u : 0u);
        ext = ((lyy == 0 ? 1u : 0u) | (lyy + 1 == T.th ? 2u : 0u) | (lx + 1 == T.tw ? 4u : 0u) |
               (lx == 0 ? 8u : 0u)) & exist;
        intl = exist & ~ext;
        c.deg = __popc(exist);
        bedge = ((c.y == S.row0 && c.y > 0) ? 1u : 0u) | ((c.y + 1 == S.row0 + S.rows && c.y + 1 < S.H) ? 2u : 0u);
#pragma unroll
        for (uint32_t d = 0; d < 4; ++d) {
            uint32_t m = c.l, mi = 0;
            switch (d) {
            case PN: m = c.l - S.W; if ((intl >> d) & 1u) mi = tile_slot(T, lx, lyy - 1); break;
            case PS: m = c.l + S.W; if ((intl >> d) & 1u) mi = tile_slot(T, lx, lyy + 1); break;
            case PE: m = c.l + 1u; if ((intl >> d) & 1u) mi = tile_slot(T, lx + 1, lyy); break;
            default: m = c.l - 1u; if ((intl >> d) & 1u) mi = tile_slot(T, lx - 1, lyy); break;
            }
            if ((ext >> d) & 1u) {
                inw[d] = (uint32_t)ll_index(S, 0, d, c.l, 0);
                if ((bedge >> d) & 1u) {
                    // the receiver is in the neighbour band: its local index there
                    const uint32_t nr = S.nloc_nb[d];
                    const uint32_t lr = d == PN ? c.l - S.W + nr : c.l + S.W - S.nloc;
                    outw[d] = (uint32_t)(((size_t)(d ^ 1u) * nr + lr) * 4u);
                } else {
                    outw[d] = (uint32_t)ll_index(S, 0, d ^ 1u, m, 0);
                }
            }
            snb[d * np + i] = mi;
        }
        // internal inputs of cycle t0 (spilled by the previous launch)
        const uint32_t fl = S.flag[b0][c.l];
        const uint8_t s0 = stamp_of(t0);
#pragma unroll
        for (uint32_t d = 0; d < 4; ++d) {
            const uint32_t si = (b0 * 4u + d) * np + i;
            bool has = false;
            if (((intl >> d) & 1u) && ((fl >> (8u * d)) & 0xFFu) == s0) {
                sflit[si] = S.flit[b0][(size_t)d * S.nloc + c.l];
                has = true;
            }
            sst[si] = has ? (uint32_t)t0 : (uint32_t)t0 - 1u;
            sst[((b0 ^ 1u) * 4u + d) * np + i] = (uint32_t)t0 - 1u;
        }
    }
    __syncthreads();

    const uint32_t pstride = 16u * S.nloc;
    Sink K{scnt, shist, true};
    Acc acc = {0, 0, 0, 0};
    Flit pend = {0, 0, 0, 0};
    bool has_pend = false;

    for (uint32_t cc = 0; cc < ncyc; ++cc) {
        const uint64_t t = t0 + cc;
        const uint32_t pb = (uint32_t)t & 1u, nb1 = pb ^ 1u;
        const uint32_t st = (uint32_t)t, stn = st + 1u;
        bool busy = false;
        if (active) {
            unsigned long long *const llp = S.ll + (size_t)pb * pstride;   // this cycle's boundary inputs
            // issue the boundary polls first (all four words of each slot)
            unsigned long long xa[4] = {0, 0, 0, 0}, xb[4] = {0, 0, 0, 0}, xc[4] = {0, 0, 0, 0},
                               xd[4] = {0, 0, 0, 0};
#pragma unroll
            for (uint32_t d = 0; d < 4; ++d)
                if ((ext >> d) & 1u) {
                    const bool sys = (bedge >> d) & 1u;
                    ll_load2(sys, llp + inw[d], xa[d], xb[d]);
                    ll_load2(sys, llp + inw[d] + 2, xc[d], xd[d]);
                }

            // deferred Phase 3 of cycle t-1
            if (has_pend) { phase3(S, K, c, pend, t - 1, acc); has_pend = false; }

            // Phase 1
            if (MODE == 0u) phase1_ur(S, K, c, t);
            else phase1_lspd(S, K, c, t);

            // Phase 2: which input slots hold a flit this cycle.  All
            // flits stay in shared memory (slot k<4: sflit, k=4: sinj).
            uint32_t present = 0;
#pragma unroll
            for (uint32_t d = 0; d < 4; ++d)
                if (((intl >> d) & 1u) && sst[(pb * 4u + d) * np + i] == st) present |= 1u << d;
            // boundary inputs: spin on the LL stamps, then stage the flit
            if (ext) {
#pragma unroll
                for (uint32_t d = 0; d < 4; ++d) {
                    if (!((ext >> d) & 1u)) continue;
                    const unsigned long long *slot = llp + inw[d];
                    uint32_t spins = 0;
                    unsigned long long w0 = xa[d], w1 = xb[d], w2 = xc[d], w3 = xd[d];
                    // complete when word 0 carries this cycle's stamp and, for a
                    // flit (not EMPTY), so do words 1..3
                    while ((uint32_t)w0 != st ||
                           ((uint32_t)(w0 >> 32) != LL_EMPTY &&
                            ((uint32_t)w1 != st || (uint32_t)w2 != st || (uint32_t)w3 != st))) {
                        if (++spins > (1u << 22)) { atomicOr(S.err, 0x80000000u); s_abort = 1; break; }
                        const bool sys = (bedge >> d) & 1u;
                        ll_load2(sys, slot, w0, w1);
                        ll_load2(sys, slot + 2, w2, w3);
                    }
                    const uint32_t x = (uint32_t)(w0 >> 32);
                    if ((uint32_t)w0 == st && x != LL_EMPTY) {
                        sflit[(pb * 4u + d) * np + i] =
                            make_uint4(x, (uint32_t)(w1 >> 32), (uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32));
                        present |= 1u << d;
                    }
                }
            }
            {
                Flit fi;
                if (inject_flit(S, c, (uint32_t)__popc(present), t, acc, fi)) {
                    sinj[i] = make_uint4(fi.x, fi.y, fi.z, fi.w);
                    present |= 16u;
                }
            }
            auto slot_flit = [&](uint32_t k) -> Flit {
                const uint4 v = k < 4u ? sflit[(pb * 4u + k) * np + i] : sinj[i];
                return Flit{v.x, v.y, v.z, v.w};
            };
            auto out = [&](uint32_t p, const Flit &f) {
                const uint32_t slot = p ^ 1u;   // opp(p): N<->S (0,1), E<->W (2,3)
                if ((ext >> p) & 1u) {
                    const bool sys = (bedge >> p) & 1u;
                    unsigned long long *o = ll_out(S, sys, p, nb1, pstride) + pick4(outw, p);
                    ll_store2(sys, o + 2, llw(stn, f.z), llw(stn, f.w));
                    ll_store2(sys, o, llw(stn, f.x), llw(stn, f.y));
                } else {
                    const uint32_t so = (nb1 * 4u + slot) * np + snb[p * np + i];
                    sflit[so] = make_uint4(f.x, f.y, f.z, f.w);
                    sst[so] = stn;
                }
            };
            Flit ej;
            bool has_ej = false;
            uint32_t used = 0;
            if (present) {
                // fast path over the present slots only: if the first choices
                // are pairwise distinct, every flit takes its first choice
                uint32_t seen = 0, fcs = 0;
                bool coll = false;
                for (uint32_t m = present; m; m &= m - 1u) {
                    const uint32_t k = __ffs(m) - 1u;
                    const uint32_t fc = first_choice(S, c, slot_flit(k), st, errf);
                    coll |= (seen >> fc) & 1u;
                    seen |= 1u << fc;
                    fcs |= fc << (4u * k);
                }
                if (!coll) {
                    for (uint32_t m = present; m; m &= m - 1u) {
                        const uint32_t k = __ffs(m) - 1u, fc = (fcs >> (4u * k)) & 15u;
                        const Flit f = slot_flit(k);
                        if (fc == PX) { ej = f; has_ej = true; continue; }
                        ++acc.hops;
                        out(fc, f);
                    }
                    used = seen & 15u;
                } else {
                    // general case: full ranking + greedy
                    Inputs in;
                    in.present = present;
#pragma unroll
                    for (uint32_t k = 0; k < 5; ++k)
                        if ((present >> k) & 1u) in.f[k] = slot_flit(k);
                    used = route_select(S, c, in, t, acc, ej, has_ej, out);
                }
            }
            // boundary ports without a flit carry an explicit EMPTY every cycle
            const uint32_t idle_ext = ext & ~used;
#pragma unroll
            for (uint32_t p = 0; p < 4; ++p)
                if ((idle_ext >> p) & 1u) {
                    const bool sys = (bedge >> p) & 1u;
                    ll_store1(sys, ll_out(S, sys, p, nb1, pstride) + outw[p], llw(stn, LL_EMPTY));
                }
            if (has_ej) {
                // while draining, quiescence is judged at the end of each cycle,
                // so the service is not deferred there
                if (DRAIN) phase3(S, K, c, ej, t, acc);
                else { pend = ej; has_pend = true; if (MODE == 1u) prefetch_service(S, c, ej); }
            }
            if (DRAIN) busy = used != 0u || has_pend || q_count(c.qctl) > 0u || core_mode(c.hot) != MIDLE;
            // the generation draw of cycle t+1, off the critical path
            predraw(S, c, t + 1);
        }
        // The cycle barrier is a full BAR.SYNC: it orders this cycle's shared-
        // memory link stores before the next cycle's loads (a reducing barrier,
        // __syncthreads_or, measurably did not on sm_100a).
        if (DRAIN && busy) s_busy[cc & 1u] = cc + 1u;
        __syncthreads();
        if (DRAIN && i == 0 && s_busy[cc & 1u] == cc + 1u) atomicAdd(&activity[cc], 1u);
        if (s_abort) break;
    }

    // ---- epilogue: finish the last deferred service, spill state
    const uint64_t tend = t0 + ncyc;
    if (active) {
        if (has_pend) phase3(S, K, c, pend, tend - 1, acc);
        if (errf) atomicOr(S.err, errf);
        S.fifo_ctl[c.l] = c.qctl;
        if (MODE == 1u) {
            S.core_hot[c.l] = c.hot;
            S.core_cold[c.l] = c.cold;
        }
        const uint32_t be = (uint32_t)tend & 1u;
        const uint8_t ste = stamp_of(tend);
        uint32_t gfl = 0;
#pragma unroll
        for (uint32_t d = 0; d < 4; ++d) {
            const uint32_t si = (be * 4u + d) * np + i;
            if (((intl >> d) & 1u) && sst[si] == (uint32_t)tend) {
                S.flit[be][(size_t)d * S.nloc + c.l] = sflit[si];
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
size_t tiled_smem_bytes(const Dev &S, uint32_t np, bool with_hist)
{
    return (size_t)np * (9u * 16u + 12u * 4u) + 4u * NCOUNTERS + (with_hist ? 12u * (size_t)S.nb : 0u);
}

// Pick TX x TY tiles for one band (<= tiles_budget CTAs, <= TILE_BLOCK_MAX
// nodes each) minimising the largest tile, then its perimeter.  Host only.
bool tiled_plan(Dev &S, uint32_t tiles_budget, uint32_t *tiles, uint32_t *np)
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
    if (bx == 0 || best_tn > TILE_BLOCK_MAX) return false;
    S.TX = bx;
    S.TY = by;
    *tiles = bx * by;
    *np = (uint32_t)((best_tn + 31u) / 32u * 32u);
    return true;
}

// Shared-memory attribute and co-residency check for one launch of
// total_tiles CTAs of np threads.
cudaError_t tiled_prepare(uint32_t mode, uint32_t nb, uint32_t np, uint32_t total_tiles, int device,
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
    const void *fns[2] = {mode == 1u ? (const void *)k_tiled<1, false> : (const void *)k_tiled<0, false>,
                          mode == 1u ? (const void *)k_tiled<1, true> : (const void *)k_tiled<0, true>};
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
    const void *fn = P.d[0].mode == 1u ? (dr ? (const void *)k_tiled<1, true> : (const void *)k_tiled<1, false>)
                                       : (dr ? (const void *)k_tiled<0, true> : (const void *)k_tiled<0, false>);
    return cudaLaunchCooperativeKernel(fn, dim3(P.tile0[P.nbands]), dim3(tpad), args, smem, st);
}

cudaError_t launch_ll_reset(const Dev &S, uint64_t t, cudaStream_t st)
{
    k_ll_reset<<<256, 256, 0, st>>>(S, t);
    return cudaGetLastError();
}

}  // namespace noc
