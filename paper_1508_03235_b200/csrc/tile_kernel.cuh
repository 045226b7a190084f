// tile_kernel.cuh -- the TILED engine's node-step kernel.
// Instantiated per traffic mode in tile_m0.cu / tile_m1.cu / tile_m2.cu (the
// translation units compile in parallel); host code in tile_engine.cu.
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
#pragma once
#include "node_logic.cuh"
#include "kernels.h"

namespace noc {

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
// The ring starts at the first warp boundary after the interior and is spread
// evenly over its warps (`per` lanes each; C3's 30x10 tiles: 76 ring nodes as
// 26 + 25 + 25 instead of 32 + 32 + 12) when the block has room for it:
// the ring warps are the cycle's critical path, and a warp with fewer nodes
// meets fewer of the rare, long per-node events each cycle.
struct RingMap {
    uint32_t ic;    // interior nodes (threads 0 .. ic-1)
    uint32_t rs;    // first ring thread
    uint32_t per;   // ring nodes per ring warp
};
__device__ __forceinline__ RingMap ring_map(const TileShape &T, uint32_t np)
{
    RingMap m;
    if (T.tw < 3 || T.th < 3) { m.ic = 0; m.rs = 0; m.per = 32; return m; }   // all ring, linear
    m.ic = (T.tw - 2) * (T.th - 2);
    const uint32_t ring = T.tn - m.ic;
    const uint32_t rs = (m.ic + 31u) & ~31u, nw0 = (ring + 31u) / 32u;
    const uint32_t avail = np > rs ? (np - rs) / 32u : 0u;
    const uint32_t nw = min((ring + TILE_RING_CAP - 1u) / TILE_RING_CAP, avail);
#ifndef NOC_NO_RING_BALANCE
    if (nw >= nw0 && nw > 0u) { m.rs = rs; m.per = (ring + nw - 1u) / nw; return m; }
#endif
    m.rs = m.ic;   // contiguous
    m.per = 32u;
    return m;
}

// node of thread i (false: no node, a padding lane)
__device__ __forceinline__ bool tile_pos(const TileShape &T, const RingMap &M, uint32_t i, uint32_t &lx, uint32_t &ly)
{
    if (T.tw < 3 || T.th < 3) { lx = i % T.tw; ly = i / T.tw; return i < T.tn; }
    const uint32_t iw = T.tw - 2;
    if (i < M.ic) { lx = 1 + i % iw; ly = 1 + i / iw; return true; }
    if (i < M.rs) return false;
    const uint32_t r = i - M.rs, ln = r & 31u;
    if (ln >= M.per) return false;
    uint32_t j = (r >> 5) * M.per + ln;
    if (j >= T.tn - M.ic) return false;
    if (j < T.tw) { lx = j; ly = 0; return true; }
    j -= T.tw;
    if (j < T.tw) { lx = j; ly = T.th - 1; return true; }
    j -= T.tw;
    if (j < T.th - 2) { lx = 0; ly = 1 + j; return true; }
    j -= T.th - 2;
    lx = T.tw - 1; ly = 1 + j;
    return true;
}

// thread of node (lx, ly)
__device__ __forceinline__ uint32_t tile_slot(const TileShape &T, const RingMap &M, uint32_t lx, uint32_t ly)
{
    if (T.tw < 3 || T.th < 3) return ly * T.tw + lx;
    const uint32_t iw = T.tw - 2;
    if (lx >= 1 && lx + 1 < T.tw && ly >= 1 && ly + 1 < T.th) return (ly - 1) * iw + (lx - 1);
    uint32_t j;
    if (ly == 0) j = lx;
    else if (ly + 1 == T.th) j = T.tw + lx;
    else if (lx == 0) j = 2 * T.tw + (ly - 1);
    else j = 2 * T.tw + (T.th - 2) + (ly - 1);
    return M.rs + (j / M.per) * 32u + j % M.per;
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

// Dynamic shared memory layout (np = blockDim.x node slots):
//   uint4    sflit[2][4][np]   link flits (input slot d of node slot i, by parity)
//   uint32_t sfl[2][np]        occupancy word of node slot i: byte d is 1 iff
//                              input slot d holds a flit.  The receiver clears
//                              its word when it reads it; the next writes to
//                              that parity come a cycle later, after the cycle
//                              barrier, so no stamp (and no ABA) is needed
//   uint32_t scnt[NCOUNTERS]
//   uint32_t shist[3][nb]      (optional)
//
// The cycle body is written for few instructions per warp: 32 nodes share a
// warp, so any per-node branch costs the warp its full length whenever one
// lane takes it.  Hence (i) the occupancy of all four slots is one shared
// load, (ii) the routing decision of the common case is a handful of
// predicated operations per present flit, and the general case (two flits
// want the same port) works on packed 8-bit port preferences and ranks from a
// 6-comparison tournament, (iii) the LSPD generation draws (one Philox4x32-10
// per idle node-cycle, DESIGN 3.3) are evaluated 32 cycles at a time by the
// whole warp, one lane per cycle, instead of by one lane per cycle.
// Per-warp cycle trace (tools/trace_tiled.py; built only with -DNOC_TRACE):
// for each traced cycle and warp, the cycle-start clock, the clock offsets at
// which the boundary inputs were complete and the warp reached the cycle
// barrier, and the OR of its lanes' event bits (1 deferred Phase 3, 2 Phase-1
// state change, 4 Phase-1 enqueue, 8 draw-window refresh, 16 port conflict,
// 32 injection, 64 flits present, 128 boundary node).
#if defined(NOC_TRACE) && defined(NOC_TRACE_OWNER)
constexpr uint32_t TRACE_CYC = 1024, TRACE_WARPS = 1536;
__device__ uint4 g_trace[TRACE_CYC][TRACE_WARPS][2];
__device__ int g_trace_on;
#define TRACE_DECL long long tr_c0 = clock64(), tr_x = 0, tr_p3 = 0, tr_p1 = 0, tr_pub = 0; uint32_t tr_ev = 0;
#define TRACE_EV(b) tr_ev |= (b);
#define TRACE_P3_DONE tr_p3 = clock64();
#define TRACE_P1_DONE tr_p1 = clock64();
#define TRACE_EXT_DONE tr_x = clock64();
#define TRACE_PUB_DONE tr_pub = clock64();
#define TRACE_OFS(v) __reduce_max_sync(0xFFFFFFFFu, (v) ? (uint32_t)((v) - tr_c0) : 0u)
#define TRACE_END                                                                                       \
    {                                                                                                   \
        const uint32_t ev = __reduce_or_sync(0xFFFFFFFFu, tr_ev);                                       \
        const long long tr_a = clock64();                                                               \
        const uint32_t xw = TRACE_OFS(tr_x), p3w = TRACE_OFS(tr_p3), p1w = TRACE_OFS(tr_p1),            \
                       pbw = TRACE_OFS(tr_pub);                                                         \
        const uint32_t wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);                        \
        if (g_trace_on && (threadIdx.x & 31u) == 0u && cc < TRACE_CYC && wg < TRACE_WARPS) {            \
            g_trace[cc][wg][0] = make_uint4((uint32_t)tr_c0, (uint32_t)(tr_a - tr_c0), ev, xw);         \
            g_trace[cc][wg][1] = make_uint4(p3w, p1w, pbw, 0u);                                         \
        }                                                                                               \
    }
extern "C" int noc_trace_ctl(int on, void *host, size_t bytes)
{
    if (host) return (int)cudaMemcpyFromSymbol(host, g_trace, bytes < sizeof(g_trace) ? bytes : sizeof(g_trace));
    return (int)cudaMemcpyToSymbol(g_trace_on, &on, sizeof(int));
}
#else
#define TRACE_DECL
#define TRACE_EV(b)
#define TRACE_P3_DONE
#define TRACE_P1_DONE
#define TRACE_EXT_DONE
#define TRACE_PUB_DONE
#define TRACE_END
#endif

// Shared-memory access by 32-bit shared-window address (no generic->shared
// conversion in the loop); the stores are predicated, not branched around.
__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts32_if(bool c, uint32_t a, uint32_t v)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.u32 [%1], %2;\n\t}"
                 ::"r"((uint32_t)c), "r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void lds128_if(bool c, uint32_t a, Flit &f)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t@q ld.shared.v4.u32 {%0, %1, %2, %3}, [%5];\n\t}"
                 : "+r"(f.x), "+r"(f.y), "+r"(f.z), "+r"(f.w) : "r"((uint32_t)c), "r"(a) : "memory");
}
__device__ __forceinline__ void sts128_if(bool c, uint32_t a, const Flit &v)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.v4.u32 [%1], {%2, %3, %4, %5};\n\t}"
                 ::"r"((uint32_t)c), "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts8_if(bool c, uint32_t a)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.u8 [%1], %2;\n\t}"
                 ::"r"((uint32_t)c), "r"(a), "r"(1u) : "memory");
}

// Cluster exchange (FEAT bit 3): the whole band is ONE thread-block cluster of
// <= 16 tiles; a link to another tile is a store into that CTA's shared-memory
// slot (DSMEM, st.shared::cluster at the address mapa gives), and the cycle
// barrier is the cluster barrier (arrive.release / wait.acquire), which orders
// those stores before the next cycle's latch: no boundary polling at all.
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t a, const Flit &v)
{
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_cluster_u8(uint32_t a)
{
    asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(a), "r"(1u) : "memory");
}
__device__ __forceinline__ void cluster_barrier()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Split cycle barrier (DESIGN 6.3): one shared-memory mbarrier, one arrival
// per warp per cycle (lane 0, after __syncwarp), release / acquire at CTA
// scope; try_wait sleeps the warp in hardware until the phase completes.
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a)
{
    asm volatile("{\n\t.reg .b64 tok;\n\tmbarrier.arrive.release.cta.shared::cta.b64 tok, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" ::"r"(a), "r"(parity) : "memory");
}

// First choice of a flit with destination dst at node (n, x, y): eject at the
// destination, else the x-port while dx != 0, else the y-port (PMDR).
// Written as predicated selects (the nested ternary compiled to a branch
// region per slot).
__device__ __forceinline__ uint32_t first_port(uint32_t dst, uint32_t n, uint32_t x, uint32_t y, uint32_t W,
                                               uint32_t wmagic)
{
    const uint32_t dy = __umulhi(dst, wmagic), dx = dst - dy * W;
    uint32_t p;
    asm("{\n\t.reg .pred q;\n\t.reg .u32 px;\n\t"
        "setp.gt.u32 q, %2, %4;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t"          // y-port: S (1) if dy > y else N (0)
        "setp.gt.u32 q, %1, %3;\n\t"
        "selp.u32 px, 2, 3, q;\n\t"          // x-port: E (2) if dx > x else W (3)
        "setp.ne.u32 q, %1, %3;\n\t"
        "selp.u32 %0, px, %0, q;\n\t"
        "setp.eq.u32 q, %5, %6;\n\t"
        "selp.u32 %0, 4, %0, q;\n\t"          // eject (4) at the destination
        "}"
        : "=r"(p) : "r"(dx), "r"(dy), "r"(x), "r"(y), "r"(dst), "r"(n));
    return p;
}

// f[k] for a runtime k in [0, 5) without indexing a local array
__device__ __forceinline__ Flit pick5(const Flit (&f)[5], uint32_t k)
{
    Flit r = f[4];
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j)
        if (k == j) r = f[j];
    return r;
}

// One cross-tile input port of a boundary node: where its LL words are read.
struct ExtIn {
    uint32_t port;   // N, S, E or W; NOPORT if none
    uint32_t inw;    // LL word index (parity 0) of this node's input slot
    uint32_t outw;   // LL word index (parity 0) of the receiver's slot for output `port`
    bool sys;        // crosses the band edge (system scope)
};
constexpr uint32_t NOPORT = 8u;

// FEAT: the NEXT-f4 variants as compile-time bits (bit 0: strict-XY routing, R39;
// bit 1: an ejecting flit frees its port for injection, R43): a runtime check on
// these per-cycle paths measurably cost 1.5-5 % at C3 (profiles/r01_ab_engines.txt)
// MODE: 0 uniform random, 1 LSPD, 2 LSPD with the NEXT-f1 private L1 (the L1
// timer checks compiled in only there)
template <uint32_t MODE, bool DRAIN, uint32_t FEAT>
__global__ void __launch_bounds__(TILE_THREADS_MAX, TILE_MIN_BLOCKS)
k_tiled(const __grid_constant__ DevSet P, uint64_t t0, uint32_t ncyc, uint32_t smem_hist, uint32_t *activity)
{
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    constexpr bool CL = (FEAT & 8u) != 0u;   // cluster exchange (one band, <= 16 tiles)
    // this CTA's band and tile
    // FEAT bit 2: several bands in this launch (virtual bands).  With one band
    // the parameters are read at constant offsets (constant-bank operands of
    // the instructions themselves) instead of indexed constant loads that the
    // register-starved loop would otherwise re-issue every cycle
    uint32_t band = 0;
    if (FEAT & 4u)
        while (band + 1 < P.nbands && blockIdx.x >= P.tile0[band + 1]) ++band;
    const Dev &S = P.d[(FEAT & 4u) ? band : 0u];
    const uint32_t tile = blockIdx.x - ((FEAT & 4u) ? P.tile0[band] : 0u);
    extern __shared__ uint4 smem4[];
    const uint32_t np = blockDim.x;
    uint4 *sflit = smem4;
    uint32_t *sfl = reinterpret_cast<uint32_t *>(sflit + 8u * np);
    uint32_t *sna = sfl + 2u * np;   // [4][np]: na[] of each node slot (neighbour slot offsets by port)
    unsigned int *scnt = sna + 4u * np;
    unsigned int *shist = smem_hist ? scnt + NCOUNTERS : nullptr;
    __shared__ int s_abort;
    __shared__ uint32_t s_busy[2];
    // split cycle barrier (DESIGN 6.3), UR traffic only: there every warp has
    // routing-heavy cycles and a Phase 1 draw after the publish, which the
    // split lets overlap the other warps' routing (saturated 208x208 UR
    // -6 %); with LSPD's rare, heavy-tailed services it measured 3 % slower
    // than BAR.SYNC in the bench window (profiles/r02_ab_split_barrier.txt).
    // Not in drain launches (they reduce a busy flag over the whole cycle)
    // nor with the cluster exchange.
#ifdef NOC_NO_SPLIT_BAR
    constexpr bool SPLIT = false;
#else
    constexpr bool SPLIT = !DRAIN && !CL && MODE == 0u;
#endif
    __shared__ __align__(8) unsigned long long s_mbar;
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
    // a one-warp tile or a single-tile mesh keeps BAR.SYNC: without boundary
    // waits to overlap, the mbarrier round trip only costs (4x4: +9 %,
    // 16x16 in one CTA: +24 %)
    const bool split = SPLIT && blockDim.x > 32u && gridDim.x > 1u;

    const uint32_t i = threadIdx.x, lane = i & 31u;
    const TileShape T = tile_shape(S, tile);
    const RingMap RM = ring_map(T, blockDim.x);
    uint32_t lx = 0, lyy = 0;
    const bool active = tile_pos(T, RM, i, lx, lyy);

    {
        const uint32_t nsm = NCOUNTERS + (smem_hist ? 3u * S.nb : 0u);
        for (uint32_t k = i; k < nsm; k += blockDim.x) scnt[k] = 0u;
        if (i == 0) {
            s_abort = 0;
            s_busy[0] = s_busy[1] = 0u;
            if (split) mbar_init(mbar, blockDim.x / 32u);
        }
    }
    // shared-window addresses: flit slot d of node slot j at parity b is
    // fa + b*FSTR + (d*np + j)*16; its occupancy byte oa + b*OSTR + j*4 + d
    const uint32_t fa = (uint32_t)__cvta_generic_to_shared(sflit);
    const uint32_t oa = (uint32_t)__cvta_generic_to_shared(sfl);
    const uint32_t FSTR = 64u * np, OSTR = 4u * np;

    // ---- node registers (persist for the whole launch)
    NodeCtx c;
    c.x = T.x0 + lx;
    c.y = T.y0 + lyy;
    c.n = c.y * S.W + c.x;
    c.l = c.n - S.n0;
    c.head_ok = false;
    c.nd_ok = false;
    c.nd_t = 0u;
    c.nd_val = 0u;
    c.cold_loaded = true;
    c.q_dirty = c.hot_dirty = c.cold_dirty = false;
    c.busy_flit = false;
    uint32_t errf = 0;     // overflow flags seen by this thread (R32), reported once
    c.qctl = 0u;
    c.hot = 0u;
    c.cold = make_uint4(0, 0, 0, 0);
    uint32_t exist = 0;    // bit d: port d has a neighbour
    uint32_t ext = 0;      // bit d: port d crosses the tile boundary
    uint32_t intl = 0;     // bit d: port d exists inside the tile
    uint32_t na[4] = {0, 0, 0, 0};   // internal port p: neighbour's flit slot offset | occupancy byte offset << 16
    ExtIn ex[4] = {{NOPORT, 0, 0, false}, {NOPORT, 0, 0, false}, {NOPORT, 0, 0, false}, {NOPORT, 0, 0, false}};
    uint32_t nex = 0;
    c.deg = 0;
    const uint32_t b0 = (uint32_t)t0 & 1u;
    if (active) {
        c.qctl = S.fifo_ctl[c.l];
        if (MODE != 0u) {
            c.hot = S.core_hot[c.l];
            c.cold = S.core_cold[c.l];
        }
        if (q_count(c.qctl)) { c.head = fifo_of(S, c.l).p[q_head(c.qctl)]; c.head_ok = true; }
        exist = (c.y > 0 ? 1u : 0u) | (c.y + 1 < S.H ? 2u : 0u) | (c.x + 1 < S.W ? 4u : 0u) | (c.x > 0 ? 8u : 0u);
        ext = ((lyy == 0 ? 1u : 0u) | (lyy + 1 == T.th ? 2u : 0u) | (lx + 1 == T.tw ? 4u : 0u) |
               (lx == 0 ? 8u : 0u)) & exist;
        intl = exist & ~ext;
        c.deg = __popc(exist);
        const uint32_t bedge =
            ((c.y == S.row0 && c.y > 0) ? 1u : 0u) | ((c.y + 1 == S.row0 + S.rows && c.y + 1 < S.H) ? 2u : 0u);
#pragma unroll
        for (uint32_t d = 0; d < 4; ++d) {
            uint32_t m = c.l, mi = 0;
            switch (d) {
            case PN: m = c.l - S.W; if ((intl >> d) & 1u) mi = tile_slot(T, RM, lx, lyy - 1); break;
            case PS: m = c.l + S.W; if ((intl >> d) & 1u) mi = tile_slot(T, RM, lx, lyy + 1); break;
            case PE: m = c.l + 1u; if ((intl >> d) & 1u) mi = tile_slot(T, RM, lx + 1, lyy); break;
            default: m = c.l - 1u; if ((intl >> d) & 1u) mi = tile_slot(T, RM, lx - 1, lyy); break;
            }
            if ((intl >> d) & 1u) na[d] = (((d ^ 1u) * np + mi) * 16u) | ((mi * 4u + (d ^ 1u)) << 16);
            sna[d * np + i] = na[d];
            if (CL && ((ext >> d) & 1u)) {
                // the receiver's tile (= cluster rank) and its slot there
                const uint32_t vx = c.x + (d == PE ? 1u : 0u) - (d == PW ? 1u : 0u);
                const uint32_t vy = c.y + (d == PS ? 1u : 0u) - (d == PN ? 1u : 0u);
                const uint32_t rb = tile_of(vy - S.row0, S.rows, S.TY) * S.TX + tile_of(vx, S.W, S.TX);
                const TileShape R = tile_shape(S, rb);
                const uint32_t mr = tile_slot(R, ring_map(R, blockDim.x), vx - R.x0, vy - R.y0);
                ExtIn e;
                e.port = d;
                e.inw = rb;
                e.outw = (((d ^ 1u) * np + mr) * 16u) | ((mr * 4u + (d ^ 1u)) << 16);
                e.sys = false;
#pragma unroll
                for (uint32_t j = 0; j < 4; ++j)
                    if (j == nex) ex[j] = e;
                ++nex;
            } else if ((ext >> d) & 1u) {
                ExtIn e;
                e.port = d;
                e.inw = (uint32_t)ll_index(S, 0, d, c.l, 0);
                e.sys = (bedge >> d) & 1u;
                if (e.sys) {
                    // the receiver is in the neighbour band: its local index there
                    const uint32_t nr = S.nloc_nb[d];
                    const uint32_t lr = d == PN ? c.l - S.W + nr : c.l + S.W - S.nloc;
                    e.outw = (uint32_t)(((size_t)(d ^ 1u) * nr + lr) * 4u);
                } else {
                    e.outw = (uint32_t)ll_index(S, 0, d ^ 1u, m, 0);
                }
#pragma unroll
                for (uint32_t j = 0; j < 4; ++j)
                    if (j == nex) ex[j] = e;
                ++nex;
            }
        }
        // internal inputs of cycle t0 (spilled by the previous launch)
        const uint32_t fl = S.flag[b0][c.l];
        const uint8_t s0 = stamp_of(t0);
        uint32_t occ = 0;
#pragma unroll
        for (uint32_t d = 0; d < 4; ++d) {
            if ((((CL ? exist : intl) >> d) & 1u) && ((fl >> (8u * d)) & 0xFFu) == s0) {
                sflit[(b0 * 4u + d) * np + i] = S.flit[b0][flit_at(S.nloc, d, c.l)];
                occ |= 1u << (8u * d);
            }
        }
        sfl[b0 * np + i] = occ;
        sfl[(b0 ^ 1u) * np + i] = 0u;
    }

    // Draw window (LSPD): bit k of wmask = the draw of cycle wbase+k fires.
    // Lanes that need a window for cycle tn (idle, or possibly idle by then)
    // get one: the warp evaluates the 32 draws of one requester at a time.
    uint32_t wbase = (uint32_t)t0 - 64u, wmask = 0u;
    auto refresh = [&](bool need, uint64_t tn) {
        uint32_t nm = __ballot_sync(FULL, need);
        while (nm) {
            const uint32_t j = __ffs(nm) - 1u;
            nm &= nm - 1u;
            const uint32_t nj = __shfl_sync(FULL, c.n, j);
            const uint64_t tk = tn + lane;
            uint32_t r[4];
            philox4x32_10(S.seed_lo, S.seed_hi, nj, (uint32_t)tk, (uint32_t)(tk >> 32), 0u, r);
            const uint32_t m = __ballot_sync(FULL, r[0] < S.thr_inj);
            const uint32_t src = m ? __ffs(m) - 1u : 0u;
            const uint32_t r1 = __shfl_sync(FULL, r[1], src);
            const uint32_t r2 = __shfl_sync(FULL, r[2], src);
            const uint32_t r3 = __shfl_sync(FULL, r[3], src);
            if (lane == j) {
                wbase = (uint32_t)tn;
                wmask = m;
                c.nd_ok = m != 0u;
                if (m) {
                    c.nd_t = (uint32_t)tn + src;
                    c.nd_val = draw_value(S, c.n, r1, r2, r3);
                    prefetch_l1(set_ptr(S, c, c.nd_val));
                }
            }
        }
    };
    const bool windows = MODE != 0u && S.gen && !S.has_script;
    // windows for cycle tn: idle cores and cores whose wait expires at tn
    auto need_window = [&](uint64_t tn) {
        if (!active) return false;
        const uint32_t mode = core_mode(c.hot);
        const bool expiring = (mode == ML2WAIT || mode == MMEMWAIT) && (((c.hot ^ (uint32_t)tn) & 0x1FFFFFFFu) == 0u);
        if (expiring && mode == MMEMWAIT && (c.cold.w & 3u)) prefetch_l1(set_ptr(S, c, c.cold.z));
        return (mode == MIDLE || expiring) && (uint32_t)tn - wbase >= 32u;
    };
    // LSPD with draw windows: Phase 1 of a node has work only at its next due
    // cycle `wake` -- its timer expiry (L2 hit, memory fill, L1 miss), the next
    // firing draw of its window while IDLE, or the window's end (refresh) --
    // or in the cycle after a Phase-3 state change.  Other cycles skip it.
    uint32_t wake = 0;
    auto wake_from = [&](uint32_t tc) -> uint32_t {   // next due cycle after tc
        const uint32_t mode = core_mode(c.hot);
        if (mode == MIDLE) {
            const uint32_t k = tc + 1u - wbase;
            if (k >= 32u) return tc + 1u;
            const uint32_t m = wmask >> k;
            return m ? tc + (uint32_t)__ffs(m) : wbase + 32u;
        }
        if (mode == MWAITDIR || mode == MWAITDATA || mode == MMEMFETCH) return tc;   // woken by Phase 3 only
        return tc + ((c.hot - tc) & 0x1FFFFFFFu);                // the timer (ready mod 2^29)
    };
    const uint32_t pstride = 16u * S.nloc;
    Sink K{scnt, shist, true};
    Acc acc = {0, 0, 0, 0};
    const uint32_t own_f = fa + i * 16u, own_o = oa + i * 4u;
    const ExtIn &e0 = ex[0], &e1 = ex[1];

    // Cycle order (DESIGN 6.3): Phase 1 of cycle t runs at the END of cycle
    // t-1 (after its Phase 2 and 3; it reads only node-local state and the
    // draw of (n, t)), so a cycle starts directly with the latch and the
    // routing, and the boundary outputs -- the critical path of the
    // neighbouring tiles -- are published first.  The boundary polls of cycle
    // t+1 are issued right after cycle t's outputs are published, so their
    // latency overlaps the rest of cycle t (Phase 3, Phase 1 of t+1, the
    // barrier).  Phase 1 of the first cycle runs in the prologue.
    unsigned long long a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0w = 0, b1w = 0, b2w = 0, b3w = 0;
    if (!CL && active && ext) {
        const unsigned long long *const llp = S.ll + (size_t)b0 * pstride;
        ll_load2(e0.sys, llp + e0.inw, a0, a1);
        ll_load2(e0.sys, llp + e0.inw + 2, a2, a3);
        if (e1.port != NOPORT) {
            ll_load2(e1.sys, llp + e1.inw, b0w, b1w);
            ll_load2(e1.sys, llp + e1.inw + 2, b2w, b3w);
        }
    }
    if (windows) refresh(need_window(t0), t0);
    if (active) {
        if (MODE == 0u) phase1_ur(S, K, c, t0);
        else phase1_lspd_win<MODE == 2u>(S, K, c, t0, wbase, wmask);
        if (windows) wake = wake_from((uint32_t)t0);
    }
    // cluster exchange: every CTA's slots are initialised before any remote store
    if (CL) cluster_barrier();
    else __syncthreads();

    for (uint32_t cc = 0; cc < ncyc; ++cc) {
        const uint64_t t = t0 + cc;
        const uint32_t pb = (uint32_t)t & 1u, nb1 = pb ^ 1u;
        const uint32_t st = (uint32_t)t, stn = st + 1u;
        const bool last = cc + 1u == ncyc;
        bool busy = false;
        // split barrier: every warp's link stores of cycle t-1 are visible
        if (split && cc > 0u) {
            mbar_wait(mbar, (cc - 1u) & 1u);
            if (s_abort) break;
        }
        TRACE_DECL
        Flit gej = Flit{0, 0, 0, 0};   // the flit ejected this cycle (<= 1)
        bool ej = false;
        uint32_t usedo = 0;
        if (active) {
            const unsigned long long *const llp = S.ll + (size_t)pb * pstride;   // this cycle's boundary inputs
            // (1) latch.  Slots 0..3 = link inputs N,S,E,W,
            // slot 4 = the injection register.  The occupancy word
            // is consumed (cleared) here.
            const uint32_t ow = own_o + pb * OSTR;
            const uint32_t occ = lds32(ow);
            sts32_if(occ != 0u, ow, 0u);
            uint32_t present = ((occ & 0x01010101u) * 0x01020408u) >> 24;   // byte d -> bit d
            const uint32_t fw = own_f + pb * FSTR;
            // boundary inputs: the polls were issued at the end of the previous
            // cycle; re-poll until each cross-tile slot is complete for cycle t
            // (word 0 carries stamp t and, for a flit rather than EMPTY, so do
            // words 1..3); a flit is parked in the node's own shared slot so
            // all four link inputs are latched alike below
            if (!CL && ext) {
                bool w0 = true, w1 = e1.port != NOPORT, w2 = ex[2].port != NOPORT, w3 = ex[3].port != NOPORT;
                uint32_t spins = 0;
                while (true) {
#pragma unroll
                    for (uint32_t j = 2; j < 4; ++j) {
                        bool &wj = j == 2 ? w2 : w3;
                        if (!wj) continue;
                        unsigned long long c0, c1, c2, c3;
                        ll_load2(ex[j].sys, llp + ex[j].inw, c0, c1);
                        ll_load2(ex[j].sys, llp + ex[j].inw + 2, c2, c3);
                        if ((uint32_t)c0 != st) continue;
                        const uint32_t x = (uint32_t)(c0 >> 32);
                        if (x == LL_EMPTY) wj = false;
                        else if ((uint32_t)c1 == st && (uint32_t)c2 == st && (uint32_t)c3 == st) {
                            wj = false;
                            sts128_if(true, fw + ex[j].port * 16u * np,
                                      Flit{x, (uint32_t)(c1 >> 32), (uint32_t)(c2 >> 32), (uint32_t)(c3 >> 32)});
                            present |= 1u << ex[j].port;
                        }
                    }
                    if (w0 && (uint32_t)a0 == st) {
                        const uint32_t x = (uint32_t)(a0 >> 32);
                        if (x == LL_EMPTY) w0 = false;
                        else if ((uint32_t)a1 == st && (uint32_t)a2 == st && (uint32_t)a3 == st) {
                            w0 = false;
                            sts128_if(true, fw + e0.port * 16u * np,
                                      Flit{x, (uint32_t)(a1 >> 32), (uint32_t)(a2 >> 32), (uint32_t)(a3 >> 32)});
                            present |= 1u << e0.port;
                        }
                    }
                    if (w1 && (uint32_t)b0w == st) {
                        const uint32_t x = (uint32_t)(b0w >> 32);
                        if (x == LL_EMPTY) w1 = false;
                        else if ((uint32_t)b1w == st && (uint32_t)b2w == st && (uint32_t)b3w == st) {
                            w1 = false;
                            sts128_if(true, fw + e1.port * 16u * np,
                                      Flit{x, (uint32_t)(b1w >> 32), (uint32_t)(b2w >> 32), (uint32_t)(b3w >> 32)});
                            present |= 1u << e1.port;
                        }
                    }
                    if (!(w0 || w1 || w2 || w3)) break;
                    if (++spins > (1u << 22)) { atomicOr(S.err, 0x80000000u); s_abort = 1; break; }
                    if (w0) {
                        ll_load2(e0.sys, llp + e0.inw, a0, a1);
                        ll_load2(e0.sys, llp + e0.inw + 2, a2, a3);
                    }
                    if (w1) {
                        ll_load2(e1.sys, llp + e1.inw, b0w, b1w);
                        ll_load2(e1.sys, llp + e1.inw + 2, b2w, b3w);
                    }
                }
            }
            TRACE_EXT_DONE
            Flit f[5];
#pragma unroll
            for (uint32_t d = 0; d < 5; ++d) f[d] = Flit{0, 0, 0, 0};
#pragma unroll
            for (uint32_t d = 0; d < 4; ++d) lds128_if((present >> d) & 1u, fw + d * 16u * np, f[d]);
            // NEXT-f4 (FEAT bit 1): injection mode 1 (R43), an ejecting flit
            // frees its port; mode 2 (R53), queued flits fill every free input
            // slot (the empty link slots; ranking ties: sec_key)
            const bool fill_all = (FEAT & 2u) && S.inject_mode == 2u;
            if (fill_all) {
#pragma unroll
                for (uint32_t d = 0; d < 4; ++d)
                    if (!((present >> d) & 1u) && inject_flit(S, c, (uint32_t)__popc(present), t, acc, f[d]))
                        present |= 1u << d;
            } else {
                uint32_t frees = 0u;
                if (FEAT & 2u)
#pragma unroll
                    for (uint32_t d = 0; d < 4; ++d) frees |= ((present >> d) & 1u) && f_dst(f[d]) == c.n;
                if (inject_flit(S, c, (uint32_t)__popc(present), t, acc, f[4], frees)) present |= 16u;
            }
            TRACE_EV(((present & 16u) ? 32u : 0u) | (present ? 64u : 0u) | (ext ? 128u : 0u));

            // (2) first choices (eject at the destination, else x-port, else
            // y-port: PMDR).  If they are pairwise distinct every flit
            // takes its first choice whatever the ranking.  port[k] in
            // `ports` nibble k; inv nibble p = the slot routed to port p
            // (p = 4: the ejected flit)
            uint32_t seen = 0, coll = 0, ports = 0, inv = 0;
#pragma unroll
            for (uint32_t k = 0; k < 5; ++k) {
                const uint32_t pk = (present >> k) & 1u;
                const uint32_t fc = first_port(f_dst(f[k]), c.n, c.x, c.y, S.W, S.wmagic);
                const uint32_t b = pk << fc;
                coll |= seen & b;
                seen |= b;
                ports |= fc << (4u * k);
                inv |= pk ? k << (4u * fc) : 0u;
            }
            // R32 lifetime limit: a flit's lifetime only grows, so it is checked
            // where a flit leaves the tile's registers for good -- at ejection,
            // at a cross-tile hop and at the end of the launch (spill) -- which
            // flags every overflow by the end of the run, as the oracle does
            uint32_t used = seen & 15u;
            bool has_ej = (seen >> PX) & 1u;
            TRACE_EV(coll ? 16u : 0u);
            if (coll) {
                // two flits want the same port: rank them ("Priority Sort",
                // P:L129; R1, R2) and let each take, in rank order, the eject
                // link if at its destination and still free, else its first
                // free productive port, else the first free existing port in
                // N,S,E,W with age+1 (R3-R6).
                // The injected flit (lowest age, lifetime 0) always ranks last.
                uint64_t key[4];
                uint64_t prefs = 0;
#pragma unroll
                for (uint32_t k = 0; k < 5; ++k) {
                    const uint32_t dst = f_dst(f[k]);
                    const uint32_t dy = row_of(S, dst), dx = dst - dy * S.W;
                    const uint32_t xp = dx > c.x ? PE : PW, yp = dy > c.y ? PS : PN;
                    const uint32_t pw = dst == c.n ? 1u
                                                   : ((dx != c.x ? 2u | (xp << 2) : 0u) |
                                                      (dy != c.y && ((FEAT & 1u) == 0u || dx == c.x) ? 16u | (yp << 5) : 0u));
                    prefs |= (uint64_t)pw << (8u * k);
                    if (k < 4) {
                        const uint32_t life = st - f[k].z;
                        key[k] = ((uint64_t)(life > LIFE_MAX ? LIFE_MAX : life) << 21) | (NODE_MASK - f_src(f[k]));
                        if (S.prio == 0u) key[k] |= (uint64_t)f_age(f[k]) << 48;
                        if (!((present >> k) & 1u)) key[k] = 0ull;
                    }
                }
                uint32_t rk[4] = {0, 0, 0, 0};
#pragma unroll
                for (uint32_t a = 0; a < 4; ++a)
#pragma unroll
                    for (uint32_t b = a + 1; b < 4; ++b) {
                        // equal keys only under fill-all (flits one node injected
                        // together): the smaller secondary key ranks first (R53)
                        const bool first = (FEAT & 2u) && key[a] == key[b] && key[a] != 0ull
                                               ? sec_key(f[a]) < sec_key(f[b]) : key[a] > key[b];
                        if (first) ++rk[b];
                        else ++rk[a];
                    }
                uint32_t ord = 4u << 16;
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k) ord |= k << (4u * rk[k]);
                used = 0;
                ports = 0;
                inv = 0;
                has_ej = false;
                uint32_t dm = 0;
#pragma unroll
                for (uint32_t r = 0; r < 5; ++r) {
                    const uint32_t k = (ord >> (4u * r)) & 15u;
                    if (!((present >> k) & 1u)) continue;
                    const uint32_t pw = (uint32_t)(prefs >> (8u * k)) & 0xFFu;
                    const uint32_t xp = (pw >> 2) & 3u, yp = (pw >> 5) & 3u;
                    uint32_t p;
                    if ((pw & 1u) && !has_ej) {
                        has_ej = true;
                        p = PX;
                    } else {
                        if ((pw & 2u) && !((used >> xp) & 1u)) p = xp;
                        else if ((pw & 16u) && !((used >> yp) & 1u)) p = yp;
                        else { p = defl_port(exist & ~used, FEAT & 1u); dm |= 1u << k; }
                        used |= 1u << p;
                    }
                    ports |= p << (4u * k);
                    inv |= k << (4u * p);
                }
                // P:L116 age increment of the deflected flits
#pragma unroll
                for (uint32_t k = 0; k < 5; ++k) {
                    if (!((dm >> k) & 1u)) continue;
                    uint32_t a = f_age(f[k]) + 1u;
                    if (a > AGE_MAX) { errf |= ERR_AGE; a = AGE_MAX; }
                    f_set_age(f[k], a);
                }
                acc.defl += __popc(dm);
            }
            acc.hops += __popc(used);
            // (3) outputs across the tile boundary first: they are on the
            // critical path of the neighbouring tiles.  A routed flit, else an
            // explicit EMPTY, on every boundary port every cycle.  Then the
            // polls of the next cycle's boundary inputs.
            if (CL && ext) {
                // cluster exchange: a routed flit goes straight into the
                // receiving CTA's slot of cycle t+1 (no EMPTY words needed)
#pragma unroll
                for (uint32_t j = 0; j < 4; ++j) {
                    const ExtIn &e = ex[j];
                    if (e.port == NOPORT || !((used >> e.port) & 1u)) continue;
                    const Flit g = pick5(f, (inv >> (4u * e.port)) & 15u);
                    if (st - g.z > LIFE_MAX) errf |= ERR_AGE;   // R32, at a cross-tile hop
                    st_cluster_v4(mapa_rank(fa + nb1 * FSTR + (e.outw & 0xFFFFu), e.inw), g);
                    st_cluster_u8(mapa_rank(oa + nb1 * OSTR + (e.outw >> 16), e.inw));
                }
            } else if (ext) {
#pragma unroll
                for (uint32_t j = 0; j < 4; ++j) {
                    const ExtIn &e = ex[j];
                    if (e.port == NOPORT) continue;
                    unsigned long long *o = ll_out(S, e.sys, e.port, nb1, pstride) + e.outw;
                    if ((used >> e.port) & 1u) {
                        const Flit g = pick5(f, (inv >> (4u * e.port)) & 15u);
                        if (st - g.z > LIFE_MAX) errf |= ERR_AGE;   // R32, at a cross-tile hop
                        ll_store2(e.sys, o + 2, llw(stn, g.z), llw(stn, g.w));
                        ll_store2(e.sys, o, llw(stn, g.x), llw(stn, g.y));
                    } else {
                        ll_store1(e.sys, o, llw(stn, LL_EMPTY));
                    }
                }
                if (!last) {
                    const unsigned long long *const lln = S.ll + (size_t)nb1 * pstride;
                    ll_load2(e0.sys, lln + e0.inw, a0, a1);
                    ll_load2(e0.sys, lln + e0.inw + 2, a2, a3);
                    if (e1.port != NOPORT) {
                        ll_load2(e1.sys, lln + e1.inw, b0w, b1w);
                        ll_load2(e1.sys, lln + e1.inw + 2, b2w, b3w);
                    }
                }
            }
            TRACE_PUB_DONE
            // (4) flits that stay in the tile: predicated shared-memory stores
            // into the neighbour's slot opp(p) of cycle t+1
            if (used & intl) {
                const uint32_t nf = fa + nb1 * FSTR, no = oa + nb1 * OSTR;
#pragma unroll
                for (uint32_t k = 0; k < 5; ++k) {
                    const uint32_t p = (ports >> (4u * k)) & 15u;
                    const bool go = ((present >> k) & 1u) && p < 4u && ((intl >> p) & 1u);
                    const uint32_t w = sna[(p & 3u) * np + i];   // a shared load instead of a select chain
                    sts128_if(go, nf + (w & 0xFFFFu), f[k]);
                    sts8_if(go, no + (w >> 16));
                }
            }
            if (has_ej) {
                gej = pick5(f, (inv >> 16) & 15u);
                ej = true;
            }
            usedo = used;
        }
        // split barrier: this warp's link stores of cycle t are done.  What
        // follows (Phase 3 of t, Phase 1 of t+1) is node-local, so it
        // overlaps the other warps' routing and the boundary-input latency
        // instead of extending every warp's cycle
        if (split) {
            __syncwarp();
            if (lane == 0u) mbar_arrive(mbar);
        }
        if (active) {
            // (5) Phase 3: the ejected flit (<= 1) is delivered and
            // serviced now, after this cycle's outputs are out
            if (ej) {
                if (st - gej.z > LIFE_MAX) errf |= ERR_AGE;   // R32
                TRACE_EV(1u);
                phase3(S, K, c, gej, t, acc);
                if (windows) wake = wake_from(st);
            }
            if (DRAIN) busy = usedo != 0u || q_count(c.qctl) > 0u || core_mode(c.hot) != MIDLE;
        }
        TRACE_P3_DONE
        // (6) Phase 1 of cycle t+1, after the draw windows it needs
        if (!last) {
            if (windows) {
                const bool due = active && stn == wake;
                const bool need = due && stn - wbase >= 32u;
                // the set a memory fill installs into one cycle ahead (L1 prefetch)
                if (active && stn + 1u == wake && core_mode(c.hot) == MMEMWAIT && (c.cold.w & 3u))
                    prefetch_l1(set_ptr(S, c, c.cold.z));
                if (__any_sync(FULL, need)) {
                    TRACE_EV(8u);
                    refresh(need, t + 1);
                }
                if (due) {
                    const uint32_t h0 = c.hot, q0 = c.qctl;
                    phase1_lspd_win<MODE == 2u>(S, K, c, t + 1, wbase, wmask);
                    wake = wake_from(stn);
                    TRACE_EV((c.hot != h0 ? 2u : 0u) | (c.qctl != q0 ? 4u : 0u));
                }
            } else if (active) {
                const uint32_t h0 = c.hot, q0 = c.qctl;
                if (MODE == 0u) phase1_ur(S, K, c, t + 1);
                else phase1_lspd_win<MODE == 2u>(S, K, c, t + 1, wbase, wmask);
                TRACE_EV((c.hot != h0 ? 2u : 0u) | (c.qctl != q0 ? 4u : 0u));
            }
        }
        TRACE_P1_DONE
        TRACE_END
        // The cycle barrier is a full BAR.SYNC: it orders this cycle's shared-
        // memory link stores before the next cycle's loads.
        if (DRAIN && busy) s_busy[cc & 1u] = cc + 1u;
        if (CL) cluster_barrier();
        else if (!split) __syncthreads();
        if (DRAIN && i == 0 && s_busy[cc & 1u] == cc + 1u) atomicAdd(&activity[cc], 1u);
        if (!split && s_abort) break;
    }
    // the last cycle's link stores of every warp before the spill reads them
    if (split) __syncthreads();

    // ---- epilogue: spill state
    const uint64_t tend = t0 + ncyc;
    if (active) {
        S.fifo_ctl[c.l] = c.qctl;
        if (MODE != 0u) {
            S.core_hot[c.l] = c.hot;
            S.core_cold[c.l] = c.cold;
        }
        const uint32_t be = (uint32_t)tend & 1u;
        const uint8_t ste = stamp_of(tend);
        const uint32_t occ = sfl[be * np + i];
        uint32_t gfl = 0;
#pragma unroll
        for (uint32_t d = 0; d < 4; ++d) {
            if ((((CL ? exist : intl) >> d) & 1u) && ((occ >> (8u * d)) & 0xFFu)) {
                const uint4 v = sflit[(be * 4u + d) * np + i];
                if ((uint32_t)tend - v.z > LIFE_MAX) errf |= ERR_AGE;   // R32
                S.flit[be][flit_at(S.nloc, d, c.l)] = v;
                gfl |= (uint32_t)ste << (8u * d);
            }
        }
        S.flag[be][c.l] = gfl;
        if (errf) atomicOr(S.err, errf);
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

}  // namespace noc
