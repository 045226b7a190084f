// node_logic.cuh -- the per-cycle, per-node step as
// device functions, shared by every engine (per-cycle launches, persistent
// kernels).  One CUDA thread advances one node through Phase 1 (core step,
// P:L257), Phase 2 (rank + port assignment / deflection) and
// Phase 3 (eject, reassembly, directory / L2 service, Fig. 4)
// of cycle t.  All cross-node communication goes through the double-buffered
// link slots of cycle t+1; everything else a node touches is owned by it
// (SURVEY 8(c.5)), so no atomics touch the datapath: atomics are used only for
// the order-independent statistics.
#pragma once
#include "common.cuh"

namespace noc {

// Statistic sink.  Rare counters / histogram bins go to shared memory (u32)
// when the kernel provides it, else straight to global u64 atomics.
// When a node's state is replicated across several lanes (TILED engine), every
// lane executes the same model code and performs the same (idempotent) global
// stores; only the lead lane (on = true) counts.
struct Sink {
    unsigned int *scnt;    // [NCOUNTERS] or nullptr
    unsigned int *shist;   // [3][nb] or nullptr
    bool on;
    __device__ __forceinline__ void cnt(const Dev &S, uint32_t i, uint32_t v = 1u) const
    {
        if (!on) return;
        if (scnt) atomicAdd(&scnt[i], v);
        else atomicAdd(&S.cnt[i], (unsigned long long)v);
    }
    __device__ __forceinline__ void hist(const Dev &S, uint32_t h, uint32_t v) const
    {
        if (!on) return;
        uint32_t b = v < S.nb - 1u ? v : S.nb - 1u;
        if (shist) atomicAdd(&shist[h * S.nb + b], 1u);
        else atomicAdd(&S.hist[(size_t)h * S.nb + b], 1ull);
    }
};

// Hot counters accumulated in registers and reduced once per launch.
struct Acc {
    uint32_t injected, ejected, hops, defl;
};

// Registers of one node for one cycle.
struct NodeCtx {
    uint32_t l, n, x, y;
    uint32_t deg;        // number of existing neighbours (router degree)
    uint32_t qctl;
    uint32_t hot;
    uint4 cold;
    uint2 head;          // cached head packet of the send FIFO (valid iff head_ok)
    bool head_ok;
    // generation draw computed one cycle ahead (valid iff nd_ok and nd_t == t)
    bool nd_ok, nd_fire;
    uint32_t nd_t, nd_val;
    bool q_dirty, hot_dirty, cold_dirty, cold_loaded;
    bool busy_flit;      // sent a flit this cycle (drain detection)
};

__device__ __forceinline__ void load_cold(const Dev &S, NodeCtx &c)
{
    if (!c.cold_loaded) { c.cold = S.core_cold[c.l]; c.cold_loaded = true; }
}

__device__ __forceinline__ void set_mode(NodeCtx &c, uint32_t mode, uint64_t ready)
{
    c.hot = (mode << 29) | ((uint32_t)ready & 0x1FFFFFFFu);
    c.hot_dirty = true;
}

// ENQ (DESIGN 3.3; bounded send FIFO, R21)
__device__ __forceinline__ void enq(const Dev &S, const Sink &K, NodeCtx &c, uint32_t kind, uint32_t dst,
                                    uint32_t payload, uint32_t nfl)
{
    uint32_t h = q_head(c.qctl), cnt = q_count(c.qctl);
    if (cnt == S.qcap) {
        K.cnt(S, C_DROPS + kind);
        // R21: in LSPD mode a dropped protocol message would leave a core or a
        // directory entry waiting for ever, so the run is invalid: poison it
        if (S.mode != 0u) atomicOr(S.err, ERR_DROP);
        return;
    }
    uint32_t slot = (h + cnt) & (S.qcap - 1u);
    const uint2 pkt = make_uint2(dst | (kind << 21) | (nfl << 24), payload);
    S.fifo_pkt[(size_t)c.l * S.qcap + slot] = pkt;
    if (cnt == 0u) { c.head = pkt; c.head_ok = true; }
    c.qctl = q_make(h, cnt + 1u, q_next(c.qctl));
    c.q_dirty = true;
    K.cnt(S, C_ENQ);
}

// Home node of tag T: T mod N (distributed, R12), or the one directory node
// (centralized, the paper's location array; R40)
__device__ __forceinline__ uint32_t home_of(const Dev &S, uint32_t T)
{
    return S.dir_mode ? S.dir_node : T % S.N;
}

// Entry of tag T in this band's part of the location array (only called at
// T's home): distributed = [T / N][home - n0]; centralized = [T] in the band of
// the directory node
__device__ __forceinline__ size_t loc_index(const Dev &S, uint32_t T)
{
    if (S.dir_mode) return T;
    uint32_t q = T / S.N, h = T - q * S.N;
    return (size_t)q * S.nloc + (h - S.n0);
}

// L2HIT: stamp update on a hit (R23)
__device__ __forceinline__ bool l2_hit(const Dev &S, const NodeCtx &c, uint32_t T, uint64_t t)
{
    uint32_t set = T % S.sets;
    uint4 *L = S.l2 + ((size_t)c.l * S.sets + set) * S.ways;
    for (uint32_t w = 0; w < S.ways; ++w) {
        uint4 v = L[w];
        if (v.x == T + 1u) {
            L[w] = make_uint4(v.x, (uint32_t)t, (uint32_t)(t >> 32), 0u);
            return true;
        }
    }
    return false;
}

// EVHANDLER at home (R13)
__device__ __forceinline__ void ev_handler(const Dev &S, const Sink &K, uint32_t T, uint32_t src)
{
    size_t i = loc_index(S, T);
    uint32_t e = S.loc[i];
    uint32_t h1 = e & HOLDER_MASK, pend = e >> HOLDER_BITS;
    if (h1 != src + 1u) atomicOr(S.err, ERR_EVHOLDER);
    if (pend > 0) --pend;
    else h1 = 0;
    S.loc[i] = h1 | (pend << HOLDER_BITS);
    K.cnt(S, C_EVRCVD);
}

// INSTALL (victim: first invalid, else min stamp, ties lowest way, R23)
static __device__ void install(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint64_t t)
{
    uint32_t set = T % S.sets;
    uint4 *L = S.l2 + ((size_t)c.l * S.sets + set) * S.ways;
    uint32_t victim = 0;
    uint64_t best = ~0ull;
    bool found_invalid = false;
    uint4 vline = make_uint4(0, 0, 0, 0);
    for (uint32_t w = 0; w < S.ways; ++w) {
        uint4 v = L[w];
        if (v.x == 0u) {
            if (!found_invalid) { victim = w; vline = v; found_invalid = true; }
        } else if (!found_invalid) {
            uint64_t st = ((uint64_t)v.z << 32) | v.y;
            if (st < best) { best = st; victim = w; vline = v; }
        }
    }
    if (vline.x != 0u) {
        uint32_t V = vline.x - 1u;
        uint32_t hv = home_of(S, V);
        K.cnt(S, C_EVICTIONS);
        K.cnt(S, C_EVSENT);
        if (hv == c.n) ev_handler(S, K, V, c.n);
        else enq(S, K, c, KEV, hv, V, 1u);
    }
    L[victim] = make_uint4(T + 1u, (uint32_t)t, (uint32_t)(t >> 32), 0u);
    K.cnt(S, C_INSTALLS);
}

// ---------------------------------------------------------------------------
// Private write-through L1 (NEXT-f1, R42): LRU like L2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool l1_hit(const Dev &S, const NodeCtx &c, uint32_t T, uint64_t t)
{
    uint4 *L = S.l1 + ((size_t)c.l * S.l1_sets + T % S.l1_sets) * S.l1_ways;
    for (uint32_t w = 0; w < S.l1_ways; ++w) {
        const uint4 v = L[w];
        if (v.x == T + 1u) {
            L[w] = make_uint4(v.x, (uint32_t)t, (uint32_t)(t >> 32), v.w);
            return true;
        }
    }
    return false;
}

// Fill block T supplied by `owner`'s slice; the victim is written back to the
// slice that supplied it (1-flit EV with WB_BIT), absorbed when that is ours.
static __device__ void l1_fill(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint32_t owner, uint64_t t);

__device__ __forceinline__ void complete(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t)
{
    load_cold(S, c);
    uint64_t start = ((uint64_t)c.cold.y << 32) | c.cold.x;
    uint64_t lat = t - start;
    K.hist(S, 2, lat > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)lat);
    K.cnt(S, C_COMPLETED);
    set_mode(c, MIDLE, 0);
}

__device__ __forceinline__ void receive_ndr(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t)
{
    if (core_mode(c.hot) != MWAITDIR) atomicOr(S.err, ERR_PROTO);
    K.cnt(S, C_MEMREQ);
    load_cold(S, c);
    c.cold.w = (c.cold.w & ~1u) | 1u;          // install = 1
    c.cold_dirty = true;
    set_mode(c, MMEMWAIT, t + S.mem_lat);
}

__device__ __forceinline__ void receive_dr(const Dev &S, const Sink &K, NodeCtx &c, uint32_t holder)
{
    if (core_mode(c.hot) != MWAITDIR) atomicOr(S.err, ERR_PROTO);
    K.cnt(S, C_REQMADE);
    load_cold(S, c);
    enq(S, K, c, KRQ, holder, c.cold.z, 1u);
    set_mode(c, MWAITDATA, 0);
}

static __device__ void l1_fill(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint32_t owner, uint64_t t)
{
    if (!S.l1_sets) return;
    uint4 *L = S.l1 + ((size_t)c.l * S.l1_sets + T % S.l1_sets) * S.l1_ways;
    uint32_t victim = 0;
    uint64_t best = ~0ull;
    bool found_invalid = false;
    uint4 vline = make_uint4(0, 0, 0, 0);
    for (uint32_t w = 0; w < S.l1_ways; ++w) {
        const uint4 v = L[w];
        if (v.x == 0u) {
            if (!found_invalid) { victim = w; vline = v; found_invalid = true; }
        } else if (!found_invalid) {
            const uint64_t st = ((uint64_t)v.z << 32) | v.y;
            if (st < best) { best = st; victim = w; vline = v; }
        }
    }
    if (vline.x != 0u) {
        K.cnt(S, C_WBSENT);
        if (vline.w == c.n) K.cnt(S, C_WBRCVD);
        else enq(S, K, c, KEV, vline.w, (vline.x - 1u) | WB_BIT, 1u);
    }
    L[victim] = make_uint4(T + 1u, (uint32_t)t, (uint32_t)(t >> 32), owner);
}

// DIRSERVICE at home c.n for requester r (Fig. 4 steps 1-2; R12-R14, R28)
static __device__ void dir_service(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint32_t r, uint64_t t)
{
    K.cnt(S, C_DIRSEARCH);
    size_t i = loc_index(S, T);
    uint32_t e = S.loc[i];
    uint32_t h1 = e & HOLDER_MASK, pend = e >> HOLDER_BITS;
    uint32_t kind, payload;
    if (h1 == 0u) {
        h1 = r + 1u; kind = KNDR; payload = T;
    } else if (h1 == r + 1u) {
        ++pend;
        if (pend > PEND_MAX) { atomicOr(S.err, ERR_PEND); pend = PEND_MAX; }
        kind = KNDR; payload = T;
    } else {
        kind = KDR; payload = h1 - 1u;
    }
    S.loc[i] = h1 | (pend << HOLDER_BITS);
    if (r == c.n) {
        if (kind == KNDR) receive_ndr(S, K, c, t);
        else receive_dr(S, K, c, payload);
    } else {
        enq(S, K, c, kind, r, payload, 1u);
    }
}

// The local L2 part of an access (Fig. 4): hit, else the directory
static __device__ void l2_access(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint64_t t)
{
    if (l2_hit(S, c, T, t)) {
        K.cnt(S, C_L2HIT);
        if (S.l2_hit_lat == 0u) {
            l1_fill(S, K, c, T, c.n, t);
            complete(S, K, c, t);
        } else {
            set_mode(c, ML2WAIT, t + S.l2_hit_lat);
        }
    } else {
        K.cnt(S, C_L2MISS);
        set_mode(c, MWAITDIR, 0);
        uint32_t h = home_of(S, T);
        if (h == c.n) dir_service(S, K, c, T, c.n, t);
        else enq(S, K, c, KDA, h, T, 1u);
    }
}

// A new access (Phase 1; R19): the L1 first when there is one (a hit
// is served at once; a miss waits the L1 miss cycles, then the local L2)
static __device__ void start_access(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint64_t t)
{
    load_cold(S, c);
    c.cold = make_uint4((uint32_t)t, (uint32_t)(t >> 32), T, 0u);   // start, tag, install 0, rx 0
    c.cold_dirty = true;
    K.cnt(S, C_ACCESSES);
    if (S.l1_sets) {
        if (l1_hit(S, c, T, t)) {
            K.cnt(S, C_L1HIT);
            complete(S, K, c, t);
        } else {
            K.cnt(S, C_L1MISS);
            set_mode(c, ML1WAIT, t + S.l1_miss_lat);
        }
        return;
    }
    l2_access(S, K, c, T, t);
}

// Next due script event (DESIGN 3.3).  Returns true and the value if one is consumed.
__device__ __forceinline__ bool script_next(const Dev &S, const NodeCtx &c, uint64_t t, uint32_t &value)
{
    uint32_t off = S.script_off[c.l], end = S.script_off[c.l + 1];
    uint32_t pos = S.script_pos[c.l];
    if (off + pos >= end) return false;
    uint4 ev = S.script[off + pos];
    uint64_t cyc = ((uint64_t)ev.y << 32) | ev.x;
    if (cyc > t) return false;
    value = ev.z;
    S.script_pos[c.l] = pos + 1u;
    return true;
}

// ---------------------------------------------------------------------------
// Phase 1
// ---------------------------------------------------------------------------
// The Philox draw of node n for cycle t (R25): fire flag and value (UR: probe
// destination; LSPD: block tag, DESIGN 3.3).
// The value of a firing draw r1..r3 of node n (UR: probe destination; LSPD:
// block tag, DESIGN 3.3)
__device__ __forceinline__ uint32_t draw_value(const Dev &S, uint32_t n, uint32_t r1, uint32_t r2, uint32_t r3)
{
    if (S.mode == 0u) {
        uint32_t d = mulhi32(r1, S.N - 1u);
        return d + (d >= n);
    }
    if (r1 < S.thr_priv) return n * S.tpn + mulhi32(r2, S.priv);
    return mulhi32(r2, S.N) * S.tpn + S.priv + mulhi32(r3, S.tpn - S.priv);
}

__device__ __forceinline__ bool draw(const Dev &S, const NodeCtx &c, uint64_t t, uint32_t &val)
{
    uint32_t r[4];
    philox4x32_10(S.seed_lo, S.seed_hi, c.n, (uint32_t)t, (uint32_t)(t >> 32), 0u, r);
    if (r[0] >= S.thr_inj) return false;
    val = draw_value(S, c.n, r[1], r[2], r[3]);
    return true;
}

// The draw for cycle t: the one computed ahead if any, else computed now.
__device__ __forceinline__ bool draw_now(const Dev &S, NodeCtx &c, uint64_t t, uint32_t &val)
{
    if (c.nd_ok && c.nd_t == (uint32_t)t) {
        c.nd_ok = false;
        val = c.nd_val;
        return c.nd_fire;
    }
    return draw(S, c, t, val);
}

__device__ __forceinline__ void prefetch_l1(const void *p)
{
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// L2-slice set of tag T of node c (first line)
__device__ __forceinline__ const uint4 *set_ptr(const Dev &S, const NodeCtx &c, uint32_t T)
{
    return S.l2 + ((size_t)c.l * S.sets + T % S.sets) * S.ways;
}

// End of cycle t (TILED engine): compute the draw of cycle t+1 ahead when the
// core will draw then, and prefetch the L2-slice set Phase 1 will probe at t+1
// (an access start or a memory fill), so the lookup hits L1.  Pure
// prefetching: the model is unchanged.
__device__ __forceinline__ void predraw(const Dev &S, NodeCtx &c, uint64_t t1)
{
    // UR draws every cycle: computing it here would only delay the next
    // boundary poll, so only the (rarer) LSPD draws are taken ahead
    if (!S.gen || S.has_script || S.mode == 0u) return;
    const uint32_t mode = core_mode(c.hot);
    const bool expiring = (mode == ML2WAIT || mode == MMEMWAIT) && (((c.hot ^ (uint32_t)t1) & 0x1FFFFFFFu) == 0u);
    if (expiring && mode == MMEMWAIT && (c.cold.w & 1u)) prefetch_l1(set_ptr(S, c, c.cold.z));
    if (mode == MIDLE || expiring) {
        c.nd_fire = draw(S, c, t1, c.nd_val);
        c.nd_t = (uint32_t)t1;
        c.nd_ok = true;
        if (c.nd_fire) prefetch_l1(set_ptr(S, c, c.nd_val));
    }
}

// At ejection: prefetch what the (deferred) service of flit f will read.
__device__ __forceinline__ void prefetch_service(const Dev &S, const NodeCtx &c, const Flit &f)
{
    const uint32_t k = f_kind(f);
    if (k == KDA || (k == KEV && !(f.w & WB_BIT))) prefetch_l1(&S.loc[loc_index(S, f.w)]);
    else if (k == KRQ) prefetch_l1(set_ptr(S, c, f.w));
}

__device__ __forceinline__ void phase1_ur(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t)
{
    if (!S.gen) return;
    uint32_t v, dst = 0;
    bool fire = false;
    if (S.has_script && script_next(S, c, t, v)) {
        fire = true; dst = v;
    } else if (S.thr_inj != 0u) {    // at rate 0 no draw can fire (r0 < 0 never holds)
        fire = draw_now(S, c, t, dst);
    }
    if (fire) {
        K.cnt(S, C_GENERATED);
        enq(S, K, c, KPROBE, dst, 0u, 1u);
    }
}

__device__ __forceinline__ void phase1_lspd(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t)
{
    uint32_t mode = core_mode(c.hot);
    if (mode == ML1WAIT && (((c.hot ^ (uint32_t)t) & 0x1FFFFFFFu) == 0u)) {   // NEXT-f1: L1 miss countdown over
        load_cold(S, c);
        l2_access(S, K, c, c.cold.z, t);
        mode = core_mode(c.hot);
    }
    if ((mode == ML2WAIT || mode == MMEMWAIT) && (((c.hot ^ (uint32_t)t) & 0x1FFFFFFFu) == 0u)) {
        load_cold(S, c);
        if (mode == MMEMWAIT && (c.cold.w & 1u)) install(S, K, c, c.cold.z, t);
        l1_fill(S, K, c, c.cold.z, c.n, t);       // local L2 hit or memory fill: supplied locally (R42)
        complete(S, K, c, t);
        mode = MIDLE;
    }
    if (mode == MIDLE && S.gen) {
        uint32_t v, T = 0;
        bool fire = false;
        if (S.has_script && script_next(S, c, t, v)) {
            fire = true; T = v;
        } else {
            fire = draw_now(S, c, t, T);
        }
        if (fire) start_access(S, K, c, T, t);
    }
}

// Phase 1 (LSPD) with the generation draws taken from a window computed ahead
// by the whole warp (TILED engine): bit k of wmask says whether the draw of
// cycle wbase+k fires (r0 < thr_inj); the value of the window's first firing
// draw is cached in nd_val.  Outside a window the draw is computed here.  The
// model is phase1_lspd's; only where the Philox evaluations run differs.
template <bool L1>
__device__ __forceinline__ void phase1_lspd_win(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t,
                                                uint32_t wbase, uint32_t wmask)
{
    uint32_t mode = core_mode(c.hot);
    if (L1 && mode == ML1WAIT && (((c.hot ^ (uint32_t)t) & 0x1FFFFFFFu) == 0u)) {   // NEXT-f1: L1 miss countdown over
        load_cold(S, c);
        l2_access(S, K, c, c.cold.z, t);
        mode = core_mode(c.hot);
    }
    if ((mode == ML2WAIT || mode == MMEMWAIT) && (((c.hot ^ (uint32_t)t) & 0x1FFFFFFFu) == 0u)) {
        load_cold(S, c);
        if (mode == MMEMWAIT && (c.cold.w & 1u)) install(S, K, c, c.cold.z, t);
        if (L1) l1_fill(S, K, c, c.cold.z, c.n, t);   // local L2 hit or memory fill: supplied locally (R42)
        complete(S, K, c, t);
        mode = MIDLE;
    }
    if (mode == MIDLE && S.gen) {
        uint32_t v, T = 0;
        bool fire = false;
        const uint32_t k = (uint32_t)t - wbase;
        if (S.has_script && script_next(S, c, t, v)) {
            fire = true; T = v;
        } else if (k < 32u) {
            if ((wmask >> k) & 1u) {
                if (c.nd_ok && c.nd_t == (uint32_t)t) { T = c.nd_val; fire = true; }
                else fire = draw(S, c, t, T);
            }
        } else {
            fire = draw(S, c, t, T);
        }
        if (fire) start_access(S, K, c, T, t);
    }
}

// ---------------------------------------------------------------------------
// Phase 2: rank and port selection (PMDR P:L116)
// ---------------------------------------------------------------------------
// The <= 5 router inputs (4 link slots + the injection slot) held in registers.
struct Inputs {
    Flit f[5];
    uint32_t present;   // bit k: slot k holds a flit
};

// Priority key of a flit at cycle t (R1, R2): a larger key ranks first.
//   DEFLECT: age desc, then lifetime t-inj desc (= inj asc), then src asc
//   OLDEST : lifetime desc, then src asc
// Packed as age[48:64) | lifetime[21:48) | (2^21-1-src)[0:21); a lifetime of
// 2^27 cycles or more is a field-width overflow (R32).
__device__ __forceinline__ uint64_t prio_key(const Dev &S, const Flit &f, uint32_t t32)
{
    uint32_t life = t32 - f.z;
    if (life > LIFE_MAX) { atomicOr(S.err, ERR_AGE); life = LIFE_MAX; }
    uint64_t k = ((uint64_t)life << 21) | (NODE_MASK - f_src(f));
    if (S.prio == 0u) k |= (uint64_t)f_age(f) << 48;
    return k;
}

// dst -> (x, y) without a hardware divide: umulhi by ceil(2^32/W) is exact for
// node ids < 2^21 (W <= 2048)
__device__ __forceinline__ uint32_t row_of(const Dev &S, uint32_t n) { return __umulhi(n, S.wmagic); }

// Rank + port selection for the router of node c (R3-R6):
// flits are taken in priority order ("Priority Sort") by repeated
// selection of the largest key; each takes the eject link (if at its
// destination and still free), else its first free productive port (x before
// y, PMDR), else the first free existing port in N,S,E,W with age+1.
// Output callback Out(port, flit) stores a routed flit into its next-cycle slot.
// Returns the mask of output ports taken.
// First choice of flit f at node c (eject at the destination, else the x-port
// if dx != 0, else the y-port; PMDR P:L116), with the lifetime check (R32).
__device__ __forceinline__ uint32_t first_choice(const Dev &S, const NodeCtx &c, const Flit &f, uint32_t t32,
                                                 uint32_t &bad)
{
    bad |= (t32 - f.z > LIFE_MAX) ? ERR_AGE : 0u;   // reported by the caller (R32)
    const uint32_t dst = f_dst(f);
    if (dst == c.n) return PX;
    const uint32_t dy = row_of(S, dst), dx = dst - dy * S.W;
    return dx != c.x ? (dx > c.x ? PE : PW) : (dy > c.y ? PS : PN);
}

// The general case: full ranking + greedy (see route()).
template <typename Out>
__device__ __forceinline__ uint32_t route_select(const Dev &S, const NodeCtx &c, Inputs &in, uint64_t t, Acc &acc,
                                                 Flit &ej, bool &has_ej, Out &&out);

template <typename Out>
__device__ __forceinline__ uint32_t route(const Dev &S, const NodeCtx &c, Inputs &in, uint64_t t, Acc &acc,
                                          Flit &ej, bool &has_ej, Out &&out)
{
    const uint32_t t32 = (uint32_t)t;
    // Fast path: if the flits' first choices are pairwise distinct, the greedy
    // gives every flit its first choice whatever the ranking, and nothing is
    // deflected.
    {
        uint32_t fc[5], seen = 0, bad = 0;
        bool coll = false;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            fc[k] = PX;
            if ((in.present >> k) & 1u) {
                fc[k] = first_choice(S, c, in.f[k], t32, bad);
                coll |= (seen >> fc[k]) & 1u;
                seen |= 1u << fc[k];
            }
        }
        if (bad) atomicOr(S.err, bad);
        if (!coll) {
            has_ej = false;
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                if (!((in.present >> k) & 1u)) continue;
                if (fc[k] == PX) { ej = in.f[k]; has_ej = true; continue; }
                ++acc.hops;
                out(fc[k], in.f[k]);
            }
            return seen & 15u;
        }
    }
    return route_select(S, c, in, t, acc, ej, has_ej, out);
}

template <typename Out>
__device__ __forceinline__ uint32_t route_select(const Dev &S, const NodeCtx &c, Inputs &in, uint64_t t, Acc &acc,
                                                 Flit &ej, bool &has_ej, Out &&out)
{
    const uint32_t t32 = (uint32_t)t;
    uint64_t key[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) key[k] = ((in.present >> k) & 1u) ? prio_key(S, in.f[k], t32) : 0ull;
    const uint32_t exist = (c.y > 0 ? 1u : 0u) | (c.y + 1 < S.H ? 2u : 0u) | (c.x + 1 < S.W ? 4u : 0u) |
                           (c.x > 0 ? 8u : 0u);
    uint32_t used = 0, left = in.present;
    has_ej = false;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        if (!left) break;
        // the highest-priority remaining flit (keys of present flits are > 0)
        int bi = 0;
        uint64_t bk = 0;
        Flit f = in.f[0];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            if (((left >> k) & 1u) && key[k] > bk) { bk = key[k]; bi = k; f = in.f[k]; }
        }
        left &= ~(1u << bi);
        const uint32_t dst = f_dst(f);
        if (dst == c.n) {
            if (!has_ej) { ej = f; has_ej = true; continue; }
        }
        int p = -1;
        if (dst != c.n) {
            const uint32_t dy = row_of(S, dst), dx = dst - dy * S.W;
            if (dx != c.x) {
                const uint32_t xp = dx > c.x ? PE : PW;
                if (!(used & (1u << xp))) p = (int)xp;
            }
            if (p < 0 && dy != c.y && (S.route == 0u || dx == c.x)) {   // strict XY: y only once dx = 0
                const uint32_t yp = dy > c.y ? PS : PN;
                if (!(used & (1u << yp))) p = (int)yp;
            }
        }
        if (p < 0) {
            p = (int)defl_port(exist & ~used, S.route);   // first free existing port in N,S,E,W (R5) / N,E,S,W (XY)
            uint32_t a = f_age(f) + 1u;
            if (a > AGE_MAX) { atomicOr(S.err, ERR_AGE); a = AGE_MAX; }
            f_set_age(f, a);
            ++acc.defl;
        }
        used |= 1u << p;
        ++acc.hops;
        out((uint32_t)p, f);
    }
    return used;
}

// ---------------------------------------------------------------------------
// Phase 3: eject + service
// ---------------------------------------------------------------------------
static __device__ void phase3(const Dev &S, const Sink &K, NodeCtx &c, const Flit &f, uint64_t t, Acc &acc)
{
    if (K.on) ++acc.ejected;
    K.hist(S, 0, (uint32_t)t - f.z);
    K.hist(S, 1, f_age(f));
    switch (f_kind(f)) {
    case KPROBE:
        K.cnt(S, C_PROBES);
        break;
    case KDA:
        dir_service(S, K, c, f.w, f_src(f), t);
        break;
    case KDR:
        receive_dr(S, K, c, f.w);
        break;
    case KNDR:
        receive_ndr(S, K, c, t);
        break;
    case KRQ:
        K.cnt(S, C_REQRCVD);
        if (l2_hit(S, c, f.w, t)) {
            K.cnt(S, C_REPSENT);
            enq(S, K, c, KRA, f_src(f), f.w, S.nfl_ra);
        } else {
            K.cnt(S, C_TRAPSENT);
            enq(S, K, c, KTRAP, f_src(f), f.w, 1u);
        }
        break;
    case KRA: {
        if (core_mode(c.hot) != MWAITDATA) atomicOr(S.err, ERR_PROTO);
        load_cold(S, c);
        uint32_t rx = (c.cold.w >> 1) + 1u;
        if (rx == S.nfl_ra) {
            c.cold.w &= 1u;
            c.cold_dirty = true;
            K.cnt(S, C_REPRCVD);
            l1_fill(S, K, c, c.cold.z, f_src(f), t);   // supplied by the holder's slice (R42)
            complete(S, K, c, t);
        } else {
            c.cold.w = (c.cold.w & 1u) | (rx << 1);
            c.cold_dirty = true;
        }
        break;
    }
    case KTRAP:
        if (core_mode(c.hot) != MWAITDATA) atomicOr(S.err, ERR_PROTO);
        K.cnt(S, C_TRAPRCVD);
        K.cnt(S, C_MEMREQ);
        load_cold(S, c);
        c.cold.w &= ~1u;                          // install = 0 (R16)
        c.cold_dirty = true;
        set_mode(c, MMEMWAIT, t + S.mem_lat);
        break;
    default:  // KEV; with WB_BIT an L1 victim writeback, absorbed (R42)
        if (f.w & WB_BIT) K.cnt(S, C_WBRCVD);
        else ev_handler(S, K, f.w, f_src(f));
        break;
    }
}

// ---------------------------------------------------------------------------
// Injection (R7, R8): one flit of the head packet per cycle, only
// if fewer flits than ports arrived.  The injected flit takes slot 4.  When the
// head packet is popped, the next head is fetched (used at t+1 at the earliest).
// frees: 1 if, under the NEXT-f4 injection mode (R43), a present flit will
// eject and so frees its input port for this cycle's injection
__device__ __forceinline__ bool inject_flit(const Dev &S, NodeCtx &c, uint32_t npresent, uint64_t t, Acc &acc,
                                            Flit &out, uint32_t frees = 0u)
{
    const uint32_t qn = q_count(c.qctl);
    if (qn == 0u || npresent - frees >= c.deg) return false;
    const uint32_t h = q_head(c.qctl);
    uint32_t nx = q_next(c.qctl);
    if (!c.head_ok) { c.head = S.fifo_pkt[(size_t)c.l * S.qcap + h]; c.head_ok = true; }
    const uint2 p = c.head;
    const uint32_t nfl = (p.x >> 24) & 15u;
    out = f_make(p.x & NODE_MASK, (p.x >> 21) & 7u, nx, c.n, (uint32_t)t, p.y);
    f_set_age(out, S.age_base);
    ++acc.injected;
    ++nx;
    if (nx == nfl) {
        const uint32_t h1 = (h + 1u) & (S.qcap - 1u);
        c.qctl = q_make(h1, qn - 1u, 0u);
        c.head_ok = qn > 1u;
        if (c.head_ok) c.head = S.fifo_pkt[(size_t)c.l * S.qcap + h1];
    } else {
        c.qctl = q_make(h, qn, nx);
    }
    c.q_dirty = true;
    return true;
}

__device__ __forceinline__ void inject(const Dev &S, NodeCtx &c, Inputs &in, uint64_t t, Acc &acc)
{
    uint32_t frees = 0u;
    if (S.inject_mode)
#pragma unroll
        for (int k = 0; k < 4; ++k) frees |= ((in.present >> k) & 1u) && f_dst(in.f[k]) == c.n;
    if (inject_flit(S, c, (uint32_t)__popc(in.present), t, acc, in.f[4], frees)) in.present |= 16u;
}

// The whole node step of cycle t with links in global memory (SoA).
// Returns true if the node is busy at the end of the cycle (drain detection).
// ---------------------------------------------------------------------------
template <uint32_t MODE>
__device__ __forceinline__ bool node_step_global(const Dev &S, const Sink &K, uint32_t l, uint64_t t, Acc &acc)
{
    NodeCtx c;
    c.l = l;
    c.n = S.n0 + l;
    c.y = c.n / S.W;
    c.x = c.n - c.y * S.W;
    c.deg = (c.y > 0) + (c.y + 1 < S.H) + (c.x + 1 < S.W) + (c.x > 0);
    c.qctl = S.fifo_ctl[l];
    c.hot = MODE == 1u ? S.core_hot[l] : 0u;
    c.head_ok = false;
    c.nd_ok = false;
    c.q_dirty = c.hot_dirty = c.cold_dirty = c.cold_loaded = false;
    c.busy_flit = false;

    // Phase 1
    if (MODE == 0u) phase1_ur(S, K, c, t);
    else phase1_lspd(S, K, c, t);

    // Phase 2: latch inputs of cycle t
    const uint32_t b = (uint32_t)t & 1u, nb1 = b ^ 1u;
    const uint32_t st = stamp_of(t);
    uint32_t fl = __ldcg(&S.flag[b][l]);
    // consume: clear the occupancy word (its slots are re-written for cycle t+2
    // only after the cycle boundary), so a stale stamp can never match again
    if (fl) S.flag[b][l] = 0u;
    Inputs in;
    in.present = 0;
#pragma unroll
    for (uint32_t d = 0; d < 4; ++d) {
        if (((fl >> (8u * d)) & 0xFFu) == st) {
            uint4 v = __ldcg(&S.flit[b][(size_t)d * S.nloc + l]);
            in.f[d] = Flit{v.x, v.y, v.z, v.w};
            in.present |= 1u << d;
        }
    }
    inject(S, c, in, t, acc);
    Flit ej;
    bool has_ej = false;
    if (in.present) {
        const uint32_t nf = __popc(in.present);
        const uint8_t st1 = stamp_of(t + 1);
        route(S, c, in, t, acc, ej, has_ej, [&](uint32_t p, const Flit &f) {
            // neighbour's local index and its input slot opp(p); a link that
            // leaves the row band lands in the neighbour band's arrays (DESIGN 8)
            uint32_t m, slot, nl = S.nloc;
            uint4 *fl = S.flit[nb1];
            uint32_t *fg = S.flag[nb1];
            switch (p) {
            case PN:
                slot = PS;
                if (l < S.W) { nl = S.nloc_nb[0]; m = l - S.W + nl; fl = S.flit_nb[0][nb1]; fg = S.flag_nb[0][nb1]; }
                else m = l - S.W;
                break;
            case PS:
                slot = PN;
                if (l + S.W >= S.nloc) { nl = S.nloc_nb[1]; m = l + S.W - S.nloc; fl = S.flit_nb[1][nb1]; fg = S.flag_nb[1][nb1]; }
                else m = l + S.W;
                break;
            case PE: m = l + 1u; slot = PW; break;
            default: m = l - 1u; slot = PE; break;
            }
            fl[(size_t)slot * nl + m] = make_uint4(f.x, f.y, f.z, f.w);
            reinterpret_cast<uint8_t *>(fg)[(size_t)m * 4u + slot] = st1;
        });
        c.busy_flit = nf > (has_ej ? 1u : 0u);
    }

    // Phase 3
    if (has_ej) phase3(S, K, c, ej, t, acc);

    if (c.q_dirty) S.fifo_ctl[l] = c.qctl;
    if (MODE == 1u) {
        if (c.hot_dirty) S.core_hot[l] = c.hot;
        if (c.cold_dirty) S.core_cold[l] = c.cold;
    }
    return c.busy_flit || q_count(c.qctl) > 0 || core_mode(c.hot) != MIDLE;
}

}  // namespace noc
