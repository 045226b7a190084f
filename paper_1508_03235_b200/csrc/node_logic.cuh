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

// The lean TILED kernels (tile_m0.cu, tile_m1.cu define NOC_LEAN 1) compile
// out the NEXT-f1 L1, NEXT-f2 migration and memory-node paths; the host runs
// configurations that use any of them on the full kernels (tile_m2.cu and the
// other engines), so the bench kernel carries none of their code.
#ifndef NOC_LEAN
#define NOC_LEAN 0
#endif

namespace noc {

__device__ __forceinline__ uint32_t mig_on(const Dev &S) { return NOC_LEAN ? 0u : S.mig_hist; }
__device__ __forceinline__ uint32_t mem_on(const Dev &S) { return NOC_LEAN ? 0u : S.mem_mode; }
__device__ __forceinline__ uint32_t l1_on(const Dev &S) { return NOC_LEAN ? 0u : S.l1_sets; }

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

// Send-FIFO storage of local node l: its packet ring and capacity.  Hub nodes
// (the central directory node, the memory controllers) may have a larger one
// (R56); only the rare FIFO paths (enqueue, head refill) look this up.
struct FifoRef {
    uint2 *p;
    uint32_t cap;
};
__device__ __forceinline__ FifoRef fifo_of(const Dev &S, uint32_t l)
{
    if (!NOC_LEAN && S.hub_of) {
        const uint32_t h = S.hub_of[l];
        if (h) return FifoRef{S.hub_pkt + (size_t)(h - 1u) * S.hub_cap, S.hub_cap};
    }
    return FifoRef{S.fifo_pkt + (size_t)l * S.qcap, S.qcap};
}

// ENQ (DESIGN 3.3; bounded send FIFO, R21)
__device__ __forceinline__ void enq(const Dev &S, const Sink &K, NodeCtx &c, uint32_t kind, uint32_t dst,
                                    uint32_t payload, uint32_t nfl)
{
    uint32_t h = q_head(c.qctl), cnt = q_count(c.qctl);
    const FifoRef F = fifo_of(S, c.l);
    if (cnt == F.cap) {
        K.cnt(S, C_DROPS + kind);
        // R21: in LSPD mode a dropped protocol message would leave a core or a
        // directory entry waiting for ever, so the run is invalid: poison it
        if (S.mode != 0u) atomicOr(S.err, ERR_DROP);
        return;
    }
    uint32_t slot = (h + cnt) & (F.cap - 1u);
    const uint2 pkt = make_uint2(dst | (kind << 21) | (nfl << 24), payload);
    F.p[slot] = pkt;
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

// The node holding block T's memory (R54): its home, or its controller
__device__ __forceinline__ uint32_t mem_node(const Dev &S, uint32_t T)
{
    return mem_on(S) == 1u ? home_of(S, T) : mem_ctrl_node(S.W, S.H, S.mem_ctrls, T % S.mem_ctrls);
}

// A B2 block (Table I: nfl_b2 flits) of the given kind and payload to dst, as
// packets of <= 8 flits (R50)
__device__ __forceinline__ void send_b2(const Dev &S, const Sink &K, NodeCtx &c, uint32_t dst, uint32_t kind,
                                        uint32_t payload)
{
    for (uint32_t left = S.nfl_b2; left;) {
        const uint32_t k = left > 8u ? 8u : left;
        enq(S, K, c, kind, dst, payload, k);
        left -= k;
    }
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

// NEXT-f2 "statistics counter ... last N accesses" (R45): the
// ring of the last mig_hist accessor ids of line li (count / head in v.w)
static __device__ __noinline__ uint32_t record_ring(const Dev &S, size_t li, uint32_t w, uint32_t who);
__device__ __forceinline__ void record_access(const Dev &S, size_t li, uint4 &v, uint32_t who)
{
    if (mig_on(S)) v.w = record_ring(S, li, v.w, who);
}
static __device__ __noinline__ uint32_t record_ring(const Dev &S, size_t li, uint32_t vw, uint32_t who)
{
    const uint32_t N = mig_on(S);
    uint32_t cnt = lw_count(vw), head = lw_head(vw);
    if (cnt < N) {
        S.l2h[li * N + (head + cnt) % N] = who;
        ++cnt;
    } else {
        S.l2h[li * N + head] = who;
        head = (head + 1u) % N;
    }
    return lw_make(lw_state(vw), cnt, head, lw_target(vw));
}

// index of the valid line holding T in node c's slice, or -1
__device__ __forceinline__ int l2_way(const Dev &S, const NodeCtx &c, uint32_t T)
{
    const uint4 *L = S.l2 + ((size_t)c.l * S.sets + T % S.sets) * S.ways;
    for (uint32_t w = 0; w < S.ways; ++w) {
        const uint4 v = L[w];
        if (v.x == T + 1u && line_valid(v)) return (int)w;
    }
    return -1;
}

// L2HIT by accessor `who` (the owner for a local access, the requester of a
// served RQ): stamp update (R23) and, with migration, the access record
__device__ __forceinline__ bool l2_hit(const Dev &S, const NodeCtx &c, uint32_t T, uint64_t t, uint32_t who)
{
    uint32_t set = T % S.sets;
    const size_t l0 = ((size_t)c.l * S.sets + set) * S.ways;
    uint4 *L = S.l2 + l0;
    for (uint32_t w = 0; w < S.ways; ++w) {
        uint4 v = L[w];
        if (v.x == T + 1u && line_valid(v)) {
            v.y = (uint32_t)t;
            v.z = (uint32_t)(t >> 32);
            record_access(S, l0 + w, v, who);
            L[w] = v;
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
    if (mig_on(S)) {
        const uint32_t m = S.loc_mig[i];
        if (m & 1u) {
            if (h1 != src + 1u) {
                // NEXT-f2 (R47): the migration target evicted T before its
                // directory update arrived; the update leaves the entry empty
                if (m & 2u) atomicOr(S.err, ERR_PROTO);
                S.loc_mig[i] = (uint8_t)(m | 2u);
                K.cnt(S, C_EVRCVD);
                return;
            }
            S.loc_mig[i] = (uint8_t)(m & ~1u);   // the source evicted T before sending it: aborted
        }
    }
    if (h1 != src + 1u) atomicOr(S.err, ERR_EVHOLDER);
    if (pend > 0) --pend;
    else h1 = 0;
    S.loc[i] = h1 | (pend << HOLDER_BITS);
    K.cnt(S, C_EVRCVD);
}

// INSTALL (victim: first invalid, else min stamp, ties lowest way, R23)
// NEXT-f2: a forwarding ghost of T in this set is dropped
static __device__ __noinline__ void drop_ghost(const Dev &S, uint4 *L, uint32_t T)
{
    for (uint32_t w = 0; w < S.ways; ++w) {
        const uint4 v = L[w];
        if (v.x == T + 1u && lw_state(v.w) == MS_FWD) L[w] = make_uint4(0, 0, 0, 0);
    }
}

static __device__ void install(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint64_t t)
{
    uint32_t set = T % S.sets;
    const size_t l0 = ((size_t)c.l * S.sets + set) * S.ways;
    uint4 *L = S.l2 + l0;
    if (mig_on(S)) drop_ghost(S, L, T);   // NEXT-f2: T lives here again
    uint32_t victim = 0;
    uint64_t best = ~0ull;
    bool found_invalid = false;
    uint4 vline = make_uint4(0, 0, 0, 0);
    for (uint32_t w = 0; w < S.ways; ++w) {
        uint4 v = L[w];
        if (!line_valid(v)) {
            if (!found_invalid) { victim = w; vline = v; found_invalid = true; }
        } else if (!found_invalid) {
            uint64_t st = ((uint64_t)v.z << 32) | v.y;
            if (st < best) { best = st; victim = w; vline = v; }
        }
    }
    if (line_valid(vline)) {
        uint32_t V = vline.x - 1u;
        uint32_t hv = home_of(S, V);
        K.cnt(S, C_EVICTIONS);
        // NEXT-f2 (R49): a block already on its way to a migration target is
        // dropped without an EV (the target's directory update takes over)
        if (lw_state(vline.w) != MS_MIGSENT) {
            K.cnt(S, C_EVSENT);
            if (hv == c.n) ev_handler(S, K, V, c.n);
            else enq(S, K, c, KEV, hv, V, 1u);
        }
        // memory nodes (R55): the victim is written back to its memory node
        // as a B2 block (Table I "L2 Blk Replacement"), absorbed there
        if (mem_on(S) && mem_node(S, V) != c.n) {
            K.cnt(S, C_MEMWBSENT);
            send_b2(S, K, c, mem_node(S, V), KTRAP, V | MEM_BIT);
        }
    }
    uint4 nl = make_uint4(T + 1u, (uint32_t)t, (uint32_t)(t >> 32), 0u);
    record_access(S, l0 + victim, nl, c.n);   // a fresh residency: the installing access (R45)
    L[victim] = nl;
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

// core cold word w: install [0:2) (0 none, 1 install, 2 install and the
// directory counted an EV of ours, NEXT-f2 R47) | rx << 2
// A memory access of this core (install 0/1/2): off-mesh at the requester
// (R17), or -- memory nodes (R55) -- a 1-flit request to the block's memory
// node, whose B2 fill is followed by the memory latency here; a memory node
// that is this node serves it locally
__device__ __forceinline__ void mem_fetch(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t, uint32_t inst)
{
    K.cnt(S, C_MEMREQ);
    load_cold(S, c);
    c.cold.w = (c.cold.w & ~3u) | inst;
    c.cold_dirty = true;
    if (mem_on(S) && mem_node(S, c.cold.z) != c.n) {
        enq(S, K, c, KDA, mem_node(S, c.cold.z), c.cold.z | MEM_BIT, 1u);
        c.cold.w &= 3u;   // rx = 0
        set_mode(c, MMEMFETCH, 0);
        return;
    }
    set_mode(c, MMEMWAIT, t + S.mem_lat);
}

__device__ __forceinline__ void receive_ndr(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t, uint32_t payload)
{
    if (core_mode(c.hot) != MWAITDIR) atomicOr(S.err, ERR_PROTO);
    mem_fetch(S, K, c, t, (payload & NDR_NOINSTALL) ? 0u : (payload & NDR_PEND) ? 2u : 1u);
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
    if (!l1_on(S)) return;
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
    } else if (h1 == r + 1u && mig_on(S) && (S.loc_mig[i] & 1u)) {
        // NEXT-f2 (R47): r sent T away and dropped its copy; the block is on
        // its way to the target: r fetches from memory without installing
        kind = KNDR; payload = T | NDR_NOINSTALL;
    } else if (h1 == r + 1u) {
        ++pend;
        if (pend > PEND_MAX) { atomicOr(S.err, ERR_PEND); pend = PEND_MAX; }
        kind = KNDR; payload = T | (mig_on(S) ? NDR_PEND : 0u);
    } else {
        kind = KDR; payload = h1 - 1u;
    }
    S.loc[i] = h1 | (pend << HOLDER_BITS);
    if (r == c.n) {
        if (kind == KNDR) receive_ndr(S, K, c, t, payload);
        else receive_dr(S, K, c, payload);
    } else if (kind == KNDR && mem_on(S) == 1u) {
        // memory at the directory (R55): the home hands the
        // fetch to its memory and sends the B2 fill instead of the NDR
        K.cnt(S, C_MEMFILLSENT);
        send_b2(S, K, c, r, KRA, T | MEM_BIT);
    } else {
        enq(S, K, c, kind, r, payload, 1u);
    }
}

// ---------------------------------------------------------------------------
// NEXT-f2: migration and redirection (Table I; SPEC
// S:L226-243; DESIGN R44-R52).  Loopbacks (a message to the node
// itself) are handled inline without flits (R51), written out without
// recursion.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ctl_enq(const Dev &S, const Sink &K, NodeCtx &c, uint32_t to, uint32_t sub, uint32_t v,
                                        uint32_t nfl = 1u)
{
    enq(S, K, c, KPROBE, to, ctl_word(sub, v), nfl);
}

// "If a remote node have accessed it mostly, then migration get triggered"
// (SPEC should_migrate S:L235-243; R46): the node with the most
// entries in line li's history (ties: lowest id) if it is not the holder h
// and strictly ahead of h; else 0xFFFFFFFF
static __device__ uint32_t mig_target(const Dev &S, size_t li, uint32_t w, uint32_t h)
{
    const uint32_t N = mig_on(S), cnt = lw_count(w), head = lw_head(w);
    const uint32_t *H = S.l2h + li * N;
    uint32_t best = 0xFFFFFFFFu, bestc = 0, hc = 0;
    for (uint32_t i = 0; i < cnt; ++i) {
        const uint32_t a = H[(head + i) % N];
        uint32_t k = 0;
        for (uint32_t j = 0; j < cnt; ++j) k += H[(head + j) % N] == a;
        if (a == h) hc = k;
        if (k > bestc || (k == bestc && a < best)) { best = a; bestc = k; }
    }
    return (best != 0xFFFFFFFFu && best != h && bestc > hc) ? best : 0xFFFFFFFFu;
}

// the B2 block (nfl_b2 flits, Table I: 16), enqueued as <= 8-flit parts (R50)
__device__ __forceinline__ void send_block(const Dev &S, const Sink &K, NodeCtx &c, uint32_t R, uint32_t T)
{
    for (uint32_t left = S.nfl_b2; left;) {
        const uint32_t k = left > 8u ? 8u : left;
        ctl_enq(S, K, c, R, SUB_MIG, T, k);
        left -= k;
    }
}

// at home(T): a migration request from src; grant iff src holds T, no EV of T
// is pending and no migration of T is in flight (R47)
__device__ __forceinline__ bool dir_mr(const Dev &S, uint32_t T, uint32_t src)
{
    const size_t i = loc_index(S, T);
    const uint32_t e = S.loc[i];
    const bool ok = (e & HOLDER_MASK) == src + 1u && (e >> HOLDER_BITS) == 0u && !(S.loc_mig[i] & 1u);
    if (ok) S.loc_mig[i] = 1u;
    return ok;
}

// at the holder: grant -> send the block (if the line is still here), nack -> keep it
static __device__ void src_grant(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, bool ok)
{
    const int w = l2_way(S, c, T);
    if (!ok) K.cnt(S, C_MIGNACK);
    if (w < 0) return;                      // evicted meanwhile: its EV aborts the transit
    uint4 *L = S.l2 + ((size_t)c.l * S.sets + T % S.sets) * S.ways + w;
    uint4 v = *L;
    if (lw_state(v.w) != MS_MIGREQ) return;
    const uint32_t R = lw_target(v.w);
    if (ok) {
        v.w = lw_make(MS_MIGSENT, lw_count(v.w), lw_head(v.w), R);
        *L = v;
        K.cnt(S, C_MIGS);
        send_block(S, K, c, R, T);
    } else {
        v.w = lw_make(MS_NORMAL, lw_count(v.w), lw_head(v.w), 0u);
        *L = v;
    }
}

// at the old holder: "source packet invalidates its copy", keeping a
// forwarding ghost (tag, target) for redirection (R48)
__device__ __forceinline__ void src_inv(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T)
{
    K.cnt(S, C_INVAL);
    const int w = l2_way(S, c, T);
    if (w < 0) return;
    uint4 *L = S.l2 + ((size_t)c.l * S.sets + T % S.sets) * S.ways + w;
    const uint4 v = *L;
    if (lw_state(v.w) != MS_MIGSENT) return;
    *L = make_uint4(v.x, 0u, 0u, lw_make(MS_FWD, 0u, 0u, lw_target(v.w)));
}

// at home(T): the directory update from the new holder src (R47)
static __device__ void dir_du(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint32_t src)
{
    const size_t i = loc_index(S, T);
    const uint32_t m = S.loc_mig[i];
    if (!(m & 1u)) { atomicOr(S.err, ERR_PROTO); return; }
    const uint32_t e = S.loc[i];
    const uint32_t h = (e & HOLDER_MASK) - 1u;
    S.loc_mig[i] = 0u;
    K.cnt(S, C_DIRUPD);
    S.loc[i] = ((m & 2u) ? 0u : src + 1u) | (e & ~HOLDER_MASK);
    if (h == c.n) src_inv(S, K, c, T);
    else ctl_enq(S, K, c, h, SUB_INV, T);
}

// a flit of an inbound block; the last one installs it and updates the directory
static __device__ void dst_mig_flit(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint64_t t)
{
    uint2 *X = S.migrx + (size_t)c.l * 4u;
    int k = -1;
    for (int j = 0; j < 4; ++j) if (X[j].y && X[j].x == T) k = j;
    if (k < 0)
        for (int j = 0; j < 4 && k < 0; ++j) if (!X[j].y) k = j;
    if (k < 0) { atomicOr(S.err, ERR_MIGRX); return; }
    const uint32_t cnt = (X[k].y ? X[k].y : 0u) + 1u;
    if (cnt < S.nfl_b2) { X[k] = make_uint2(T, cnt); return; }
    X[k] = make_uint2(0u, 0u);
    if (l2_way(S, c, T) >= 0) { atomicOr(S.err, ERR_PROTO); return; }
    install(S, K, c, T, t);
    K.cnt(S, C_MIGINST);
    const uint32_t home = home_of(S, T);
    if (home == c.n) dir_du(S, K, c, T, c.n);
    else ctl_enq(S, K, c, home, SUB_DU, T);
}

// after an RQ served at this node: maybe start a migration (R46, R47)
static __device__ void maybe_migrate(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, int w)
{
    const size_t li = ((size_t)c.l * S.sets + T % S.sets) * S.ways + w;
    uint4 v = S.l2[li];
    if (lw_state(v.w) != MS_NORMAL) return;
    const uint32_t R = mig_target(S, li, v.w, c.n);
    if (R == 0xFFFFFFFFu) return;
    v.w = lw_make(MS_MIGREQ, lw_count(v.w), lw_head(v.w), R);
    S.l2[li] = v;
    K.cnt(S, C_MIGREQ);
    const uint32_t home = home_of(S, T);
    if (home == c.n) src_grant(S, K, c, T, dir_mr(S, T, c.n));
    else ctl_enq(S, K, c, home, SUB_MR, T);
}

// a forwarding ghost of T here: redirect the requester r to the new holder (R48)
static __device__ bool redirect(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint32_t r)
{
    const uint4 *L = S.l2 + ((size_t)c.l * S.sets + T % S.sets) * S.ways;
    for (uint32_t w = 0; w < S.ways; ++w) {
        const uint4 v = L[w];
        if (v.x == T + 1u && lw_state(v.w) == MS_FWD) {
            K.cnt(S, C_REDIR);
            ctl_enq(S, K, c, r, SUB_RR, lw_target(v.w));
            return true;
        }
    }
    return false;
}

// RQ for T from requester r at this node (Fig. 4 step 4): serve from
// the slice (RA), else redirect through a forwarding ghost (R48), else
// TRAP.  r == c.n only for a redirection to the requester itself,
// served inline (R51).
static __device__ void serve_rq(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint32_t r, uint64_t t)
{
    K.cnt(S, C_REQRCVD);
    if (l2_hit(S, c, T, t, r)) {
        K.cnt(S, C_REPSENT);
        if (r == c.n) {
            K.cnt(S, C_REPRCVD);
            l1_fill(S, K, c, T, c.n, t);
            complete(S, K, c, t);
        } else {
            enq(S, K, c, KRA, r, T, S.nfl_ra);
        }
        if (mig_on(S)) maybe_migrate(S, K, c, T, l2_way(S, c, T));
        return;
    }
    if (mig_on(S) && r != c.n && redirect(S, K, c, T, r)) return;
    K.cnt(S, C_TRAPSENT);
    if (r == c.n) {
        K.cnt(S, C_TRAPRCVD);
        K.cnt(S, C_MEMREQ);
        load_cold(S, c);
        c.cold.w &= ~3u;
        c.cold_dirty = true;
        set_mode(c, MMEMWAIT, t + S.mem_lat);
    } else {
        enq(S, K, c, KTRAP, r, T, 1u);
    }
}

// a migration / redirection message (sub, v) from src delivered here (R47, R48)
static __device__ void ctl_deliver(const Dev &S, const Sink &K, NodeCtx &c, uint32_t sub, uint32_t v, uint32_t src,
                                   uint64_t t)
{
    switch (sub) {
    case SUB_MR: ctl_enq(S, K, c, src, dir_mr(S, v, src) ? SUB_MG : SUB_MN, v); break;
    case SUB_MG: src_grant(S, K, c, v, true); break;
    case SUB_MN: src_grant(S, K, c, v, false); break;
    case SUB_MIG: dst_mig_flit(S, K, c, v, t); break;
    case SUB_DU: dir_du(S, K, c, v, src); break;
    case SUB_INV: src_inv(S, K, c, v); break;
    case SUB_RR:   // "Reply redirection" (Table I; R48): ask the new holder v
        if (core_mode(c.hot) != MWAITDATA) atomicOr(S.err, ERR_PROTO);
        K.cnt(S, C_RRRCVD);
        K.cnt(S, C_REQMADE);
        load_cold(S, c);
        if (v == c.n) serve_rq(S, K, c, c.cold.z, c.n, t);
        else enq(S, K, c, KRQ, v, c.cold.z, 1u);
        break;
    default: atomicOr(S.err, ERR_PROTO); break;
    }
}

// MEMWAIT over with an install pending; NEXT-f2 (R47): if the block
// migrated here meanwhile there is no second copy, and if the directory
// counted an EV of ours that does not exist, one is sent to even it
static __device__ void mem_fill(const Dev &S, const Sink &K, NodeCtx &c, uint64_t t)
{
    load_cold(S, c);
    const uint32_t T = c.cold.z;
    if (mig_on(S) && l2_way(S, c, T) >= 0) {
        if ((c.cold.w & 3u) == 2u) {
            const uint32_t hv = home_of(S, T);
            K.cnt(S, C_EVSENT);
            if (hv == c.n) ev_handler(S, K, T, c.n);
            else enq(S, K, c, KEV, hv, T, 1u);
        }
        return;
    }
    install(S, K, c, T, t);
}

// The local L2 part of an access (Fig. 4): hit, else the directory
static __device__ void l2_access(const Dev &S, const Sink &K, NodeCtx &c, uint32_t T, uint64_t t)
{
    if (l2_hit(S, c, T, t, c.n)) {
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
    if (l1_on(S)) {
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
    // pushed events (R57): the queue holds only events not consumed at the
    // last merge, so the next one sits at pos - base
    const uint32_t idx = off + pos - (S.script_base ? S.script_base[c.l] : 0u);
    if (idx >= end) return false;
    uint4 ev = S.script[idx];
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
    if (expiring && mode == MMEMWAIT && (c.cold.w & 3u)) prefetch_l1(set_ptr(S, c, c.cold.z));
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
        if (mode == MMEMWAIT && (c.cold.w & 3u)) mem_fill(S, K, c, t);
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
        if (mode == MMEMWAIT && (c.cold.w & 3u)) mem_fill(S, K, c, t);
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

// Tie-break of equal priority keys (R53): only flits one node injected in the
// same cycle (fill-all injection) share (age, inj, src); they rank by fid,
// kind, dst, payload ascending -- a SMALLER secondary key ranks first.  Flits
// equal in all of these are identical (either order gives the same state).
__device__ __forceinline__ uint64_t sec_key(const Flit &f)
{
    return ((uint64_t)f_fid(f) << 56) | ((uint64_t)f_kind(f) << 53) | ((uint64_t)f_dst(f) << 32) | f.w;
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
            if (!((left >> k) & 1u)) continue;
            const bool tie_first = S.inject_mode == 2u && key[k] == bk && sec_key(in.f[k]) < sec_key(f);
            if (key[k] > bk || tie_first) { bk = key[k]; bi = k; f = in.f[k]; }
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
    case KPROBE:   // = the migration / redirection messages in LSPD mode (R50)
        if (S.mode != 0u) ctl_deliver(S, K, c, f.w >> 28, f.w & 0x0FFFFFFFu, f_src(f), t);
        else K.cnt(S, C_PROBES);
        break;
    case KDA:
        if (f.w & MEM_BIT) {   // a memory request at a memory node (R55): the B2 fill
            K.cnt(S, C_MEMFILLSENT);
            send_b2(S, K, c, f_src(f), KRA, f.w);
        } else {
            dir_service(S, K, c, f.w, f_src(f), t);
        }
        break;
    case KDR:
        receive_dr(S, K, c, f.w);
        break;
    case KNDR:
        receive_ndr(S, K, c, t, f.w);
        break;
    case KRQ:
        serve_rq(S, K, c, f.w, f_src(f), t);
        break;
    case KRA: {
        if (f.w & MEM_BIT) {   // a flit of a B2 memory fill (R55)
            const uint32_t mode = core_mode(c.hot);
            if (mode != MMEMFETCH && mode != MWAITDIR) atomicOr(S.err, ERR_PROTO);
            load_cold(S, c);
            if ((f.w & ~MEM_BIT) != c.cold.z) atomicOr(S.err, ERR_PROTO);
            const uint32_t rx = (c.cold.w >> 2) + 1u;
            c.cold_dirty = true;
            if (rx == S.nfl_b2) {
                K.cnt(S, C_MEMFILLRCVD);
                uint32_t inst = c.cold.w & 3u;
                if (mode == MWAITDIR) { K.cnt(S, C_MEMREQ); inst = 1u; }   // the home's memory answered (mem_mode 1)
                c.cold.w = inst;
                set_mode(c, MMEMWAIT, t + S.mem_lat);
            } else {
                c.cold.w = (c.cold.w & 3u) | (rx << 2);
            }
            break;
        }
        if (core_mode(c.hot) != MWAITDATA) atomicOr(S.err, ERR_PROTO);
        load_cold(S, c);
        uint32_t rx = (c.cold.w >> 2) + 1u;
        if (rx == S.nfl_ra) {
            c.cold.w &= 3u;
            c.cold_dirty = true;
            K.cnt(S, C_REPRCVD);
            l1_fill(S, K, c, c.cold.z, f_src(f), t);   // supplied by the holder's slice (R42)
            complete(S, K, c, t);
        } else {
            c.cold.w = (c.cold.w & 3u) | (rx << 2);
            c.cold_dirty = true;
        }
        break;
    }
    case KTRAP:
        if (f.w & MEM_BIT) {   // a memory writeback flit at a memory node: absorbed (R55)
            K.cnt(S, C_MEMWBFLITS);
            break;
        }
        if (core_mode(c.hot) != MWAITDATA) atomicOr(S.err, ERR_PROTO);
        K.cnt(S, C_TRAPRCVD);
        mem_fetch(S, K, c, t, 0u);                // install = 0 (R16)
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
    if (!c.head_ok) { c.head = fifo_of(S, c.l).p[h]; c.head_ok = true; }
    const uint2 p = c.head;
    const uint32_t nfl = (p.x >> 24) & 15u;
    out = f_make(p.x & NODE_MASK, (p.x >> 21) & 7u, nx, c.n, (uint32_t)t, p.y);
    f_set_age(out, S.age_base);
    ++acc.injected;
    ++nx;
    if (nx == nfl) {
        const FifoRef F = fifo_of(S, c.l);
        const uint32_t h1 = (h + 1u) & (F.cap - 1u);
        c.qctl = q_make(h1, qn - 1u, 0u);
        c.head_ok = qn > 1u;
        if (c.head_ok) c.head = F.p[h1];
    } else {
        c.qctl = q_make(h, qn, nx);
    }
    c.q_dirty = true;
    return true;
}

__device__ __forceinline__ void inject(const Dev &S, NodeCtx &c, Inputs &in, uint64_t t, Acc &acc)
{
    if (S.inject_mode == 2u) {
        // NEXT-f4 fill-all (R53): queued flits fill every
        // free input slot, oldest-queued first (empty link slots, so the
        // injection register stays unused; ranking ties: sec_key)
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (!((in.present >> k) & 1u) && inject_flit(S, c, (uint32_t)__popc(in.present), t, acc, in.f[k]))
                in.present |= 1u << k;
        return;
    }
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
    c.y = __umulhi(c.n, S.wmagic);   // n / W (exact for n < 2^21)
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
            uint4 v = __ldcg(&S.flit[b][flit_at(S.nloc, d, l)]);
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
            fl[flit_at(nl, slot, m)] = make_uint4(f.x, f.y, f.z, f.w);
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
