// common.cuh -- device-side definitions shared by the kernels of libnocsim.so.
//
// Model: DESIGN.md section 3 (Kumar & Sahu, arXiv 1508.03235).  This file is
// part of the product path; it shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace noc {

// ports / input slots in the paper's order N, S, E, W; 4 = eject
enum : uint32_t { PN = 0, PS = 1, PE = 2, PW = 3, PX = 4 };
// message kinds (Table I; DESIGN 3.2)
enum : uint32_t { KPROBE = 0, KDA = 1, KDR = 2, KNDR = 3, KRQ = 4, KRA = 5, KTRAP = 6, KEV = 7 };
// core modes (DESIGN 3.2)
enum : uint32_t { MIDLE = 0, ML2WAIT = 1, MWAITDIR = 2, MWAITDATA = 3, MMEMWAIT = 4, ML1WAIT = 5,
                  MMEMFETCH = 6 /* memory nodes (R55): waiting for a B2 fill */ };
// memory nodes (R55): a memory request is a DA flit, a memory fill flit an RA
// flit, a memory writeback flit a TRAP flit, each with this payload bit
constexpr uint32_t MEM_BIT = 0x80000000u;
// an EV flit whose payload carries this bit is an L1 victim writeback (NEXT-f1, R42;
// tags are < 2^31, R32)
constexpr uint32_t WB_BIT = 0x80000000u;
// counter indices (DESIGN 3.6)
enum : uint32_t {
    C_GENERATED = 0, C_ENQ, C_INJECTED, C_EJECTED, C_HOPS, C_DEFL, C_PROBES, C_ACCESSES,
    C_COMPLETED, C_L2HIT, C_L2MISS, C_DIRSEARCH, C_REQMADE, C_REQRCVD, C_REPSENT, C_REPRCVD,
    C_TRAPSENT, C_TRAPRCVD, C_MEMREQ, C_INSTALLS, C_EVICTIONS, C_EVSENT, C_EVRCVD,
    C_DROPS = 23, C_L1HIT = 31, C_L1MISS, C_WBSENT, C_WBRCVD,
    // NEXT-f2 migration + redirection (R44-R52)
    C_MIGREQ = 35, C_MIGNACK, C_MIGS, C_MIGINST, C_DIRUPD, C_INVAL, C_REDIR, C_RRRCVD,
    // memory nodes (R54-R55)
    C_MEMFILLSENT = 43, C_MEMFILLRCVD, C_MEMWBSENT, C_MEMWBFLITS, NCOUNTERS = 47
};
// NEXT-f2 (R50): migration / redirection messages use the PROBE kind code in
// LSPD mode, the message in payload bits 28-30, a tag or node id in bits 0-27
enum : uint32_t { SUB_MR = 1, SUB_MG = 2, SUB_MN = 3, SUB_MIG = 4, SUB_DU = 5, SUB_INV = 6, SUB_RR = 7 };
__host__ __device__ __forceinline__ uint32_t ctl_word(uint32_t sub, uint32_t v) { return (sub << 28) | v; }
// NDR payload flags (NEXT-f2, R47): fetch without installing / the reply
// counted an EV of the requester in flight
constexpr uint32_t NDR_NOINSTALL = 0x80000000u, NDR_PEND = 0x40000000u;
// L2 line word w (NEXT-f2): migration state [30:32) | history count [25:30) |
// history head [21:25) | target node [0:21); state 0 NORMAL, 1 MIGREQ,
// 2 MIGSENT, 3 FWD (an invalid forwarding ghost that keeps tag and target)
enum : uint32_t { MS_NORMAL = 0, MS_MIGREQ = 1, MS_MIGSENT = 2, MS_FWD = 3 };
__host__ __device__ __forceinline__ uint32_t lw_state(uint32_t w) { return w >> 30; }
__host__ __device__ __forceinline__ uint32_t lw_count(uint32_t w) { return (w >> 25) & 31u; }
__host__ __device__ __forceinline__ uint32_t lw_head(uint32_t w) { return (w >> 21) & 15u; }
__host__ __device__ __forceinline__ uint32_t lw_target(uint32_t w) { return w & 0x1FFFFFu; }
__host__ __device__ __forceinline__ uint32_t lw_make(uint32_t st, uint32_t cnt, uint32_t head, uint32_t tgt)
{
    return (st << 30) | (cnt << 25) | (head << 21) | tgt;
}
// a line holds a block iff tag+1 != 0 and it is not a forwarding ghost
__host__ __device__ __forceinline__ bool line_valid(const uint4 &v) { return v.x != 0u && lw_state(v.w) != MS_FWD; }
// Memory-controller node k of M (mem_mode 2, R54): ceil(M/2) controllers
// evenly spaced on the top row, the others on the bottom row
__host__ __device__ __forceinline__ uint32_t mem_ctrl_node(uint32_t W, uint32_t H, uint32_t M, uint32_t k)
{
    const uint32_t Mt = (M + 1u) / 2u, Mb = M - Mt;
    if (k < Mt) return (uint32_t)(((2ull * k + 1ull) * W) / (2ull * Mt));
    const uint32_t j = k - Mt;
    return (H - 1u) * W + (uint32_t)(((2ull * j + 1ull) * W) / (2ull * Mb));
}

// error flags
enum : uint32_t { ERR_AGE = 1, ERR_PEND = 2, ERR_EVHOLDER = 4, ERR_PROTO = 8, ERR_DROP = 16, ERR_MIGRX = 32 };

constexpr uint32_t AGE_MAX = 65535u;   // R32
constexpr uint32_t LIFE_MAX = (1u << 27) - 1u;   // R32: flit lifetime t - inj
constexpr uint32_t PEND_MAX = 1023u;   // R32
constexpr uint32_t HOLDER_BITS = 22;   // loc entry = (holder+1) | pend << 22   (R36: 4 B)
constexpr uint32_t HOLDER_MASK = (1u << HOLDER_BITS) - 1u;
constexpr uint32_t NODE_MASK = (1u << 21) - 1u;

// ---------------------------------------------------------------------------
// Flit: one 16-byte record (uint4), moved with one 128-bit load/store.
//   x = dst[0:21) | kind[21:24) | fid[24:27) | age_hi5[27:32)
//   y = src[0:21) | age_lo11[21:32)
//   z = injection cycle mod 2^32
//   w = payload (tag T or holder node)
// ---------------------------------------------------------------------------
struct Flit {
    uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ uint32_t f_dst(const Flit &f) { return f.x & NODE_MASK; }
__host__ __device__ __forceinline__ uint32_t f_kind(const Flit &f) { return (f.x >> 21) & 7u; }
__host__ __device__ __forceinline__ uint32_t f_fid(const Flit &f) { return (f.x >> 24) & 7u; }
__host__ __device__ __forceinline__ uint32_t f_src(const Flit &f) { return f.y & NODE_MASK; }
__host__ __device__ __forceinline__ uint32_t f_age(const Flit &f) { return (f.x >> 27) << 11 | (f.y >> 21); }
__host__ __device__ __forceinline__ void f_set_age(Flit &f, uint32_t a)
{
    f.x = (f.x & 0x07FFFFFFu) | ((a >> 11) << 27);
    f.y = (f.y & NODE_MASK) | ((a & 0x7FFu) << 21);
}
__host__ __device__ __forceinline__ Flit f_make(uint32_t dst, uint32_t kind, uint32_t fid, uint32_t src,
                                               uint32_t inj, uint32_t payload)
{
    Flit f;
    f.x = dst | (kind << 21) | (fid << 24);
    f.y = src;
    f.z = inj;
    f.w = payload;
    return f;
}

// FIFO packet: uint2 {dst[0:21) | kind[21:24) | nfl[24:28), payload}
// FIFO control word: head[0:10) | count[10:21) | next[21:24)
__host__ __device__ __forceinline__ uint32_t q_head(uint32_t c) { return c & 1023u; }
__host__ __device__ __forceinline__ uint32_t q_count(uint32_t c) { return (c >> 10) & 2047u; }
__host__ __device__ __forceinline__ uint32_t q_next(uint32_t c) { return c >> 21; }
__host__ __device__ __forceinline__ uint32_t q_make(uint32_t h, uint32_t n, uint32_t nx)
{
    return h | (n << 10) | (nx << 21);
}

// core hot word: mode[29:32) | ready mod 2^29 ; cold record: {start_lo, start_hi, tag, install | rx<<1}
__host__ __device__ __forceinline__ uint32_t core_mode(uint32_t hot) { return hot >> 29; }

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11, Random123 constants); R25.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1,
                                                      uint32_t c2, uint32_t c3, uint32_t r[4])
{
#pragma unroll
    for (int i = 0; i < 10; ++i) {
#ifdef __CUDA_ARCH__
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    r[0] = c0; r[1] = c1; r[2] = c2; r[3] = c3;
}

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t r, uint32_t m)
{
#ifdef __CUDA_ARCH__
    return __umulhi(r, m);
#else
    return (uint32_t)(((uint64_t)r * m) >> 32);
#endif
}

// ---------------------------------------------------------------------------
// Canonical hash (DESIGN 3.7)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct TupleHash {
    uint64_t h;
    __host__ __device__ explicit TupleHash(int k) : h((uint64_t)k) {}
    __host__ __device__ TupleHash &add(uint64_t v) { h = mix64(h ^ v); return *this; }
};

__host__ __device__ __forceinline__ uint64_t hterm(uint64_t dom, uint64_t idx, uint64_t tup)
{
    return mix64(mix64((dom << 56) ^ idx) ^ tup);
}

enum : uint64_t { D_LINK = 1, D_FIFO = 2, D_FIFONEXT = 3, D_CORE = 4, D_L2 = 5, D_LOC = 6,
                  D_CNT = 7, D_HIST = 8, D_CYCLE = 9, D_SCRIPT = 10, D_L1 = 11, D_L2MIG = 12, D_LOCMIG = 13,
                  D_MIGRX = 14 };

// ---------------------------------------------------------------------------
// Device view of one simulation (passed by value to every kernel).
// All arrays are indexed by the LOCAL node index l in [0, nloc) of this rank's
// band (rows [row0, row0+rows) of the mesh): global id n = n0 + l.
// ---------------------------------------------------------------------------
struct Dev {
    // geometry and model parameters
    uint32_t W, H, N, n0, nloc, row0, rows;
    uint32_t mode, prio, route, sets, ways, tpn, priv, thr_inj, thr_priv, l2_hit_lat, mem_lat, nfl_ra;
    uint32_t dir_mode, dir_node;      // NEXT-f3: central directory at dir_node (R40)
    uint32_t l1_sets, l1_ways, l1_miss_lat;   // NEXT-f1 private L1 (R42); 0 sets = none
    uint32_t inject_mode;             // NEXT-f4: 1 an ejecting flit frees its slot (R43), 2 fill all free slots (R53)
    uint32_t age_base;                // test knob: age of an injected flit (0 = P:L259)
    uint32_t mig_hist, nfl_b2;        // NEXT-f2: accessor history length (0 = off), B2 flits
    uint32_t mem_mode, mem_ctrls;     // memory placement (R54): 0 off-mesh, 1 home node, 2 controllers
    uint32_t hub_cap;                 // send-FIFO capacity of hub nodes (R56)
    uint64_t loc_n;                   // directory entries held by this band
    uint32_t qcap, nb, seed_lo, seed_hi;
    uint32_t wmagic;                  // ceil(2^32 / W): row of a node id by umulhi
    uint32_t gen;                     // generation enabled (0 during drain)
    uint32_t has_script;
    // state
    uint4 *flit[2];                   // [2][4][nloc] links, slot d of node l
    uint32_t *flag[2];                // [2][nloc] byte d = stamp of slot d
    uint32_t *core_hot;               // [nloc]
    uint4 *core_cold;                 // [nloc]
    uint32_t *fifo_ctl;               // [nloc]
    uint2 *fifo_pkt;                  // [nloc][qcap]
    uint8_t *hub_of;                  // [nloc] 0, or 1 + index of the node's hub FIFO in hub_pkt (R56); null = no hubs
    uint2 *hub_pkt;                   // [hubs in this band][hub_cap]
    uint4 *l2;                        // [nloc][sets][ways] {tag+1 (0 = invalid), stamp_lo, stamp_hi, 0}
    uint4 *l1;                        // [nloc][l1_sets][l1_ways] {tag+1, stamp_lo, stamp_hi, owner} (NEXT-f1)
    uint32_t *loc;                    // [tpn][nloc] directory entries of tags homed in this band
    uint8_t *loc_mig;                 // NEXT-f2: per entry bit 0 migration in transit, bit 1 early EV
    uint32_t *l2h;                    // NEXT-f2: [nloc][sets][ways][mig_hist] accessor ring
    uint2 *migrx;                     // NEXT-f2: [nloc][4] inbound migrations {tag, flits} (flits 0 = free)
    const uint4 *script;              // [n_script] {cycle_lo, cycle_hi, value, 0} grouped by node
    const uint32_t *script_off;       // [nloc+1]
    uint32_t *script_pos;             // [nloc] events consumed
    uint32_t *script_base;            // [nloc] events consumed before the last merge of pushed
                                      // events (NEXT-f3 streaming, R57); null = 0
    unsigned long long *cnt;          // [NCOUNTERS]
    unsigned long long *hist;         // [3][nb]
    uint32_t *err;                    // [1] error flags
    // TILED engine: TX x TY tiles over the band; links that cross a tile
    // boundary live in "LL" slots: [2 parity][4 slot][nloc][4 words] u64, each
    // word = stamp (lo32 = cycle it is an input of) | data (hi32).  Word 0 data
    // is flit.x or LL_EMPTY; words 1..3 carry flit.y, .z, .w.  Null otherwise.
    uint32_t TX, TY;
    unsigned long long *ll;
    // row bands (DESIGN 8): the LL arrays of the bands north (0) and south (1)
    // of this one, and their node counts; a link leaving the band is written
    // into the receiver band's array (another GPU's memory, mapped by CUDA
    // IPC, when bands are processes).  Null / 0 at the mesh edge.
    unsigned long long *ll_nb[2];
    uint32_t nloc_nb[2];
    // PERSIST engine with row bands: this band's per-CTA progress counters and
    // nodes per CTA, and the north (0) / south (1) neighbour band's flit and
    // flag arrays (by parity), progress counters and nodes per CTA; a link
    // leaving the band is written into the receiver band's arrays (CUDA IPC
    // mappings when bands are processes).  Null at the mesh edge.
    uint32_t *progress;
    uint32_t npc;
    uint4 *flit_nb[2][2];
    uint32_t *flag_nb[2][2];
    uint32_t *prog_nb[2];
    uint32_t npc_nb[2];
};

// Deflection port: the first free existing port in N,S,E,W (R5), or in
// N,E,S,W under the strict-XY mode (route 1).  freem != 0.
__device__ __forceinline__ uint32_t defl_port(uint32_t freem, uint32_t route)
{
    if (route == 0u) return (uint32_t)(__ffs(freem) - 1);
    if (freem & 1u) return PN;
    if (freem & 4u) return PE;
    if (freem & 2u) return PS;
    return PW;
}

// Link flit arrays flit[parity]: input slot d of local node l.  Node-major
// (the four slots of a node in one 64-byte block: a node's present flits share
// sectors, and the per-cycle hot set is a quarter as spread) unless built with
// NOC_FLIT_SLOT_MAJOR (the round-1 layout, d * nloc + l) for A/B.
__host__ __device__ __forceinline__ size_t flit_at(uint32_t nloc, uint32_t d, uint32_t l)
{
#ifdef NOC_FLIT_SLOT_MAJOR
    return (size_t)d * nloc + l;
#else
    (void)nloc;
    return (size_t)l * 4u + d;
#endif
}

constexpr uint32_t LL_EMPTY = 0xFFFFFFFFu;   // dst field all ones: never a node (N <= 2^21-1)

__host__ __device__ __forceinline__ uint8_t stamp_of(uint64_t cycle) { return (uint8_t)(0x80u | (cycle & 0x7Fu)); }

// LL word index of (parity b, input slot d, local node l, word w)
__host__ __device__ __forceinline__ size_t ll_index(const Dev &S, uint32_t b, uint32_t d, uint32_t l, uint32_t w)
{
    return (((size_t)b * 4u + d) * S.nloc + l) * 4u + w;
}

// tile column / row of a mesh coordinate for the TILED engine (x0(tx) = tx*W/TX)
__host__ __device__ __forceinline__ uint32_t tile_of(uint32_t x, uint32_t W, uint32_t TX)
{
    return (uint32_t)((((uint64_t)x + 1u) * TX + W - 1u) / W) - 1u;
}

// true if input slot d of node (x, y) is fed by a node of another tile
__host__ __device__ __forceinline__ bool slot_external(const Dev &S, uint32_t x, uint32_t y, uint32_t d)
{
    if (!S.ll) return false;
    const uint32_t ly = y - S.row0;
    switch (d) {
    case PN: return y > 0 && (ly == 0 || tile_of(ly, S.rows, S.TY) != tile_of(ly - 1u, S.rows, S.TY));
    case PS: return y + 1 < S.H && (ly + 1 == S.rows || tile_of(ly, S.rows, S.TY) != tile_of(ly + 1u, S.rows, S.TY));
    case PE: return x + 1 < S.W && tile_of(x, S.W, S.TX) != tile_of(x + 1u, S.W, S.TX);
    default: return x > 0 && tile_of(x, S.W, S.TX) != tile_of(x - 1u, S.W, S.TX);
    }
}

}  // namespace noc
