/*
 * noc_oracle.c -- TEST INFRASTRUCTURE ONLY (see noc_oracle.h).
 *
 * A plain, slow, obviously-correct, single-threaded CPU simulator of the
 * per-cycle, per-node step of the paper's simulator (Kumar & Sahu,
 * arXiv 1508.03235):
 *   - array-of-structs state, exactly the paper's serial structure
 *     "for(i..RouterCount) Phase1(i); Phase2(i); Phase3(i)";
 *   - Phase 1 = core memory-access state machine,
 *     Phase 2 = age sort + port assignment / deflection,
 *     Phase 3 = eject / reassemble / service / transfer;
 *   - the LSPD directory protocol of Fig. 4 with the readings
 *     R1..R35 of DESIGN.md section 3.
 * No blocking, no fusion, no bit packing, no SIMD, no threads.  It shares no
 * code with the CUDA library; only the written model
 * is common.
 */
#include "noc_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* Router port order N, S, E, W = Input[0..3]; 4 = eject link X */
enum { DIR_N = 0, DIR_S = 1, DIR_E = 2, DIR_W = 3, PORT_EJECT = 4 };
/* message kinds: Table I + readings R16, R18, R13 */
enum { K_PROBE = 0, K_DA = 1, K_DR = 2, K_NDR = 3, K_RQ = 4, K_RA = 5, K_TRAP = 6, K_EV = 7 };
/* NEXT-f2 (R50): migration / redirection messages travel in LSPD mode under
 * the kind code of PROBE (unused there), the message in payload bits 28-30
 * and a tag or node id in bits 0-27 */
#define K_CTL K_PROBE
enum { SUB_MR = 1, SUB_MG = 2, SUB_MN = 3, SUB_MIG = 4, SUB_DU = 5, SUB_INV = 6, SUB_RR = 7 };
#define CTL(sub, v) (((uint32_t)(sub) << 28) | (v))
/* core modes ("miss under a miss is not allowed"; DESIGN 3.4) */
enum { M_IDLE = 0, M_L2WAIT = 1, M_WAIT_DIR = 2, M_WAIT_DATA = 3, M_MEMWAIT = 4, M_L1WAIT = 5,
       M_MEMFETCH = 6 /* memory nodes (R55): waiting for a B2 fill from the memory node */ };
/* memory nodes (R55): a memory request is a DA flit, a fill flit an RA flit,
 * a writeback flit a TRAP flit, each with this payload bit (tags < 2^31) */
#define MEM_BIT 0x80000000u

#define HOLDER_NONE 0xFFFFFFFFu
#define AGE_MAX     65535u   /* R32: field width of the deflection age */
#define PEND_MAX    1023u    /* R32: field width of the pending-EV count */
#define LIFE_MAX    ((1ull << 27) - 1)  /* R32: cycles a flit may stay in the network */

typedef struct {
    int present;
    uint32_t dst, src, kind, fid;   /* struct Flit: DstX/Y, SrcX/Y, FlitId */
    uint64_t age;                   /* "incremented ... each time when it get deflected" */
    uint64_t inj;                   /* injection cycle (R1, R2) */
    uint32_t payload;               /* tag T or holder id (no FlitData, R18) */
} Flit;

typedef struct { uint32_t kind, dst, payload, nfl; } Packet;   /* ToBeSend entry */

/* L2 line: tag, LRU stamp and, with migration (NEXT-f2, R44-R52),
 * the "statistics counter" of the last N accessors as a ring,
 * the migration state and its target: MIGREQ = migration requested from the
 * directory, MIGSENT = block sent to mtarget, the source still serving
 * (P:L78), FWD = an invalid "forwarding ghost" that remembers where the
 * block went */
enum { MS_NORMAL = 0, MS_MIGREQ = 1, MS_MIGSENT = 2, MS_FWD = 3 };
#define MIG_HIST_MAX 16
typedef struct {
    int valid; uint32_t tag; uint64_t stamp;
    int mstate; uint32_t mtarget;
    uint32_t hist[MIG_HIST_MAX]; uint32_t hcount, hhead;
} Line;

typedef struct {                                               /* location array */
    uint32_t holder; uint32_t pend;
    int transit;      /* NEXT-f2: a granted migration of T is in flight (R47)  */
    int early_ev;     /* ... and its target already evicted T (R47)          */
} LocEntry;

/* private L1 line (NEXT-f1, R42): the block tag, last touch, and the node
 * whose L2 slice supplied it (where the victim writeback goes) */
typedef struct { int valid; uint32_t tag; uint64_t stamp; uint32_t owner; } L1Line;
#define WB_BIT 0x80000000u   /* an EV flit whose payload carries this bit is an L1 writeback */

typedef struct {
    Flit in[4];        /* Router.Input[4]: flits to be read this cycle        */
    Flit nin[4];       /* inputs of the next cycle, written by neighbours      */
    int has_ej;        /* Router.XToProc: the flit ejected this cycle          */
    Flit ej;
    Packet *fifo;      /* Core.ToBeSend as a FIFO of packets (R21)             */
    uint32_t cap;      /* its capacity (hub nodes may have more, R56)          */
    uint32_t head, count, next;   /* next = NextFlitAddress          */
    int mode;          /* Core.Wait, refined (DESIGN 3.4)                      */
    uint64_t ready, start;
    uint32_t tag;
    int install;
    uint32_t rx;       /* Core.ReOrderBuffer, reduced to a counter (R20)       */
    Line *l2;          /* Core.L2 LSPDSlice                                    */
    L1Line *l1;        /* Core.L1 (NEXT-f1), l1_sets x l1_ways                 */
    uint64_t script_pos, script_end;
    uint64_t script_used;
    uint64_t script_last;  /* cycle of the node's last scripted event so far (pushes, R57) */
    struct { uint32_t tag, count; int used; } migrx[4];   /* inbound B2 reassembly (R52) */
} Node;

struct orc_sim {
    orc_config cfg;
    uint32_t W, H, N;
    uint64_t t;
    Node *nodes;
    Packet *fifo_store;
    Line *l2_store;
    L1Line *l1_store;
    LocEntry *loc;
    uint64_t ntags;
    orc_event *script;
    uint64_t n_script;
    orc_counters c;
    uint64_t *hl, *hd, *ha;
    int gen_enabled;
    int debug;
    int err;
};

static __thread char g_err[512];
static void set_err(const char *msg) { snprintf(g_err, sizeof g_err, "%s", msg); }
const char *orc_last_error(void) { return g_err; }

static void fail(orc_sim *s, int code, const char *msg)
{
    if (s->err == 0) {
        s->err = code;
        snprintf(g_err, sizeof g_err, "cycle %llu: %s", (unsigned long long)s->t, msg);
    }
}

/* ------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11; Random123 constants).  Reading R25:
 * the trace source of P:L233 is replaced by a counter-based generator keyed on
 * (seed, node, cycle).
 * ---------------------------------------------------------------------- */
void orc_philox(uint32_t k0, uint32_t k1, const uint32_t cin[4], uint32_t out[4])
{
    uint32_t c0 = cin[0], c1 = cin[1], c2 = cin[2], c3 = cin[3];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void draw(const orc_sim *s, uint32_t n, uint64_t t, uint32_t r[4])
{
    uint32_t ctr[4] = { n, (uint32_t)t, (uint32_t)(t >> 32), 0u };
    orc_philox((uint32_t)s->cfg.seed, (uint32_t)(s->cfg.seed >> 32), ctr, r);
}

/* mulhi(r, m) = floor(r * m / 2^32): an integer draw in [0, m) (R25) */
static uint32_t mulhi(uint32_t r, uint32_t m) { return (uint32_t)(((uint64_t)r * m) >> 32); }

/* ------------------------------------------------------------------------
 * Mesh geometry.  x = column, y = row, North = y-1 (R10); non-toroidal (R9).
 * ---------------------------------------------------------------------- */
static uint32_t xof(const orc_sim *s, uint32_t n) { return n % s->W; }
static uint32_t yof(const orc_sim *s, uint32_t n) { return n / s->W; }

static int has_nbr(uint32_t W, uint32_t H, uint32_t n, int d)
{
    uint32_t x = n % W, y = n / W;
    switch (d) {
    case DIR_N: return y > 0;
    case DIR_S: return y + 1 < H;
    case DIR_E: return x + 1 < W;
    default:    return x > 0;
    }
}

static uint32_t nbr(uint32_t W, uint32_t n, int d)
{
    switch (d) {
    case DIR_N: return n - W;
    case DIR_S: return n + W;
    case DIR_E: return n + 1;
    default:    return n - 1;
    }
}

static int opp(int d)
{
    switch (d) {
    case DIR_N: return DIR_S;
    case DIR_S: return DIR_N;
    case DIR_E: return DIR_W;
    default:    return DIR_E;
    }
}

static int degree(uint32_t W, uint32_t H, uint32_t n)
{
    int k = 0;
    for (int d = 0; d < 4; ++d) k += has_nbr(W, H, n, d);
    return k;
}

/* ------------------------------------------------------------------------
 * Statistics helpers (R31)
 * ---------------------------------------------------------------------- */
static void hist_add(const orc_sim *s, uint64_t *h, uint64_t v)
{
    uint64_t nb = s->cfg.hist_bins;
    h[v < nb - 1 ? v : nb - 1] += 1;
}

/* ------------------------------------------------------------------------
 * Send FIFO (Core.ToBeSend; bounded, R21)
 * ---------------------------------------------------------------------- */
static void enq(orc_sim *s, uint32_t n, uint32_t kind, uint32_t dst, uint32_t payload,
                uint32_t nfl)
{
    Node *c = &s->nodes[n];
    if (dst == n) fail(s, ORC_EASSERT, "packet addressed to its own node");
    if (c->count == c->cap) {
        s->c.drops[kind] += 1;
        /* R21: an LSPD protocol message that is dropped leaves its requester
         * (or a directory entry) waiting for ever: the run is invalid */
        if (s->cfg.mode == ORC_MODE_LSPD) fail(s, ORC_EOVERFLOW, "send FIFO overflow in LSPD mode (R21)");
        return;
    }
    Packet *p = &c->fifo[(c->head + c->count) % c->cap];
    p->kind = kind; p->dst = dst; p->payload = payload; p->nfl = nfl;
    c->count += 1;
    s->c.packets_enqueued += 1;
}

/* ------------------------------------------------------------------------
 * L2 slice: set-associative, LRU with invalid-first and lowest-way ties
 * ("local victim selection"; R23, R24)
 * ---------------------------------------------------------------------- */
/* the valid line holding T in n's slice, or NULL */
static Line *l2_find(orc_sim *s, uint32_t n, uint32_t T)
{
    uint32_t set = T % s->cfg.l2_sets;
    Line *L = &s->nodes[n].l2[(uint64_t)set * s->cfg.l2_ways];
    for (uint32_t w = 0; w < s->cfg.l2_ways; ++w)
        if (L[w].valid && L[w].tag == T) return &L[w];
    return NULL;
}

/* NEXT-f2 "statistics counter ... last N accesses" (R45): a ring
 * of the last mig_hist accessor ids, oldest dropped */
static void record_access(orc_sim *s, Line *L, uint32_t who)
{
    uint32_t N = s->cfg.mig_hist;
    if (!N) return;
    if (L->hcount < N) {
        L->hist[(L->hhead + L->hcount) % N] = who;
        L->hcount += 1;
    } else {
        L->hist[L->hhead] = who;
        L->hhead = (L->hhead + 1) % N;
    }
}

/* L2HIT by accessor `who` (the owner for a local access, the requester for a
 * served RQ): stamp update (R23) and, with migration, the access record */
static int l2_hit(orc_sim *s, uint32_t n, uint32_t T, uint32_t who)
{
    Line *L = l2_find(s, n, T);
    if (!L) return 0;
    L->stamp = s->t;
    record_access(s, L, who);
    return 1;
}

/* Home node of tag T: the distributed directory (R12, T mod N) or, in the
 * centralized organisation the paper simulates (NEXT-f3),
 * the one directory node for every tag (R40). */
static uint32_t home_of(const orc_sim *s, uint32_t T)
{
    return s->cfg.dir_mode ? s->cfg.dir_node : T % s->N;
}

/* Memory-controller node k of M (mem_mode 2, R54): ceil(M/2) controllers
 * evenly spaced on the top row, the others on the bottom row */
static uint32_t mem_ctrl_node(const orc_sim *s, uint32_t k)
{
    uint32_t M = s->cfg.mem_ctrls, Mt = (M + 1) / 2, Mb = M - Mt;
    if (k < Mt) return (uint32_t)(((2ull * k + 1) * s->W) / (2ull * Mt));
    uint32_t j = k - Mt;
    return (s->H - 1) * s->W + (uint32_t)(((2ull * j + 1) * s->W) / (2ull * Mb));
}

/* The node holding block T's memory (R54) */
static uint32_t mem_node(const orc_sim *s, uint32_t T)
{
    return s->cfg.mem_mode == 1 ? home_of(s, T) : mem_ctrl_node(s, T % s->cfg.mem_ctrls);
}

/* A B2 block (Table I: 16 flits) of the given kind and payload from n to dst,
 * as packets of <= 8 flits (the send FIFO entry and fid hold 8, R50) */
static void send_b2(orc_sim *s, uint32_t n, uint32_t dst, uint32_t kind, uint32_t payload)
{
    uint32_t left = s->cfg.nfl_b2;
    while (left) {
        uint32_t k = left > 8 ? 8 : left;
        enq(s, n, kind, dst, payload, k);
        left -= k;
    }
}

/* EV handler at home h (R13): the only writer of loc[T] besides DIRSERVICE */
static void ev_handler(orc_sim *s, uint32_t h, uint32_t T, uint32_t src)
{
    (void)h;
    LocEntry *e = &s->loc[T];
    if (e->transit) {
        if (e->holder != src) {
            /* NEXT-f2 (R47): the migration target evicted T before its
             * directory update arrived; the update leaves the entry empty */
            if (e->early_ev) fail(s, ORC_EASSERT, "two early EVs during one migration");
            e->early_ev = 1;
            s->c.evs_received += 1;
            return;
        }
        e->transit = 0;   /* the source evicted T before sending it: migration aborted (R47) */
    }
    if (e->holder != src) fail(s, ORC_EASSERT, "EV from a node that is not the recorded holder");
    if (e->pend > 0) e->pend -= 1;
    else e->holder = HOLDER_NONE;
    s->c.evs_received += 1;
}

/* Replacement event "when a new cache block comes to L2 cache from main
 * memory"; the victim's directory entry is deleted by a
 * message to its home (R13). */
static void install(orc_sim *s, uint32_t n, uint32_t T)
{
    uint32_t set = T % s->cfg.l2_sets;
    Line *L = &s->nodes[n].l2[(uint64_t)set * s->cfg.l2_ways];
    uint32_t w, victim = 0;
    int found_invalid = 0;
    /* NEXT-f2: a forwarding ghost of T itself is dropped (T lives here again) */
    for (w = 0; w < s->cfg.l2_ways; ++w)
        if (!L[w].valid && L[w].mstate == MS_FWD && L[w].tag == T) { L[w].mstate = MS_NORMAL; L[w].tag = 0; L[w].mtarget = 0; }
    for (w = 0; w < s->cfg.l2_ways; ++w) {
        if (!L[w].valid) { victim = w; found_invalid = 1; break; }   /* invalid (or a ghost) first */
    }
    if (!found_invalid) {
        victim = 0;
        for (w = 1; w < s->cfg.l2_ways; ++w)
            if (L[w].stamp < L[victim].stamp) victim = w;
    }
    if (L[victim].valid) {
        uint32_t V = L[victim].tag;
        uint32_t hv = home_of(s, V);
        s->c.evictions += 1;
        if (L[victim].mstate == MS_MIGSENT) {
            /* NEXT-f2 (R49): V is already on its way to the migration target,
             * whose directory update takes the entry over: no EV */
        } else {
            s->c.evs_sent += 1;
            if (hv == n) ev_handler(s, n, V, n);
            else enq(s, n, K_EV, hv, V, 1);
        }
        /* memory nodes (R55): "The evicted block need to be written back to
         * the memory" -- a B2 block (Table I "L2 Blk Replacement",
         * 16 flits) to V's memory node, absorbed there; none if it is here */
        if (s->cfg.mem_mode && mem_node(s, V) != n) {
            s->c.mem_wbs_sent += 1;
            send_b2(s, n, mem_node(s, V), K_TRAP, V | MEM_BIT);
        }
    }
    L[victim].valid = 1;
    L[victim].tag = T;
    L[victim].stamp = s->t;
    L[victim].mstate = MS_NORMAL;          /* a fresh residency: its history holds the
                                              installing node's own access (R45) */
    L[victim].mtarget = 0;
    L[victim].hcount = 0;
    L[victim].hhead = 0;
    memset(L[victim].hist, 0, sizeof L[victim].hist);
    record_access(s, &L[victim], n);
    s->c.installs += 1;
}

/* ------------------------------------------------------------------------
 * Private write-through L1 (NEXT-f1, reading R42):
 * same block size as L2 (Table III, 43k config: 32,2,32 / 32,2,32), LRU by
 * last touch like L2 (R23).  A hit touches the line.
 * ---------------------------------------------------------------------- */
static int l1_hit(orc_sim *s, uint32_t n, uint32_t T)
{
    uint32_t set = T % s->cfg.l1_sets;
    L1Line *L = &s->nodes[n].l1[(uint64_t)set * s->cfg.l1_ways];
    for (uint32_t w = 0; w < s->cfg.l1_ways; ++w)
        if (L[w].valid && L[w].tag == T) { L[w].stamp = s->t; return 1; }
    return 0;
}

/* "A L1 cache block replacement happens when a new block comes in to local
 * L1 cache either from local L2 cache or from remote L2 cache ... The evicted
 * block need to be written back to ... corresponding L2 block":
 * the victim goes back to the slice that supplied it, as a 1-flit writeback
 * (an EV flit with WB_BIT), or is absorbed locally when that slice is ours. */
static void l1_fill(orc_sim *s, uint32_t n, uint32_t T, uint32_t owner)
{
    if (!s->cfg.l1_sets) return;
    uint32_t set = T % s->cfg.l1_sets;
    L1Line *L = &s->nodes[n].l1[(uint64_t)set * s->cfg.l1_ways];
    uint32_t w, victim = 0;
    int found_invalid = 0;
    for (w = 0; w < s->cfg.l1_ways; ++w)
        if (!L[w].valid) { victim = w; found_invalid = 1; break; }
    if (!found_invalid)
        for (w = 1; w < s->cfg.l1_ways; ++w)
            if (L[w].stamp < L[victim].stamp) victim = w;
    if (L[victim].valid) {
        s->c.wb_sent += 1;
        if (L[victim].owner == n) s->c.wb_received += 1;
        else enq(s, n, K_EV, L[victim].owner, L[victim].tag | WB_BIT, 1);
    }
    L[victim].valid = 1;
    L[victim].tag = T;
    L[victim].stamp = s->t;
    L[victim].owner = owner;
}

/* An access is complete: record its latency (R31) and free the core */
static void complete(orc_sim *s, uint32_t n)
{
    Node *c = &s->nodes[n];
    hist_add(s, s->ha, s->t - c->start);
    s->c.completed += 1;
    c->mode = M_IDLE;
}

/* Negative directory reply: fetch from memory, install at the requester
 * ("new request to next higher level memory"; P:L75 local placement). */
#define NDR_NOINSTALL 0x80000000u   /* NEXT-f2 (R47): fetch without installing */
#define NDR_PEND      0x40000000u   /* NEXT-f2 (R47): the reply counted an EV of the requester in flight */
/* A memory access of the requester n (install: R14 / R16 / R47): off-mesh at
 * the requester (R17), or -- memory nodes (R55) -- a 1-flit memory request
 * to the block's memory node, whose B2 fill is followed by the memory latency
 * at the requester; a memory node that is n itself serves it locally */
static void mem_fetch(orc_sim *s, uint32_t n, int install)
{
    Node *c = &s->nodes[n];
    s->c.mem_requests += 1;
    c->install = install;
    if (s->cfg.mem_mode && mem_node(s, c->tag) != n) {
        enq(s, n, K_DA, mem_node(s, c->tag), c->tag | MEM_BIT, 1);
        c->mode = M_MEMFETCH;
        c->rx = 0;
        return;
    }
    c->mode = M_MEMWAIT;
    c->ready = s->t + s->cfg.mem_lat;
}

static void receive_ndr(orc_sim *s, uint32_t n, uint32_t payload)
{
    Node *c = &s->nodes[n];
    if (c->mode != M_WAIT_DIR) fail(s, ORC_EASSERT, "NDR at a core that is not waiting for the directory");
    mem_fetch(s, n, (payload & NDR_NOINSTALL) ? 0 : (payload & NDR_PEND) ? 2 : 1);
}

/* Positive directory reply: request the holder (Fig. 4 step 3) */
static void receive_dr(orc_sim *s, uint32_t n, uint32_t holder)
{
    Node *c = &s->nodes[n];
    if (c->mode != M_WAIT_DIR) fail(s, ORC_EASSERT, "DR at a core that is not waiting for the directory");
    s->c.requests_made += 1;
    enq(s, n, K_RQ, holder, c->tag, 1);
    c->mode = M_WAIT_DATA;
}

/* Directory lookup at home h for requester r (Fig. 4 steps 1-2; R12-R14, R28) */
static void dir_service(orc_sim *s, uint32_t h, uint32_t T, uint32_t r)
{
    LocEntry *e = &s->loc[T];
    uint32_t kind, payload;
    s->c.dir_searches += 1;
    if (e->holder == HOLDER_NONE) {
        e->holder = r;                     /* reserve: local placement */
        kind = K_NDR; payload = T;
    } else if (e->holder == r && e->transit) {
        /* NEXT-f2 (R47): r sent T away and dropped its copy; the block is on
         * its way to the target: r fetches from memory without installing */
        kind = K_NDR; payload = T | NDR_NOINSTALL;
    } else if (e->holder == r) {
        e->pend += 1;                      /* r's EV of T is still in flight (R13) */
        if (e->pend > PEND_MAX) fail(s, ORC_EOVERFLOW, "directory pend count overflow");
        kind = K_NDR; payload = T | (s->cfg.mig_hist ? NDR_PEND : 0u);
    } else {
        kind = K_DR; payload = e->holder;
    }
    if (r == h) {                          /* loopback: no flits (R28) */
        if (kind == K_NDR) receive_ndr(s, r, payload);
        else receive_dr(s, r, payload);
    } else if (kind == K_NDR && s->cfg.mem_mode == 1) {
        /* memory at the directory (R55): "negative-DR -> memory
         * fetch is a local handoff at that node followed by a ... reply to the
         * requester": the home sends the B2 fill instead of the NDR */
        s->c.mem_fills_sent += 1;
        send_b2(s, h, r, K_RA, T | MEM_BIT);
    } else {
        enq(s, h, kind, r, payload, 1);
    }
}

/* ------------------------------------------------------------------------
 * NEXT-f2: migration and redirection (Table I; SPEC
 * S:L226-243; readings R44-R52 of DESIGN.md).
 * ---------------------------------------------------------------------- */
static void ctl_deliver(orc_sim *s, uint32_t at, uint32_t sub, uint32_t v, uint32_t src);
static void serve_rq(orc_sim *s, uint32_t n, uint32_t T, uint32_t r);

/* a 1-flit control message (sub, v) from `from` to `to`, or handled inline
 * when to == from (no flits, R51) */
static void ctl_send(orc_sim *s, uint32_t from, uint32_t to, uint32_t sub, uint32_t v)
{
    if (to == from) ctl_deliver(s, to, sub, v, from);
    else enq(s, from, K_CTL, to, CTL(sub, v), 1);
}

/* "If a remote node have accessed it mostly, then migration get triggered.
 * If a local node have accessed it most time than there is no need of
 * migration" (SPEC should_migrate S:L235-243; R46): the node with the
 * most history entries (ties: lowest id), if it is not the holder h and is
 * strictly ahead of h; else none */
static uint32_t mig_target(const orc_sim *s, const Line *L, uint32_t h)
{
    uint32_t N = s->cfg.mig_hist, best = HOLDER_NONE, bestc = 0, hc = 0;
    for (uint32_t i = 0; i < L->hcount; ++i) {
        uint32_t a = L->hist[(L->hhead + i) % N], cnt = 0;
        for (uint32_t j = 0; j < L->hcount; ++j) cnt += L->hist[(L->hhead + j) % N] == a;
        if (a == h) hc = cnt;
        if (cnt > bestc || (cnt == bestc && a < best)) { best = a; bestc = cnt; }
    }
    return (best != HOLDER_NONE && best != h && bestc > hc) ? best : HOLDER_NONE;
}

/* "The check for a local cache migration may get triggered when a request
 * comes from remote nodes": after an RQ served at h (R46, R47) */
static void maybe_migrate(orc_sim *s, uint32_t h, Line *L)
{
    if (!s->cfg.mig_hist || L->mstate != MS_NORMAL) return;
    uint32_t R = mig_target(s, L, h);
    if (R == HOLDER_NONE) return;
    L->mstate = MS_MIGREQ;
    L->mtarget = R;
    s->c.mig_requests += 1;
    ctl_send(s, h, home_of(s, L->tag), SUB_MR, L->tag);
}

/* "whole cache block will be sent/migrate to that remote node":
 * the B2 packet of nfl_b2 flits (Table I: 16), enqueued as <= 8-flit parts */
static void send_block(orc_sim *s, uint32_t h, uint32_t R, uint32_t T)
{
    uint32_t left = s->cfg.nfl_b2;
    while (left) {
        uint32_t k = left > 8 ? 8 : left;
        enq(s, h, K_CTL, R, CTL(SUB_MIG, T), k);
        left -= k;
    }
}

static void ctl_deliver(orc_sim *s, uint32_t at, uint32_t sub, uint32_t v, uint32_t src)
{
    switch (sub) {
    case SUB_MR: {   /* at home(T): grant iff src holds T, no EV of T pending, none in flight */
        LocEntry *e = &s->loc[v];
        int ok = e->holder == src && e->pend == 0 && !e->transit;
        if (ok) { e->transit = 1; e->early_ev = 0; }
        ctl_send(s, at, src, ok ? SUB_MG : SUB_MN, v);
        break;
    }
    case SUB_MG: {   /* at the holder: the block goes to the target (if still here) */
        Line *L = l2_find(s, at, v);
        if (!L || L->mstate != MS_MIGREQ) break;   /* evicted meanwhile: its EV aborts the transit (R47) */
        L->mstate = MS_MIGSENT;
        s->c.migrations += 1;
        send_block(s, at, L->mtarget, v);
        break;
    }
    case SUB_MN: {   /* refused: the line stays */
        Line *L = l2_find(s, at, v);
        s->c.mig_nacks += 1;
        if (!L || L->mstate != MS_MIGREQ) break;
        L->mstate = MS_NORMAL;
        L->mtarget = 0;
        break;
    }
    case SUB_MIG: {  /* a flit of an inbound block; the last one installs it */
        Node *c = &s->nodes[at];
        int k = -1;
        for (int i = 0; i < 4; ++i) if (c->migrx[i].used && c->migrx[i].tag == v) k = i;
        if (k < 0)
            for (int i = 0; i < 4 && k < 0; ++i) if (!c->migrx[i].used) k = i;
        if (k < 0) { fail(s, ORC_EOVERFLOW, "more than 4 inbound migrations at one node (R52)"); break; }
        if (!c->migrx[k].used) { c->migrx[k].used = 1; c->migrx[k].tag = v; c->migrx[k].count = 0; }
        c->migrx[k].count += 1;
        if (c->migrx[k].count < s->cfg.nfl_b2) break;
        c->migrx[k].used = 0; c->migrx[k].tag = 0; c->migrx[k].count = 0;
        if (l2_find(s, at, v)) { fail(s, ORC_EASSERT, "migrated block already present at the target"); break; }
        install(s, at, v);
        s->c.mig_installs += 1;
        ctl_send(s, at, home_of(s, v), SUB_DU, v);   /* "directory get updated" */
        break;
    }
    case SUB_DU: {   /* at home(T): the target holds T now; the source invalidates */
        LocEntry *e = &s->loc[v];
        if (!e->transit) { fail(s, ORC_EASSERT, "directory update without a migration in flight"); break; }
        uint32_t h = e->holder;
        e->transit = 0;
        s->c.dir_updates += 1;
        if (e->early_ev) { e->early_ev = 0; e->holder = HOLDER_NONE; }
        else e->holder = src;
        ctl_send(s, at, h, SUB_INV, v);
        break;
    }
    case SUB_INV: {  /* "source packet invalidates its copy": a forwarding ghost stays */
        Line *L = l2_find(s, at, v);
        s->c.invalidations += 1;
        if (!L || L->mstate != MS_MIGSENT) break;   /* already replaced (R49) */
        L->valid = 0;
        L->mstate = MS_FWD;                    /* tag and mtarget kept (R48) */
        L->stamp = 0;
        L->hcount = 0; L->hhead = 0;
        memset(L->hist, 0, sizeof L->hist);
        break;
    }
    case SUB_RR: {   /* "Reply redirection" (Table I; R48): ask the new holder v */
        Node *c = &s->nodes[at];
        if (c->mode != M_WAIT_DATA) { fail(s, ORC_EASSERT, "redirection at a core not waiting for data"); break; }
        s->c.rr_received += 1;
        s->c.requests_made += 1;
        if (v == at) serve_rq(s, at, c->tag, at);   /* the block came to the requester itself */
        else enq(s, at, K_RQ, v, c->tag, 1);
        break;
    }
    default:
        fail(s, ORC_EASSERT, "unknown control message");
    }
}

/* RQ for T from requester r at node n (Fig. 4 step 4): serve from the
 * slice (RA, nfl_ra flits), else redirect through a forwarding ghost
 * (NEXT-f2), else TRAP.  r == n only for a redirection to the
 * requester itself, served inline (R51). */
static void serve_rq(orc_sim *s, uint32_t n, uint32_t T, uint32_t r)
{
    s->c.requests_received += 1;
    Line *L = l2_find(s, n, T);
    if (L) {
        L->stamp = s->t;
        record_access(s, L, r);
        s->c.replies_sent += 1;
        if (r == n) {
            s->c.replies_received += 1;
            l1_fill(s, n, T, n);
            complete(s, n);
        } else {
            enq(s, n, K_RA, r, T, s->cfg.nfl_ra);
        }
        maybe_migrate(s, n, L);
        return;
    }
    if (s->cfg.mig_hist && r != n) {
        uint32_t set = T % s->cfg.l2_sets;
        Line *G = &s->nodes[n].l2[(uint64_t)set * s->cfg.l2_ways];
        for (uint32_t w = 0; w < s->cfg.l2_ways; ++w) {
            if (!G[w].valid && G[w].mstate == MS_FWD && G[w].tag == T) {
                s->c.redirections += 1;
                ctl_send(s, n, r, SUB_RR, G[w].mtarget);
                return;
            }
        }
    }
    s->c.traps_sent += 1;                         /* "send the invalid packet" */
    if (r == n) {
        Node *c = &s->nodes[n];
        s->c.traps_received += 1;
        s->c.mem_requests += 1;
        c->mode = M_MEMWAIT;
        c->install = 0;
        c->ready = s->t + s->cfg.mem_lat;
    } else {
        enq(s, n, K_TRAP, r, T, 1);
    }
}

/* The local L2 part of an access (Fig. 4): hit, else the directory */
static void l2_access(orc_sim *s, uint32_t n, uint32_t T)
{
    Node *c = &s->nodes[n];
    if (l2_hit(s, n, T, n)) {
        s->c.l2_hits += 1;
        if (s->cfg.l2_hit_lat == 0) {
            l1_fill(s, n, T, n);
            complete(s, n);
        } else {
            c->mode = M_L2WAIT;
            c->ready = s->t + s->cfg.l2_hit_lat;
        }
    } else {
        uint32_t h = home_of(s, T);        /* home node of T (R12, R40) */
        s->c.l2_misses += 1;
        c->mode = M_WAIT_DIR;
        if (h == n) dir_service(s, n, T, n);
        else enq(s, n, K_DA, h, T, 1);
    }
}

/* A new access by the core of n to block T (Phase 1; R19): the L1
 * first when there is one (a hit is served at once; a miss waits the L1 miss
 * cycles before the local L2 is accessed), else the L2 directly */
static void start_access(orc_sim *s, uint32_t n, uint32_t T)
{
    Node *c = &s->nodes[n];
    c->tag = T;
    c->start = s->t;
    c->rx = 0;
    s->c.accesses += 1;
    if (s->cfg.l1_sets) {
        if (l1_hit(s, n, T)) {
            s->c.l1_hits += 1;
            complete(s, n);
            return;
        }
        s->c.l1_misses += 1;
        c->mode = M_L1WAIT;
        c->ready = s->t + s->cfg.l1_miss_lat;
        return;
    }
    l2_access(s, n, T);
}

/* The generator call of node n at cycle t (R25, R35):
 * fires iff r0 < thr_inj.  UR: the destination is uniform over the N-1 other
 * nodes, d = mulhi(r1, N-1), skipping self.  LSPD: with probability p_priv
 * (r1 < thr_priv) a private block T = n*TPN + mulhi(r2, PRIV), else a shared
 * block T = mulhi(r2, N)*TPN + PRIV + mulhi(r3, TPN-PRIV).  Returns fire. */
static int gen_draw(const orc_sim *s, uint32_t n, uint64_t t, uint32_t *value)
{
    uint32_t r[4];
    draw(s, n, t, r);
    if (r[0] >= s->cfg.thr_inj) return 0;
    if (s->cfg.mode == ORC_MODE_UR) {
        uint32_t d = mulhi(r[1], s->N - 1);
        if (d >= n) d += 1;                  /* skip self */
        *value = d;
        return 1;
    }
    uint32_t TPN = s->cfg.tags_per_node, PRIV = s->cfg.priv_tags;
    if (r[1] < s->cfg.thr_priv)
        *value = n * TPN + mulhi(r[2], PRIV);                             /* private */
    else
        *value = mulhi(r[2], s->N) * TPN + PRIV + mulhi(r[3], TPN - PRIV); /* shared */
    return 1;
}

/* Next script event of node n that is due at cycle t, if any. */
static int script_next(orc_sim *s, uint32_t n, uint32_t *value)
{
    Node *c = &s->nodes[n];
    if (c->script_pos < c->script_end && s->script[c->script_pos].cycle <= s->t) {
        *value = s->script[c->script_pos].value;
        c->script_pos += 1;
        c->script_used += 1;
        return 1;
    }
    return 0;
}

/* ------------------------------------------------------------------------
 * Phase 1: the core step.
 * ---------------------------------------------------------------------- */
static void phase1(orc_sim *s, uint32_t n)
{
    Node *c = &s->nodes[n];
    uint32_t v;

    if (s->cfg.mode == ORC_MODE_UR) {
        /* uniform-random probes, open loop (R26) */
        if (!s->gen_enabled) return;
        uint32_t dst = 0;
        int fire = 0;
        if (script_next(s, n, &v)) {
            fire = 1; dst = v;
        } else {
            fire = gen_draw(s, n, s->t, &dst);
        }
        if (fire) {
            s->c.generated += 1;
            enq(s, n, K_PROBE, dst, 0, 1);
        }
        return;
    }

    /* LSPD */
    if (c->mode == M_L1WAIT && c->ready == s->t) l2_access(s, n, c->tag);
    if (c->mode == M_L2WAIT && c->ready == s->t) {
        l1_fill(s, n, c->tag, n);
        complete(s, n);
    }
    if (c->mode == M_MEMWAIT && c->ready == s->t) {
        if (c->install && s->cfg.mig_hist && l2_find(s, n, c->tag)) {
            /* NEXT-f2 (R47): the block migrated here while this fetch was in
             * flight: no second copy; if the directory counted an EV of ours
             * that does not exist, one is sent to even it */
            if (c->install == 2) {
                uint32_t hv = home_of(s, c->tag);
                s->c.evs_sent += 1;
                if (hv == n) ev_handler(s, n, c->tag, n);
                else enq(s, n, K_EV, hv, c->tag, 1);
            }
        } else if (c->install) {
            install(s, n, c->tag);
        }
        l1_fill(s, n, c->tag, n);                 /* R42: a memory fill is supplied locally */
        complete(s, n);
    }
    if (c->mode == M_IDLE && s->gen_enabled) {
        uint32_t T = 0;
        int fire = 0;
        if (script_next(s, n, &v)) {
            fire = 1; T = v;
        } else {
            fire = gen_draw(s, n, s->t, &T);
        }
        if (fire) start_access(s, n, T);
    }
}

/* ------------------------------------------------------------------------
 * Phase 2: "sort the all incoming flits including injection
 * flits according to age and assign output port according to their priority.
 * If there is a conflict it simply deflect to any free port except the
 * ejection port."
 * ---------------------------------------------------------------------- */
typedef struct { uint32_t dst, src; uint64_t age, inj; uint32_t fid, kind, payload; } ArbFlit;

/* 1 if a ranks strictly before b (R1, R2).  Equal (age, inj, src) happens
 * only for flits one node injected in the same cycle (fill-all injection,
 * R53): they rank by fid, kind, dst, payload ascending; flits equal in all of
 * these are identical and either order gives the same state */
static int ranks_before(uint32_t prio, const ArbFlit *a, const ArbFlit *b)
{
    if (prio == ORC_PRIO_DEFLECT && a->age != b->age) return a->age > b->age;
    if (a->inj != b->inj) return a->inj < b->inj;
    if (a->src != b->src) return a->src < b->src;
    if (a->fid != b->fid) return a->fid < b->fid;
    if (a->kind != b->kind) return a->kind < b->kind;
    if (a->dst != b->dst) return a->dst < b->dst;
    return a->payload < b->payload;
}

/* Router decision for flits F[0..nf-1] at node n.  Writes port[i] and
 * deflected[i].  Returns -1 if nf exceeds the degree. */
static int arbitrate(uint32_t W, uint32_t H, uint32_t n, uint32_t prio, uint32_t route, uint32_t nf,
                     const ArbFlit *F, int *port, int *deflected)
{
    uint32_t order[5];
    int used[4] = { 0, 0, 0, 0 };
    int eject_taken = 0;
    uint32_t x = n % W, y = n / W;

    /* at most one flit per existing port, plus one if a flit ejects (R7; the
     * NEXT-f4 injection mode can fill a router to degree + 1) */
    int at_dst = 0;
    for (uint32_t i = 0; i < nf; ++i) at_dst |= F[i].dst == n;
    if ((int)nf > degree(W, H, n) + at_dst) return -1;
    /* ranking component: "Priority Sort", insertion sort */
    for (uint32_t i = 0; i < nf; ++i) {
        uint32_t j = i;
        order[i] = i;
        while (j > 0 && ranks_before(prio, &F[order[j]], &F[order[j - 1]])) {
            uint32_t tmp = order[j]; order[j] = order[j - 1]; order[j - 1] = tmp;
            --j;
        }
    }
    /* port-selection component: "considers the flits one by one in the order
     * of their age ... assigns to each flit the output port with highest
     * priority that has not yet been assigned" */
    for (uint32_t k = 0; k < nf; ++k) {
        uint32_t i = order[k];
        const ArbFlit *f = &F[i];
        deflected[i] = 0;
        if (f->dst == n && !eject_taken) {        /* one eject link X (R6) */
            port[i] = PORT_EJECT;
            eject_taken = 1;
            continue;
        }
        if (f->dst != n) {
            uint32_t dx = f->dst % W, dy = f->dst / W;
            int p = -1;
            if (dx != x) {                         /* PMDR: x first, then y (R3) */
                int xp = dx > x ? DIR_E : DIR_W;
                if (!used[xp]) p = xp;
            }
            /* strict XY: the y-port is preferred only once dx = 0 */
            if (p < 0 && dy != y && (route == ORC_ROUTE_PMDR || dx == x)) {
                int yp = dy > y ? DIR_S : DIR_N;
                if (!used[yp]) p = yp;
            }
            if (p >= 0) {
                used[p] = 1;
                port[i] = p;
                continue;
            }
        }
        /* deflection: first free existing port in N,S,E,W (R4, R5), or in
         * N,E,S,W under the strict-XY mode */
        static const int scan_pmdr[4] = { DIR_N, DIR_S, DIR_E, DIR_W };
        static const int scan_xy[4] = { DIR_N, DIR_E, DIR_S, DIR_W };
        const int *scan = route == ORC_ROUTE_XY ? scan_xy : scan_pmdr;
        for (int k2 = 0; k2 < 4; ++k2) {
            const int d = scan[k2];
            if (has_nbr(W, H, n, d) && !used[d]) {
                used[d] = 1;
                port[i] = d;
                deflected[i] = 1;
                break;
            }
        }
    }
    return 0;
}

int orc_arbitrate_ex(uint32_t mesh_w, uint32_t mesh_h, uint32_t node, uint32_t prio, uint32_t route,
                     uint32_t nf, uint32_t stride, const uint64_t *flits, int *out_port, uint64_t *out_age)
{
    ArbFlit F[5] = {{0, 0, 0, 0, 0, 0, 0}};
    int defl[5];
    if (nf > 5 || (stride != 4 && stride != 7)) return -1;
    for (uint32_t i = 0; i < nf; ++i) {
        const uint64_t *v = flits + (size_t)stride * i;
        F[i].dst = (uint32_t)v[0];
        F[i].src = (uint32_t)v[1];
        F[i].age = v[2];
        F[i].inj = v[3];
        if (stride == 7) {
            F[i].fid = (uint32_t)v[4];
            F[i].kind = (uint32_t)v[5];
            F[i].payload = (uint32_t)v[6];
        }
    }
    if (arbitrate(mesh_w, mesh_h, node, prio, route, nf, F, out_port, defl) != 0) return -1;
    for (uint32_t i = 0; i < nf; ++i) out_age[i] = F[i].age + (uint64_t)defl[i];
    return 0;
}

int orc_arbitrate(uint32_t mesh_w, uint32_t mesh_h, uint32_t node, uint32_t prio, uint32_t route,
                  uint32_t nf, const uint64_t *flits, int *out_port, uint64_t *out_age)
{
    return orc_arbitrate_ex(mesh_w, mesh_h, node, prio, route, nf, 4, flits, out_port, out_age);
}

static void phase2(orc_sim *s, uint32_t n)
{
    Node *c = &s->nodes[n];
    Flit F[5];
    ArbFlit A[5];
    int port[5], defl[5];
    uint32_t nf = 0;
    int deg = degree(s->W, s->H, n);

    for (int d = 0; d < 4; ++d) {
        if (c->in[d].present) {
            F[nf++] = c->in[d];
            c->in[d].present = 0;
        }
    }
    /* injection: one flit per cycle through InFromProc, only if a free input
     * port exists (R7, R8); under the NEXT-f4 mode 1 (R43) a flit
     * that will eject frees its input port for the same cycle;
     * under mode 2 (R53) queued flits fill every free input port, oldest-queued
     * first, all injected this cycle (R8) */
    int frees = 0;
    if (s->cfg.inject_mode == 1)
        for (uint32_t i = 0; i < nf; ++i) frees |= F[i].dst == n;
    const uint32_t max_inj = s->cfg.inject_mode == 2 ? 4u : 1u;
    for (uint32_t k = 0; k < max_inj && (int)nf - frees < deg && c->count > 0; ++k) {
        Packet *p = &c->fifo[c->head];
        Flit f;
        f.present = 1;
        f.dst = p->dst; f.src = n; f.kind = p->kind; f.fid = c->next;
        f.age = s->cfg.age_base;                 /* "Newly injected flits age is set to zero";
                                                    age_base is a test knob, 0 by default */
        f.inj = s->t;
        f.payload = p->payload;
        F[nf++] = f;
        s->c.injected += 1;
        c->next += 1;
        if (c->next == p->nfl) {
            c->head = (c->head + 1) % c->cap;
            c->count -= 1;
            c->next = 0;
        }
    }
    if (nf == 0) return;
    for (uint32_t i = 0; i < nf; ++i) {
        A[i].dst = F[i].dst; A[i].src = F[i].src; A[i].age = F[i].age; A[i].inj = F[i].inj;
        A[i].fid = F[i].fid; A[i].kind = F[i].kind; A[i].payload = F[i].payload;
        if (s->t - F[i].inj > LIFE_MAX) fail(s, ORC_EOVERFLOW, "flit lifetime overflow");
    }
    if (arbitrate(s->W, s->H, n, s->cfg.prio, s->cfg.route, nf, A, port, defl) != 0) {
        fail(s, ORC_EASSERT, "more flits than ports at a router");
        return;
    }
    if (s->debug & ORC_DBG_INVARIANTS) {
        /* top-priority progress: the rank-1 flit ejects or takes its
         * first productive port */
        uint32_t best = 0;
        for (uint32_t i = 1; i < nf; ++i)
            if (ranks_before(s->cfg.prio, &A[i], &A[best])) best = i;
        if (defl[best]) fail(s, ORC_EASSERT, "top-priority flit was deflected");
        if (A[best].dst != n) {
            uint32_t x = xof(s, n), y = yof(s, n), dx = A[best].dst % s->W, dy = A[best].dst / s->W;
            int want = dx != x ? (dx > x ? DIR_E : DIR_W) : (dy > y ? DIR_S : DIR_N);
            if (port[best] != want) fail(s, ORC_EASSERT, "top-priority flit not on its first productive port");
        } else if (port[best] != PORT_EJECT) {
            fail(s, ORC_EASSERT, "top-priority flit at destination not ejected");
        }
    }
    for (uint32_t i = 0; i < nf; ++i) {
        Flit f = F[i];
        if (port[i] == PORT_EJECT) {
            c->has_ej = 1;
            c->ej = f;
            continue;
        }
        if (defl[i]) {
            f.age += 1;                           /* "When a flit get deflected its age get incremented" */
            s->c.deflections += 1;
            if (f.age > AGE_MAX) fail(s, ORC_EOVERFLOW, "flit age overflow");
        }
        if (!has_nbr(s->W, s->H, n, port[i])) {
            fail(s, ORC_EASSERT, "flit routed off the mesh");
            continue;
        }
        uint32_t m = nbr(s->W, n, port[i]);
        int slot = opp(port[i]);
        if (s->nodes[m].nin[slot].present) fail(s, ORC_EASSERT, "two flits on one link");
        s->nodes[m].nin[slot] = f;
        s->c.hops += 1;
    }
}

/* ------------------------------------------------------------------------
 * Phase 3: eject, re-assemble, service the
 * delivered packet (Fig. 4; trap P:L201).
 * ---------------------------------------------------------------------- */
static void phase3(orc_sim *s, uint32_t n)
{
    Node *c = &s->nodes[n];
    if (!c->has_ej) return;
    c->has_ej = 0;
    Flit f = c->ej;
    s->c.ejected += 1;
    hist_add(s, s->hl, s->t - f.inj);
    hist_add(s, s->hd, f.age);
    switch (f.kind) {
    case K_PROBE:                                 /* = K_CTL in LSPD mode (R50) */
        if (s->cfg.mode == ORC_MODE_LSPD) ctl_deliver(s, n, f.payload >> 28, f.payload & 0x0FFFFFFFu, f.src);
        else s->c.probes_delivered += 1;
        break;
    case K_DA:
        if (f.payload & MEM_BIT) {                /* memory request at a memory node (R55) */
            s->c.mem_fills_sent += 1;
            send_b2(s, n, f.src, K_RA, f.payload);
        } else {
            dir_service(s, n, f.payload, f.src);
        }
        break;
    case K_DR:
        receive_dr(s, n, f.payload);
        break;
    case K_NDR:
        receive_ndr(s, n, f.payload);
        break;
    case K_RQ:
        serve_rq(s, n, f.payload, f.src);
        break;
    case K_RA:
        if (f.payload & MEM_BIT) {                /* a flit of a B2 memory fill (R55) */
            if (c->mode != M_MEMFETCH && c->mode != M_WAIT_DIR) fail(s, ORC_EASSERT, "fill flit at a core not fetching");
            if ((f.payload & ~MEM_BIT) != c->tag) fail(s, ORC_EASSERT, "fill flit of another block");
            c->rx += 1;
            if (c->rx == s->cfg.nfl_b2) {
                c->rx = 0;
                s->c.mem_fills_received += 1;
                if (c->mode == M_WAIT_DIR) {      /* the home's memory answered the DA (mem_mode 1) */
                    s->c.mem_requests += 1;
                    c->install = 1;
                }
                c->mode = M_MEMWAIT;
                c->ready = s->t + s->cfg.mem_lat;
            }
            break;
        }
        if (c->mode != M_WAIT_DATA) fail(s, ORC_EASSERT, "RA flit at a core not waiting for data");
        c->rx += 1;
        if (c->rx == s->cfg.nfl_ra) {
            c->rx = 0;
            s->c.replies_received += 1;
            l1_fill(s, n, c->tag, f.src);         /* supplied by the holder's slice */
            complete(s, n);
        }
        break;
    case K_TRAP:
        if (f.payload & MEM_BIT) {                /* a writeback flit at a memory node: absorbed (R55) */
            s->c.mem_wb_flits += 1;
            break;
        }
        if (c->mode != M_WAIT_DATA) fail(s, ORC_EASSERT, "TRAP at a core not waiting for data");
        s->c.traps_received += 1;
        mem_fetch(s, n, 0);                       /* R16: no install */
        break;
    case K_EV:
        if (f.payload & WB_BIT) s->c.wb_received += 1;   /* L1 writeback: absorbed (R42) */
        else ev_handler(s, n, f.payload, f.src);
        break;
    default:
        fail(s, ORC_EASSERT, "unknown flit kind");
    }
}

/* ------------------------------------------------------------------------
 * Debug invariants (DESIGN 3.5 / SURVEY P2, P3, P9)
 * ---------------------------------------------------------------------- */
static void check_invariants(orc_sim *s)
{
    int64_t occ = 0;
    for (uint32_t n = 0; n < s->N; ++n) {
        int k = 0;
        for (int d = 0; d < 4; ++d) {
            if (s->nodes[n].in[d].present) {
                ++k;
                if (!has_nbr(s->W, s->H, n, d)) fail(s, ORC_EASSERT, "flit on a missing link");
            }
        }
        if (k > degree(s->W, s->H, n)) fail(s, ORC_EASSERT, "more flits than degree");
        occ += k;
    }
    if (s->c.injected != s->c.ejected + occ) fail(s, ORC_EASSERT, "flit conservation violated");
    if (s->cfg.mode == ORC_MODE_LSPD) {
        /* single copy: each T valid in <= 1 slice; holder NONE => pend 0 */
        uint32_t lines = s->cfg.l2_sets * s->cfg.l2_ways;
        uint8_t *seen = calloc(s->ntags, 1);
        if (!seen) return;
        for (uint32_t n = 0; n < s->N; ++n)
            for (uint32_t i = 0; i < lines; ++i) {
                Line *L = &s->nodes[n].l2[i];
                if (!L->valid || L->mstate == MS_MIGSENT) continue;   /* + one source copy in transit (R47) */
                if (seen[L->tag]) fail(s, ORC_EASSERT, "block valid in two slices");
                seen[L->tag] = 1;
            }
        free(seen);
        for (uint64_t T = 0; T < s->ntags; ++T)
            if (s->loc[T].holder == HOLDER_NONE && s->loc[T].pend != 0)
                fail(s, ORC_EASSERT, "pend without holder");
    }
}

/* ------------------------------------------------------------------------
 * One simulated cycle: the serial main loop body.
 * ---------------------------------------------------------------------- */
static void cycle(orc_sim *s)
{
    uint32_t N = s->N;
    int rev = (s->debug & ORC_DBG_REVERSE) != 0;
    for (uint32_t i = 0; i < N; ++i) phase1(s, rev ? N - 1 - i : i);
    for (uint32_t i = 0; i < N; ++i) phase2(s, rev ? N - 1 - i : i);
    for (uint32_t i = 0; i < N; ++i) phase3(s, rev ? N - 1 - i : i);
    /* transfer: outputs of t become the inputs of t+1 (R11) */
    for (uint32_t n = 0; n < N; ++n) {
        Node *c = &s->nodes[n];
        for (int d = 0; d < 4; ++d) {
            c->in[d] = c->nin[d];
            c->nin[d].present = 0;
        }
    }
    s->t += 1;
    s->c.cycle = (int64_t)s->t;
    if (s->debug & ORC_DBG_INVARIANTS) check_invariants(s);
}

/* ------------------------------------------------------------------------
 * Public API
 * ---------------------------------------------------------------------- */
static int cmp_event(const void *a, const void *b)
{
    const orc_event *x = a, *y = b;
    if (x->node != y->node) return x->node < y->node ? -1 : 1;
    if (x->cycle != y->cycle) return x->cycle < y->cycle ? -1 : 1;
    return 0;
}

int orc_create(const orc_config *cfg, orc_sim **out)
{
    *out = NULL;
    if (!cfg) { set_err("null config"); return ORC_EINVAL; }
    uint32_t W = cfg->mesh_w, H = cfg->mesh_h;
    if (W < 2 || H < 2 || W > 2048 || H > 2048 || (uint64_t)W * H > (1u << 21)) {
        set_err("mesh must be 2..2048 per side and at most 2^21 nodes"); return ORC_EINVAL;
    }
    if (cfg->mode > 1 || cfg->prio > 1 || cfg->route > 1 || cfg->inject_mode > 2) {
        set_err("bad mode/prio/route/inject_mode");
        return ORC_EINVAL;
    }
    if (cfg->mode == ORC_MODE_LSPD && cfg->l1_sets &&
        (cfg->l1_sets > 65536 || cfg->l1_ways < 1 || cfg->l1_ways > 16 || cfg->l1_miss_lat < 1 ||
         cfg->l1_miss_lat >= (1u << 29))) {
        set_err("l1 geometry: sets 0..65536, ways 1..16, miss latency 1..2^29-1");
        return ORC_EINVAL;
    }
    if (cfg->dir_mode > 1 || (cfg->dir_mode && (uint64_t)cfg->dir_node >= (uint64_t)cfg->mesh_w * cfg->mesh_h)) {
        set_err("bad dir_mode/dir_node");
        return ORC_EINVAL;
    }
    if (cfg->sendq_cap == 0 || cfg->sendq_cap > 1024 || (cfg->sendq_cap & (cfg->sendq_cap - 1))) {
        set_err("sendq_cap must be a power of two in 1..1024"); return ORC_EINVAL;
    }
    if (cfg->hist_bins == 0 || cfg->hist_bins > 65536) { set_err("hist_bins must be 1..65536"); return ORC_EINVAL; }
    if (cfg->age_base > AGE_MAX) { set_err("age_base > 65535 (R32)"); return ORC_EINVAL; }
    if (cfg->mig_hist > MIG_HIST_MAX) { set_err("mig_hist must be 0..16"); return ORC_EINVAL; }
    if (cfg->mig_hist && (cfg->mode != ORC_MODE_LSPD || cfg->nfl_b2 < 1 || cfg->nfl_b2 > 16 ||
                          (uint64_t)cfg->tags_per_node * cfg->mesh_w * cfg->mesh_h > (1ull << 28))) {
        set_err("migration needs LSPD mode, nfl_b2 1..16 and a tag space <= 2^28 (R50)");
        return ORC_EINVAL;
    }
    if (cfg->nfl_ra < 1 || cfg->nfl_ra > 8) { set_err("nfl_ra must be 1..8"); return ORC_EINVAL; }
    if (cfg->mem_mode > 2 || (cfg->mem_mode && (cfg->mode != ORC_MODE_LSPD || cfg->mig_hist ||
                                                cfg->nfl_b2 < 1 || cfg->nfl_b2 > 16))) {
        set_err("memory nodes (mem_mode 1/2) need LSPD mode, no migration and nfl_b2 1..16 (R54)");
        return ORC_EINVAL;
    }
    if (cfg->mem_mode == 2 && (cfg->mem_ctrls < 1 || cfg->mem_ctrls > 64 || (cfg->mem_ctrls + 1) / 2 > W)) {
        set_err("mem_ctrls must be 1..64 with ceil(M/2) <= mesh_w"); return ORC_EINVAL;
    }
    if (cfg->hub_sendq_cap && (cfg->hub_sendq_cap < cfg->sendq_cap || cfg->hub_sendq_cap > 1024 ||
                               (cfg->hub_sendq_cap & (cfg->hub_sendq_cap - 1)))) {
        set_err("hub_sendq_cap must be 0 or a power of two in sendq_cap..1024"); return ORC_EINVAL;
    }
    uint64_t N = (uint64_t)W * H;
    if (cfg->mode == ORC_MODE_LSPD) {
        if (cfg->l2_sets < 1 || cfg->l2_sets > 65536 || cfg->l2_ways < 1 || cfg->l2_ways > 16) {
            set_err("l2 geometry out of range"); return ORC_EINVAL;
        }
        if (cfg->tags_per_node < 2 || cfg->priv_tags < 1 || cfg->priv_tags >= cfg->tags_per_node) {
            set_err("need 1 <= priv_tags < tags_per_node"); return ORC_EINVAL;
        }
        if ((uint64_t)cfg->tags_per_node * N > (1ull << 31)) { set_err("tag space exceeds 2^31"); return ORC_EINVAL; }
        if (cfg->mem_lat < 1 || cfg->mem_lat >= (1u << 30) || cfg->l2_hit_lat >= (1u << 30)) {
            set_err("latency out of range"); return ORC_EINVAL;
        }
    }
    for (uint64_t i = 0; i < cfg->n_script; ++i) {
        const orc_event *e = &cfg->script[i];
        if (e->node >= N) { set_err("script node out of range"); return ORC_EINVAL; }
        if (cfg->mode == ORC_MODE_UR && (e->value >= N || e->value == e->node)) {
            set_err("script probe destination invalid"); return ORC_EINVAL;
        }
        if (cfg->mode == ORC_MODE_LSPD && (uint64_t)e->value >= (uint64_t)cfg->tags_per_node * N) {
            set_err("script tag out of range"); return ORC_EINVAL;
        }
    }

    orc_sim *s = calloc(1, sizeof *s);
    if (!s) { set_err("out of memory"); return ORC_ENOMEM; }
    s->cfg = *cfg;
    s->W = W; s->H = H; s->N = (uint32_t)N;
    s->gen_enabled = 1;
    s->nodes = calloc(N, sizeof(Node));
    /* hub nodes (R56): the central directory node and the memory controllers */
    const uint32_t hub_cap = cfg->hub_sendq_cap ? cfg->hub_sendq_cap : cfg->sendq_cap;
    s->fifo_store = calloc(N * cfg->sendq_cap + (uint64_t)65 * hub_cap, sizeof(Packet));
    s->hl = calloc(cfg->hist_bins, sizeof(uint64_t));
    s->hd = calloc(cfg->hist_bins, sizeof(uint64_t));
    s->ha = calloc(cfg->hist_bins, sizeof(uint64_t));
    int bad = !s->nodes || !s->fifo_store || !s->hl || !s->hd || !s->ha;
    if (cfg->mode == ORC_MODE_LSPD && !bad) {
        uint64_t lines = (uint64_t)cfg->l2_sets * cfg->l2_ways;
        s->ntags = (uint64_t)cfg->tags_per_node * N;
        s->l2_store = calloc(N * lines, sizeof(Line));
        s->loc = malloc(s->ntags * sizeof(LocEntry));
        const uint64_t l1lines = (uint64_t)cfg->l1_sets * cfg->l1_ways;
        s->l1_store = calloc(N * l1lines + 1, sizeof(L1Line));
        bad = !s->l2_store || !s->loc || !s->l1_store;
        if (!bad) {
            for (uint64_t T = 0; T < s->ntags; ++T) {
                s->loc[T].holder = HOLDER_NONE; s->loc[T].pend = 0; s->loc[T].transit = 0; s->loc[T].early_ev = 0;
            }
            for (uint64_t n = 0; n < N; ++n) {
                s->nodes[n].l2 = &s->l2_store[n * lines];
                s->nodes[n].l1 = &s->l1_store[n * l1lines];
            }
        }
    }
    if (cfg->n_script && !bad) {
        s->script = malloc(cfg->n_script * sizeof(orc_event));
        bad = !s->script;
        if (!bad) {
            memcpy(s->script, cfg->script, cfg->n_script * sizeof(orc_event));
            /* stable order per node: (node, cycle), ties keep input order */
            for (uint64_t i = 1; i < cfg->n_script; ++i) {      /* insertion sort: stable */
                orc_event e = s->script[i];
                uint64_t j = i;
                while (j > 0 && cmp_event(&e, &s->script[j - 1]) < 0) { s->script[j] = s->script[j - 1]; --j; }
                s->script[j] = e;
            }
        }
    }
    s->cfg.script = NULL;
    if (bad) { orc_destroy(s); set_err("out of memory"); return ORC_ENOMEM; }
    for (uint64_t n = 0; n < N; ++n) {
        s->nodes[n].fifo = &s->fifo_store[n * cfg->sendq_cap];
        s->nodes[n].cap = cfg->sendq_cap;
        s->nodes[n].mode = M_IDLE;
    }
    {
        Packet *next = &s->fifo_store[N * cfg->sendq_cap];   /* hub FIFOs after the ordinary ones */
        uint32_t hubs[65], nh = 0;
        if (cfg->dir_mode == 1) hubs[nh++] = cfg->dir_node;
        if (cfg->mem_mode == 2)
            for (uint32_t k = 0; k < cfg->mem_ctrls; ++k) hubs[nh++] = mem_ctrl_node(s, k);
        for (uint32_t i = 0; i < nh; ++i) {
            Node *c = &s->nodes[hubs[i]];
            if (c->fifo >= &s->fifo_store[N * cfg->sendq_cap]) continue;   /* listed twice */
            c->fifo = next;
            c->cap = hub_cap;
            next += hub_cap;
        }
    }
    {
        uint64_t i = 0;
        for (uint64_t n = 0; n < N; ++n) {
            s->nodes[n].script_pos = i;
            while (i < cfg->n_script && s->script[i].node == n) s->nodes[n].script_last = s->script[i++].cycle;
            s->nodes[n].script_end = i;
        }
    }
    s->n_script = cfg->n_script;
    *out = s;
    return ORC_OK;
}

static int check_event(const orc_sim *s, const orc_event *e)
{
    if (e->node >= s->N) { set_err("script node out of range"); return ORC_EINVAL; }
    if (s->cfg.mode == ORC_MODE_UR && (e->value >= s->N || e->value == e->node)) {
        set_err("script probe destination invalid"); return ORC_EINVAL;
    }
    if (s->cfg.mode == ORC_MODE_LSPD && (uint64_t)e->value >= (uint64_t)s->cfg.tags_per_node * s->N) {
        set_err("script tag out of range"); return ORC_EINVAL;
    }
    return ORC_OK;
}

/* NEXT-f3 streamed trace replay (R57): append events to the nodes' script
 * queues.  The pushed events are ordered per node by cycle (stable, as at
 * create); a node's first pushed event may not be earlier than its last event
 * so far, so each node's queue stays ordered and a script pushed in pieces
 * before its events are due behaves as the whole script given at create.
 * Consumed events are dropped (the queues hold only what is still to come). */
int orc_push_script(orc_sim *s, const orc_event *ev, uint64_t n)
{
    if (s->err) return s->err;
    if (n && !ev) { set_err("null events"); return ORC_EINVAL; }
    orc_event *add = malloc((n ? n : 1) * sizeof(orc_event));
    uint64_t *cnt = calloc(s->N + 1, sizeof(uint64_t));
    if (!add || !cnt) { free(add); free(cnt); set_err("out of memory"); return ORC_ENOMEM; }
    for (uint64_t i = 0; i < n; ++i) {
        int rc = check_event(s, &ev[i]);
        if (rc) { free(add); free(cnt); return rc; }
        orc_event e = ev[i];                      /* stable insertion sort by (node, cycle) */
        uint64_t j = i;
        while (j > 0 && cmp_event(&e, &add[j - 1]) < 0) { add[j] = add[j - 1]; --j; }
        add[j] = e;
    }
    for (uint64_t i = 0; i < n; ++i) {
        const Node *c = &s->nodes[add[i].node];
        int first = i == 0 || add[i - 1].node != add[i].node;
        if (first && (c->script_used || c->script_end > c->script_pos) && add[i].cycle < c->script_last) {
            free(add); free(cnt);
            set_err("pushed events of a node must not precede its earlier events");
            return ORC_EINVAL;
        }
        cnt[add[i].node] += 1;
    }
    uint64_t total = n;
    for (uint32_t v = 0; v < s->N; ++v) total += s->nodes[v].script_end - s->nodes[v].script_pos;
    orc_event *ns = malloc((total ? total : 1) * sizeof(orc_event));
    if (!ns) { free(add); free(cnt); set_err("out of memory"); return ORC_ENOMEM; }
    uint64_t k = 0, a = 0;
    for (uint32_t v = 0; v < s->N; ++v) {
        Node *c = &s->nodes[v];
        const uint64_t p0 = k;
        for (uint64_t i = c->script_pos; i < c->script_end; ++i) ns[k++] = s->script[i];   /* still to come */
        for (uint64_t i = 0; i < cnt[v]; ++i) { ns[k] = add[a++]; c->script_last = ns[k].cycle; ++k; }
        c->script_pos = p0;
        c->script_end = k;
    }
    free(s->script);
    s->script = ns;
    s->n_script = total;
    free(add);
    free(cnt);
    return ORC_OK;
}

void orc_destroy(orc_sim *s)
{
    if (!s) return;
    free(s->nodes); free(s->fifo_store); free(s->l2_store); free(s->l1_store); free(s->loc);
    free(s->script); free(s->hl); free(s->hd); free(s->ha);
    free(s);
}

int orc_set_debug(orc_sim *s, int flags) { s->debug = flags; return ORC_OK; }

int orc_run(orc_sim *s, uint64_t n_cycles)
{
    if (s->err) return s->err;
    for (uint64_t i = 0; i < n_cycles && !s->err; ++i) cycle(s);
    return s->err;
}

static int quiescent(const orc_sim *s)
{
    for (uint32_t n = 0; n < s->N; ++n) {
        const Node *c = &s->nodes[n];
        if (c->count || c->mode != M_IDLE) return 0;
        for (int d = 0; d < 4; ++d) if (c->in[d].present) return 0;
    }
    return 1;
}

/* run with generation disabled until quiescent (R30) */
int orc_drain(orc_sim *s, uint64_t max_cycles, uint64_t *used, int *drained)
{
    uint64_t k = 0;
    int q;
    if (s->err) return s->err;
    s->gen_enabled = 0;
    while (!(q = quiescent(s)) && k < max_cycles && !s->err) { cycle(s); ++k; }
    s->gen_enabled = 1;
    if (used) *used = k;
    if (drained) *drained = q;
    return s->err;
}

int orc_stats(const orc_sim *s, orc_counters *out, uint64_t *hl, uint64_t *hd, uint64_t *ha,
              uint32_t nbins)
{
    if (out) *out = s->c;
    if (hl || hd || ha) {
        if (nbins != s->cfg.hist_bins) { set_err("nbins mismatch"); return ORC_EINVAL; }
        if (hl) memcpy(hl, s->hl, nbins * sizeof(uint64_t));
        if (hd) memcpy(hd, s->hd, nbins * sizeof(uint64_t));
        if (ha) memcpy(ha, s->ha, nbins * sizeof(uint64_t));
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------
 * Canonical state hash (DESIGN 3.7): sum over (domain, index, tuple) of
 * mix(mix(dom<<56 ^ index) ^ tuplehash) mod 2^64.
 * ---------------------------------------------------------------------- */
static uint64_t mix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static uint64_t tuple_hash(const uint64_t *v, int k)
{
    uint64_t h = (uint64_t)k;
    for (int i = 0; i < k; ++i) h = mix64(h ^ v[i]);
    return h;
}

static uint64_t term(uint64_t dom, uint64_t idx, const uint64_t *v, int k)
{
    return mix64(mix64((dom << 56) ^ idx) ^ tuple_hash(v, k));
}

enum { D_LINK = 1, D_FIFO = 2, D_FIFONEXT = 3, D_CORE = 4, D_L2 = 5, D_LOC = 6,
       D_CNT = 7, D_HIST = 8, D_CYCLE = 9, D_SCRIPT = 10, D_L1 = 11, D_L2MIG = 12, D_LOCMIG = 13,
       D_MIGRX = 14 };

uint64_t orc_state_hash(const orc_sim *s)
{
    uint64_t H = 0, v[8];
    for (uint32_t n = 0; n < s->N; ++n) {
        const Node *c = &s->nodes[n];
        for (int d = 0; d < 4; ++d) {
            const Flit *f = &c->in[d];
            if (!f->present) continue;
            v[0] = f->dst; v[1] = f->src; v[2] = f->kind; v[3] = f->fid;
            v[4] = f->payload; v[5] = f->age; v[6] = f->inj;
            H += term(D_LINK, (uint64_t)n * 4 + d, v, 7);
        }
        for (uint32_t k = 0; k < c->count; ++k) {
            const Packet *p = &c->fifo[(c->head + k) % c->cap];
            v[0] = p->kind; v[1] = p->dst; v[2] = p->payload; v[3] = p->nfl;
            H += term(D_FIFO, ((uint64_t)n << 16) + k, v, 4);
        }
        if (c->next) { v[0] = c->next; H += term(D_FIFONEXT, n, v, 1); }
        if (c->mode != M_IDLE) {
            uint64_t ready = 0, tag = 0, inst = 0, start = c->start, rx = 0;
            switch (c->mode) {
            case M_L2WAIT:    ready = c->ready; break;
            case M_WAIT_DIR:  tag = c->tag; break;
            case M_WAIT_DATA: tag = c->tag; rx = c->rx; break;
            case M_MEMWAIT:   ready = c->ready; tag = c->tag; inst = (uint64_t)c->install; break;
            case M_L1WAIT:    ready = c->ready; tag = c->tag; break;
            case M_MEMFETCH:  tag = c->tag; inst = (uint64_t)c->install; rx = c->rx; break;
            }
            v[0] = (uint64_t)c->mode; v[1] = ready; v[2] = tag; v[3] = inst; v[4] = start; v[5] = rx;
            H += term(D_CORE, n, v, 6);
        }
        if (s->cfg.mode == ORC_MODE_LSPD) {
            uint32_t S = s->cfg.l2_sets, Wy = s->cfg.l2_ways;
            for (uint32_t st = 0; st < S; ++st)
                for (uint32_t w = 0; w < Wy; ++w) {
                    const Line *L = &c->l2[(uint64_t)st * Wy + w];
                    if (!L->valid) continue;
                    v[0] = L->tag; v[1] = L->stamp;
                    H += term(D_L2, ((uint64_t)n * S + st) * Wy + w, v, 2);
                }
        }
        if (s->cfg.mode == ORC_MODE_LSPD && s->cfg.l1_sets) {
            uint32_t S = s->cfg.l1_sets, Wy = s->cfg.l1_ways;
            for (uint32_t st = 0; st < S; ++st)
                for (uint32_t w = 0; w < Wy; ++w) {
                    const L1Line *L = &c->l1[(uint64_t)st * Wy + w];
                    if (!L->valid) continue;
                    v[0] = L->tag; v[1] = L->stamp; v[2] = L->owner;
                    H += term(D_L1, ((uint64_t)n * S + st) * Wy + w, v, 3);
                }
        }
        if (c->script_used) { v[0] = c->script_used; H += term(D_SCRIPT, n, v, 1); }
        if (s->cfg.mode == ORC_MODE_LSPD && s->cfg.mig_hist) {
            /* NEXT-f2: per line (state, target, history oldest first) when any is set */
            uint32_t S = s->cfg.l2_sets, Wy = s->cfg.l2_ways;
            for (uint32_t st = 0; st < S; ++st)
                for (uint32_t w = 0; w < Wy; ++w) {
                    const Line *L = &c->l2[(uint64_t)st * Wy + w];
                    if (L->mstate == MS_NORMAL && (!L->valid || L->hcount == 0)) continue;
                    uint64_t u[4 + MIG_HIST_MAX];
                    int k = 0;
                    u[k++] = (uint64_t)L->mstate; u[k++] = L->tag; u[k++] = L->mtarget; u[k++] = L->hcount;
                    for (uint32_t i = 0; i < L->hcount; ++i) u[k++] = L->hist[(L->hhead + i) % s->cfg.mig_hist];
                    H += mix64(mix64(((uint64_t)D_L2MIG << 56) ^ (((uint64_t)n * S + st) * Wy + w)) ^ tuple_hash(u, k));
                }
            for (int i = 0; i < 4; ++i)
                if (c->migrx[i].used) {
                    v[0] = c->migrx[i].tag; v[1] = c->migrx[i].count;
                    H += term(D_MIGRX, ((uint64_t)n << 2) + (uint64_t)i, v, 2);
                }
        }
    }
    for (uint64_t T = 0; T < s->ntags; ++T) {
        const LocEntry *e = &s->loc[T];
        if (e->transit || e->early_ev) {
            v[0] = (uint64_t)e->transit; v[1] = (uint64_t)e->early_ev;
            H += term(D_LOCMIG, T, v, 2);
        }
        if (e->holder == HOLDER_NONE && e->pend == 0) continue;
        v[0] = e->holder == HOLDER_NONE ? 0 : (uint64_t)e->holder + 1;
        v[1] = e->pend;
        H += term(D_LOC, T, v, 2);
    }
    {
        const int64_t *cnt = &s->c.generated;      /* generated .. drops[7] */
        int ncnt = (int)((sizeof(orc_counters) - sizeof(int64_t)) / sizeof(int64_t));
        for (int i = 0; i < ncnt; ++i) { v[0] = (uint64_t)cnt[i]; H += term(D_CNT, (uint64_t)i, v, 1); }
    }
    {
        const uint64_t *hs[3] = { s->hl, s->hd, s->ha };
        for (int h = 0; h < 3; ++h)
            for (uint32_t b = 0; b < s->cfg.hist_bins; ++b)
                if (hs[h][b]) { v[0] = hs[h][b]; H += term(D_HIST, ((uint64_t)h << 32) + b, v, 1); }
    }
    v[0] = s->t;
    H += term(D_CYCLE, 0, v, 1);
    return H;
}

/* ------------------------------------------------------------------------
 * Test peeks
 * ---------------------------------------------------------------------- */
int64_t orc_links_occupied(const orc_sim *s, int64_t *age_sum)
{
    int64_t k = 0, a = 0;
    for (uint32_t n = 0; n < s->N; ++n)
        for (int d = 0; d < 4; ++d)
            if (s->nodes[n].in[d].present) { ++k; a += (int64_t)s->nodes[n].in[d].age; }
    if (age_sum) *age_sum = a;
    return k;
}

int64_t orc_fifo_packets(const orc_sim *s)
{
    int64_t k = 0;
    for (uint32_t n = 0; n < s->N; ++n) k += s->nodes[n].count;
    return k;
}

int64_t orc_cores_busy(const orc_sim *s)
{
    int64_t k = 0;
    for (uint32_t n = 0; n < s->N; ++n) k += s->nodes[n].mode != M_IDLE;
    return k;
}

int orc_check_directory_quiescent(const orc_sim *s)
{
    if (s->cfg.mode != ORC_MODE_LSPD) return 0;
    uint32_t lines = s->cfg.l2_sets * s->cfg.l2_ways;
    uint32_t *holder = malloc(s->ntags * sizeof(uint32_t));
    if (!holder) return -2;
    for (uint64_t T = 0; T < s->ntags; ++T) holder[T] = HOLDER_NONE;
    int bad = 0;
    for (uint32_t n = 0; n < s->N; ++n)
        for (uint32_t i = 0; i < lines; ++i) {
            const Line *L = &s->nodes[n].l2[i];
            if (!L->valid) continue;
            if (holder[L->tag] != HOLDER_NONE) bad = 1;
            holder[L->tag] = n;
        }
    for (uint64_t T = 0; T < s->ntags && !bad; ++T) {
        if (s->loc[T].holder != holder[T] || s->loc[T].pend != 0 || s->loc[T].transit || s->loc[T].early_ev) bad = 1;
    }
    free(holder);
    return bad ? -1 : 0;
}

int orc_core(const orc_sim *s, uint32_t n, uint64_t out[6])
{
    if (n >= s->N) return ORC_EINVAL;
    const Node *c = &s->nodes[n];
    out[0] = (uint64_t)c->mode; out[1] = c->ready; out[2] = c->tag;
    out[3] = (uint64_t)c->install; out[4] = c->start; out[5] = c->rx;
    return ORC_OK;
}

int orc_l2_line(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way, uint64_t out[3])
{
    if (s->cfg.mode != ORC_MODE_LSPD || n >= s->N || set >= s->cfg.l2_sets || way >= s->cfg.l2_ways)
        return ORC_EINVAL;
    const Line *L = &s->nodes[n].l2[(uint64_t)set * s->cfg.l2_ways + way];
    out[0] = (uint64_t)L->valid; out[1] = L->tag; out[2] = L->stamp;
    return ORC_OK;
}

int orc_loc(const orc_sim *s, uint32_t T, uint64_t out[2])
{
    if (T >= s->ntags) return ORC_EINVAL;
    out[0] = s->loc[T].holder; out[1] = s->loc[T].pend;
    return ORC_OK;
}

/* Link input slot d of node n (the inputs of the next cycle to run):
 * present, dst, src, kind, fid, payload, age, inj. */
int orc_link(const orc_sim *s, uint32_t n, uint32_t d, uint64_t out[8])
{
    if (n >= s->N || d >= 4) return ORC_EINVAL;
    const Flit *f = &s->nodes[n].in[d];
    out[0] = (uint64_t)f->present; out[1] = f->dst; out[2] = f->src; out[3] = f->kind;
    out[4] = f->fid; out[5] = f->payload; out[6] = f->age; out[7] = f->inj;
    return ORC_OK;
}

/* Send FIFO of node n: count and next-flit index (out[0..1]); packet k from
 * the head (k < count): kind, dst, payload, nfl (pkt[0..3]). */
int orc_fifo(const orc_sim *s, uint32_t n, uint32_t k, uint64_t out[2], uint64_t pkt[4])
{
    if (n >= s->N) return ORC_EINVAL;
    const Node *c = &s->nodes[n];
    out[0] = c->count; out[1] = c->next;
    if (k < c->count) {
        const Packet *p = &c->fifo[(c->head + k) % c->cap];
        pkt[0] = p->kind; pkt[1] = p->dst; pkt[2] = p->payload; pkt[3] = p->nfl;
    }
    return ORC_OK;
}

/* NEXT-f1 L1 line (n, set, way): valid, tag, stamp, owner. */
int orc_l1_line(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way, uint64_t out[4])
{
    if (!s->cfg.l1_sets || n >= s->N || set >= s->cfg.l1_sets || way >= s->cfg.l1_ways) return ORC_EINVAL;
    const L1Line *L = &s->nodes[n].l1[(uint64_t)set * s->cfg.l1_ways + way];
    out[0] = (uint64_t)L->valid; out[1] = L->tag; out[2] = L->stamp; out[3] = L->owner;
    return ORC_OK;
}

/* Script events consumed by node n. */
int64_t orc_script_used(const orc_sim *s, uint32_t n)
{
    return n < s->N ? (int64_t)s->nodes[n].script_used : -1;
}

/* The generator call the simulation makes for node n at cycle t (gen_draw):
 * out[0] = fired, out[1] = UR destination or LSPD block tag. */
int orc_gen(const orc_sim *s, uint32_t n, uint64_t t, uint64_t out[2])
{
    if (n >= s->N) return ORC_EINVAL;
    uint32_t v = 0;
    out[0] = (uint64_t)gen_draw(s, n, t, &v);
    out[1] = v;
    return ORC_OK;
}

/* Test-only mutation of one state field (hash sensitivity pins):
 *   field 0 link slot (n, i=d) age += value      1 link slot (n, i=d) payload ^= value
 *   2 core (n) start += value                    3 core (n) mode = value
 *   4 L2 line (n, i=set, j=way) stamp += value   5 loc entry (T=n) pend += value
 *   6 FIFO packet (n, i=k) payload ^= value      7 FIFO next (n) = value
 *   8 counter index i += value                   9 histogram (i=which, j=bin) += value
 *  10 cycle += value                            11 L1 line (n, i, j) owner ^= value
 *  12 core (n) rx += value                      13 core (n) ready += value */
int orc_poke(orc_sim *s, uint32_t field, uint32_t n, uint32_t i, uint32_t j, uint64_t value)
{
    Node *c = n < s->N ? &s->nodes[n] : NULL;
    switch (field) {
    case 0: if (!c || i >= 4) return ORC_EINVAL; c->in[i].age += value; return ORC_OK;
    case 1: if (!c || i >= 4) return ORC_EINVAL; c->in[i].payload ^= (uint32_t)value; return ORC_OK;
    case 2: if (!c) return ORC_EINVAL; c->start += value; return ORC_OK;
    case 3: if (!c) return ORC_EINVAL; c->mode = (int)value; return ORC_OK;
    case 4:
        if (!c || s->cfg.mode != ORC_MODE_LSPD || i >= s->cfg.l2_sets || j >= s->cfg.l2_ways) return ORC_EINVAL;
        c->l2[(uint64_t)i * s->cfg.l2_ways + j].stamp += value; return ORC_OK;
    case 5: if (n >= s->ntags) return ORC_EINVAL; s->loc[n].pend += (uint32_t)value; return ORC_OK;
    case 6:
        if (!c || i >= c->count) return ORC_EINVAL;
        c->fifo[(c->head + i) % c->cap].payload ^= (uint32_t)value; return ORC_OK;
    case 7: if (!c) return ORC_EINVAL; c->next = (uint32_t)value; return ORC_OK;
    case 8: {
        int ncnt = (int)((sizeof(orc_counters) - sizeof(int64_t)) / sizeof(int64_t));
        if ((int)i >= ncnt) return ORC_EINVAL;
        (&s->c.generated)[i] += (int64_t)value; return ORC_OK;
    }
    case 9: {
        uint64_t *hs[3] = { s->hl, s->hd, s->ha };
        if (i >= 3 || j >= s->cfg.hist_bins) return ORC_EINVAL;
        hs[i][j] += value; return ORC_OK;
    }
    case 10: s->t += value; s->c.cycle = (int64_t)s->t; return ORC_OK;
    case 11:
        if (!c || !s->cfg.l1_sets || i >= s->cfg.l1_sets || j >= s->cfg.l1_ways) return ORC_EINVAL;
        c->l1[(uint64_t)i * s->cfg.l1_ways + j].owner ^= (uint32_t)value; return ORC_OK;
    case 12: if (!c) return ORC_EINVAL; c->rx += (uint32_t)value; return ORC_OK;
    case 13: if (!c) return ORC_EINVAL; c->ready += value; return ORC_OK;
    }
    return ORC_EINVAL;
}

/* NEXT-f2 test hook: the migration decision of R46 on a given accessor history
 * (oldest first) for holder h: the target node, or UINT32_MAX for none. */
uint32_t orc_mig_target(const uint32_t *hist, uint32_t count, uint32_t holder)
{
    Line L;
    memset(&L, 0, sizeof L);
    orc_sim tmp;
    memset(&tmp, 0, sizeof tmp);
    tmp.cfg.mig_hist = count ? count : 1;
    for (uint32_t i = 0; i < count && i < MIG_HIST_MAX; ++i) L.hist[i] = hist[i];
    L.hcount = count < MIG_HIST_MAX ? count : MIG_HIST_MAX;
    return mig_target(&tmp, &L, holder);
}

/* NEXT-f2 peek: L2 line (n, set, way) migration state: mstate, mtarget, hcount;
 * loc entry T: transit, early_ev. */
int orc_l2_mig(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way, uint64_t out[3])
{
    if (s->cfg.mode != ORC_MODE_LSPD || n >= s->N || set >= s->cfg.l2_sets || way >= s->cfg.l2_ways)
        return ORC_EINVAL;
    const Line *L = &s->nodes[n].l2[(uint64_t)set * s->cfg.l2_ways + way];
    out[0] = (uint64_t)L->mstate; out[1] = L->mtarget; out[2] = L->hcount;
    return ORC_OK;
}

int orc_loc_mig(const orc_sim *s, uint32_t T, uint64_t out[2])
{
    if (T >= s->ntags) return ORC_EINVAL;
    out[0] = (uint64_t)s->loc[T].transit; out[1] = (uint64_t)s->loc[T].early_ev;
    return ORC_OK;
}

/* NEXT-f2 peeks: the accessor history of L2 line (n, set, way), oldest first
 * (returns the count); inbound-migration slot k of node n: used, tag, count */
int orc_l2_hist(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way, uint32_t out[16])
{
    if (s->cfg.mode != ORC_MODE_LSPD || n >= s->N || set >= s->cfg.l2_sets || way >= s->cfg.l2_ways)
        return -1;
    const Line *L = &s->nodes[n].l2[(uint64_t)set * s->cfg.l2_ways + way];
    for (uint32_t i = 0; i < L->hcount; ++i) out[i] = L->hist[(L->hhead + i) % (s->cfg.mig_hist ? s->cfg.mig_hist : 1)];
    return (int)L->hcount;
}

int orc_migrx(const orc_sim *s, uint32_t n, uint32_t k, uint64_t out[3])
{
    if (n >= s->N || k >= 4) return ORC_EINVAL;
    out[0] = (uint64_t)s->nodes[n].migrx[k].used; out[1] = s->nodes[n].migrx[k].tag; out[2] = s->nodes[n].migrx[k].count;
    return ORC_OK;
}
