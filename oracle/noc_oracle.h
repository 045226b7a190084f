/*
 * noc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Interface of the plain, slow, single-threaded CPU oracle of the
 * bufferless-NoC + LSPD-L2 cycle simulation of Kumar & Sahu,
 * arXiv 1508.03235 ("Bufferless NOC Simulation of Large Multicore System on
 * GPU Hardware").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the CUDA product library
 * (paper_1508_03235_b200/csrc, include/noc_sim.h).
 *
 * Citations: "P:Lnn" = PAPER.md line nn; readings R1..R35 are listed in
 * DESIGN.md section 3 (they follow SURVEY.md section 8(c.3)).
 */
#ifndef NOC_ORACLE_H
#define NOC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK         0
#define ORC_EINVAL    -1
#define ORC_ENOMEM    -2
#define ORC_EOVERFLOW -5
#define ORC_EASSERT   -7   /* a debug invariant failed (see orc_last_error) */

/* traffic modes (R35) */
#define ORC_MODE_UR   0    /* uniform-random 1-flit probes, open loop       */
#define ORC_MODE_LSPD 1    /* core accesses to the LSPD L2 (Fig. 4)  */
/* priority (R1) */
#define ORC_PRIO_DEFLECT 0 /* age = #deflections       */
#define ORC_PRIO_OLDEST  1 /* oldest injection cycle first         */
/* routing (R3, R5; NEXT-f4 compatibility mode) */
#define ORC_ROUTE_PMDR   0 /* productive ports x then y, deflect in N,S,E,W */
#define ORC_ROUTE_XY     1 /* SPEC: strict XY preference, deflect in N,E,S,W  */

/* debug flags for orc_set_debug */
#define ORC_DBG_REVERSE    1  /* iterate nodes in reverse order in every phase */
#define ORC_DBG_INVARIANTS 2  /* check conservation / exclusivity / directory
                                 single-copy / top-priority progress per cycle */

typedef struct {
    uint64_t cycle;   /* earliest cycle the event may be consumed          */
    uint32_t node;    /* node id y*W+x                                     */
    uint32_t value;   /* UR: probe destination node; LSPD: block tag T     */
} orc_event;

typedef struct {
    uint32_t mesh_w, mesh_h;     /* 2..2048 each, W*H <= 2^21               */
    uint32_t mode, prio;
    uint32_t l2_sets, l2_ways;   /* LSPD slice geometry (Table III)         */
    uint32_t tags_per_node;      /* TPN: tag space = TPN * N                */
    uint32_t priv_tags;          /* PRIV: private window per node, < TPN    */
    uint32_t thr_inj;            /* floor(lambda * 2^32)                    */
    uint32_t thr_priv;           /* floor(p_priv * 2^32)                    */
    uint32_t l2_hit_lat;         /* >= 0                                    */
    uint32_t mem_lat;            /* >= 1                                    */
    uint32_t nfl_ra;             /* flits of the RA data reply, Table I: 4  */
    uint32_t sendq_cap;          /* packets per send FIFO, power of two     */
    uint32_t hist_bins;          /* NB, last bin = overflow                 */
    uint64_t seed;
    const orc_event *script;     /* optional, may be NULL                   */
    uint64_t n_script;
    uint32_t route;              /* ORC_ROUTE_*                             */
    uint32_t dir_mode;           /* 0: home(T) = T mod N (R12); 1: central  */
    uint32_t dir_node;           /* dir_mode 1: the node holding the directory */
    uint32_t l1_sets, l1_ways;   /* NEXT-f1 private L1 (Table III); 0 sets = none */
    uint32_t l1_miss_lat;        /* "L1 miss cycle" countdown, >= 1 */
    uint32_t inject_mode;        /* 0: R7; 1: an ejecting flit frees its slot (NEXT-f4);
                                    2: queued flits fill every free input slot (NEXT-f4, R53) */
    uint32_t age_base;           /* test knob: age of a newly injected flit (0 = P:L259) */
    uint32_t mig_hist;           /* NEXT-f2: accessor history length N; 0 = no migration */
    uint32_t nfl_b2;             /* flits of a B2 block (Table I: 16), 1..16: migration (NEXT-f2)
                                    and memory fills / writebacks (mem_mode >= 1) */
    uint32_t mem_mode;           /* memory placement (R54): 0 off-mesh at the requester (R17);
                                    1 at the home node of the block (the directory node under
                                    the central directory); 2 mem_ctrls
                                    memory-controller nodes on the top / bottom rows (NEXT-f4) */
    uint32_t mem_ctrls;          /* mem_mode 2: number of controllers M, 1..64, ceil(M/2) <= W */
    uint32_t hub_sendq_cap;      /* send-FIFO packets at hub nodes (the central directory node,
                                    the memory controllers; R56): 0 = sendq_cap, else a power
                                    of two in sendq_cap..1024 */
} orc_config;

/* counters, in the order of DESIGN.md section 3.6 */
typedef struct {
    int64_t cycle;
    int64_t generated, packets_enqueued, injected, ejected, hops, deflections;
    int64_t probes_delivered, accesses, completed, l2_hits, l2_misses;
    int64_t dir_searches, requests_made, requests_received, replies_sent;
    int64_t replies_received, traps_sent, traps_received, mem_requests;
    int64_t installs, evictions, evs_sent, evs_received;
    int64_t drops[8];
    int64_t l1_hits, l1_misses, wb_sent, wb_received;   /* NEXT-f1 (R42) */
    int64_t mig_requests, mig_nacks, migrations, mig_installs;   /* NEXT-f2 (R44-R52) */
    int64_t dir_updates, invalidations, redirections, rr_received;
    /* memory nodes (mem_mode >= 1, R54-R55): B2 fills sent by memory nodes
     * and completed at requesters, B2 writebacks sent, writeback flits
     * absorbed by memory nodes */
    int64_t mem_fills_sent, mem_fills_received, mem_wbs_sent, mem_wb_flits;
} orc_counters;

typedef struct orc_sim orc_sim;

int  orc_create(const orc_config *cfg, orc_sim **out);
void orc_destroy(orc_sim *s);
int  orc_set_debug(orc_sim *s, int flags);
int  orc_run(orc_sim *s, uint64_t n_cycles);
int  orc_drain(orc_sim *s, uint64_t max_cycles, uint64_t *used, int *drained);
/* NEXT-f3 streamed trace replay (R57): append script events (copied); per node
 * ordered by cycle, not earlier than the node's previous events (ORC_EINVAL). */
int  orc_push_script(orc_sim *s, const orc_event *ev, uint64_t n);
int  orc_stats(const orc_sim *s, orc_counters *out, uint64_t *hist_lat,
               uint64_t *hist_defl, uint64_t *hist_acc, uint32_t nbins);
uint64_t orc_state_hash(const orc_sim *s);
const char *orc_last_error(void);

/* ---- test hooks ------------------------------------------------------ */
/* Philox4x32-10 with key {k0,k1} on counter c[4] -> out[4]. */
void orc_philox(uint32_t k0, uint32_t k1, const uint32_t c[4], uint32_t out[4]);

/* One router's stage-2 decision in isolation.
 *   flits: nf records of 4 u64 {dst, src, age, inj}
 *   out_port[i]: 0..3 = N,S,E,W output, 4 = eject
 *   out_age[i] : age after the decision
 * Returns 0, or -1 if nf > degree. */
int orc_arbitrate(uint32_t mesh_w, uint32_t mesh_h, uint32_t node, uint32_t prio, uint32_t route,
                  uint32_t nf, const uint64_t *flits, int *out_port,
                  uint64_t *out_age);
/* The same with stride 4 or 7 u64 per flit {dst, src, age, inj[, fid, kind,
 * payload]}: the last three break ties of equal (age, inj, src) -- flits one
 * node injected in the same cycle under the fill-all mode (R53). */
int orc_arbitrate_ex(uint32_t mesh_w, uint32_t mesh_h, uint32_t node, uint32_t prio, uint32_t route,
                     uint32_t nf, uint32_t stride, const uint64_t *flits, int *out_port, uint64_t *out_age);

/* In-flight flits on links (inputs of the next cycle) and their age sum. */
int64_t orc_links_occupied(const orc_sim *s, int64_t *age_sum);
/* Packets waiting in send FIFOs (all nodes). */
int64_t orc_fifo_packets(const orc_sim *s);
/* Number of cores not IDLE. */
int64_t orc_cores_busy(const orc_sim *s);
/* Directory agreement at quiescence (DESIGN 3.5): 0 if it holds. */
int  orc_check_directory_quiescent(const orc_sim *s);
/* Core record of node n: mode, ready, tag, install, start, rx. */
int  orc_core(const orc_sim *s, uint32_t n, uint64_t out[6]);
/* L2 slice line (n, set, way): valid, tag, stamp. */
int  orc_l2_line(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way,
                 uint64_t out[3]);
/* Directory entry of tag T: holder (UINT32_MAX = none) and pend. */
int  orc_loc(const orc_sim *s, uint32_t T, uint64_t out[2]);

/* Link input slot d of node n: present, dst, src, kind, fid, payload, age, inj. */
int  orc_link(const orc_sim *s, uint32_t n, uint32_t d, uint64_t out[8]);
/* Send FIFO of n: out = {count, next}; pkt = packet k from the head {kind, dst, payload, nfl}. */
int  orc_fifo(const orc_sim *s, uint32_t n, uint32_t k, uint64_t out[2], uint64_t pkt[4]);
/* NEXT-f1 L1 line: valid, tag, stamp, owner. */
int  orc_l1_line(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way, uint64_t out[4]);
/* Script events consumed by node n (-1 if n is out of range). */
int64_t orc_script_used(const orc_sim *s, uint32_t n);
/* The simulation's generator call for (n, t): out = {fired, UR dst or LSPD tag}. */
int  orc_gen(const orc_sim *s, uint32_t n, uint64_t t, uint64_t out[2]);
/* NEXT-f2: the migration decision (R46) on an accessor history, oldest first:
 * the target node, or UINT32_MAX for none (SPEC S:L235-243 examples). */
uint32_t orc_mig_target(const uint32_t *hist, uint32_t count, uint32_t holder);
/* NEXT-f2 peeks: L2 line migration state {mstate, mtarget, hcount}; loc {transit, early_ev}. */
int  orc_l2_mig(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way, uint64_t out[3]);
int  orc_loc_mig(const orc_sim *s, uint32_t T, uint64_t out[2]);
int  orc_l2_hist(const orc_sim *s, uint32_t n, uint32_t set, uint32_t way, uint32_t out[16]);
int  orc_migrx(const orc_sim *s, uint32_t n, uint32_t k, uint64_t out[3]);
/* Test-only single-field mutation (hash sensitivity pins); fields in noc_oracle.c. */
int  orc_poke(orc_sim *s, uint32_t field, uint32_t n, uint32_t i, uint32_t j, uint64_t value);

#ifdef __cplusplus
}
#endif
#endif
