/*
 * noc_sim.h -- C-ABI of the B200-native simulator of the per-cycle, per-node
 * step of a bufferless, deflection-routed 2D-mesh NoC coupled to an LSPD L2
 * (Kumar & Sahu, arXiv 1508.03235; "P:Lnn" = PAPER.md line nn).
 *
 * Library: paper_1508_03235_b200/libnocsim.so (CUDA, sm_100a).  Every
 * simulated cycle runs in the library's CUDA kernels; there is no CPU path.
 * The model (state, the three phases, counters, the state hash) is DESIGN.md
 * section 3; the calls follow the north_star problem statement
 * ("noc_sim_create(mesh WxH, cache geometry, traffic/trace params, seed),
 * noc_sim_run(n_cycles) and noc_sim_stats()") and the paper's serial loop
 * (initialize, per-cycle phases until MAXSIMCYCLE, statistics).
 *
 * Conventions
 *   - return 0 (NOC_OK) or a negative NOC_E* code; on error
 *     noc_sim_last_error() returns a thread-local message.
 *   - a handle is used by one host thread at a time; one handle per process
 *     and GPU (per rank when world_size > 1).
 *   - all pointers are HOST pointers owned by the caller unless stated.
 *     The library owns all device memory it allocates, until destroy.
 *   - node id n = y*mesh_w + x, x = column, y = row ("(2,4) = row 2,
 *     column 4"); ports N=0, S=1, E=2, W=3.
 */
#ifndef NOC_SIM_H
#define NOC_SIM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NOC_SIM_ABI_VERSION 6u   /* 2: route, dir_mode/dir_node, l1_*, inject_mode; L1 counters; 3: age_base; 4: band_streams; 5: migration; 6: memory nodes, hub FIFOs, fill-all injection */

/* error codes */
#define NOC_OK          0
#define NOC_EINVAL     -1   /* invalid config / argument                        */
#define NOC_ENOMEM     -2   /* device or host allocation failed                 */
#define NOC_ECUDA      -3   /* CUDA runtime error (no device, launch failure)   */
#define NOC_ENCCL      -4   /* NCCL error (world_size > 1)                      */
#define NOC_EOVERFLOW  -5   /* a field width was exceeded (DESIGN R32): flit
                               age > 65535 or directory pend > 1023.  The
                               handle is poisoned: later run/drain calls fail */
#define NOC_ESTATE     -6   /* call not valid in the handle's state             */

/* traffic mode (DESIGN R35) */
#define NOC_MODE_UR    0u   /* uniform-random 1-flit probes, open loop          */
#define NOC_MODE_LSPD  1u   /* core accesses to the LSPD L2 (Fig. 4)    */
/* router priority (DESIGN R1) */
#define NOC_PRIO_DEFLECT 0u /* age = deflection count      */
#define NOC_PRIO_OLDEST  1u /* oldest injection cycle first            */

/* directory organisation (DESIGN R12, R40) */
#define NOC_DIR_DISTRIBUTED 0u /* home(T) = T mod N (R12)                          */
#define NOC_DIR_CENTRAL     1u /* home(T) = dir_node for every T: the paper's
                                  centralized location array     */

/* memory placement (DESIGN R54-R55) */
#define NOC_MEM_OFFMESH 0u  /* off-mesh memory at the requester, fixed mem_lat (R17) */
#define NOC_MEM_HOME    1u  /* memory at the block's home node: the directory node
                               under NOC_DIR_CENTRAL; a negative
                               directory reply becomes a B2 fill from there (P:L69,
                               L89, Table I B2 = nfl_b2 flits)                 */
#define NOC_MEM_CTRLS   2u  /* mem_ctrls memory-controller nodes, ceil(M/2) evenly
                               spaced on the top row and the rest on the bottom
                               row; block T's memory = controller T mod M: a
                               1-flit request, a B2 fill back, B2 writebacks of
                               every L2 victim                                 */

/* routing (DESIGN R3, R5; SURVEY 8(f) NEXT-f4 compatibility mode) */
#define NOC_ROUTE_PMDR   0u /* productive ports x then y; deflect to the first free
                               existing port in N,S,E,W         */
#define NOC_ROUTE_XY     1u /* strict XY: the x-port while dx != 0, then the
                               y-port; deflect in N,E,S,W order (SPEC S:L136,
                               S:L162)                                         */
/* engine: which kernel organisation advances the cycles.  Results are
 * bit-identical for every engine. */
#define NOC_ENGINE_AUTO     0u  /* library picks: TILED if every tile fits (<= 320
                                   nodes per SM and band), else TILED4, else
                                   PERSIST                                      */
#define NOC_ENGINE_STEP     1u  /* one fused node-step launch per cycle (no bands) */
#define NOC_ENGINE_PERSIST  2u  /* persistent kernel, neighbour-progress sync; any
                                   mesh size, row bands                         */
#define NOC_ENGINE_TILED    3u  /* persistent kernel, tiles in shared memory      */
#define NOC_ENGINE_TILED4   4u  /* as TILED, 4 lanes (one per router port) per node;
                                   not with inject_mode 1                       */

/* A scripted generation event (golden tests; trace replay).
 * At each generation opportunity of node `node` at cycle t (every cycle in UR
 * mode; when the core is IDLE in LSPD mode) the first not-yet-consumed event of
 * that node with cycle <= t is consumed instead of the Philox draw.
 * value: UR = probe destination node (!= node); LSPD = block tag T. */
typedef struct noc_sim_event {
    uint64_t cycle;
    uint32_t node;
    uint32_t value;
} noc_sim_event;

typedef struct noc_sim_config {
    uint32_t mesh_w, mesh_h;   /* 2..2048 each, mesh_w*mesh_h <= 2^21-1 (R9, R32) */
    uint32_t mode;             /* NOC_MODE_*                                      */
    uint32_t prio;             /* NOC_PRIO_*                                      */
    uint32_t l2_sets, l2_ways; /* LSPD slice geometry (Table III):
                                  sets 1..65536, ways 1..16                       */
    uint32_t l2_line_bytes;    /* informational only (no data is simulated)      */
    uint32_t tags_per_node;    /* TPN: tag space = TPN*N <= 2^31                  */
    uint32_t priv_tags;        /* PRIV: private window, 1 <= PRIV < TPN           */
    uint32_t thr_inj;          /* floor(lambda * 2^32) (R25, R35)                 */
    uint32_t thr_priv;         /* floor(p_priv * 2^32)                            */
    uint32_t l2_hit_lat;       /* local L2 hit latency, cycles, < 2^29            */
    uint32_t mem_lat;          /* memory latency, 1 .. 2^29-1 (R17)               */
    uint32_t nfl_ra;           /* flits of the RA data reply, 1..8 (Table I: 4)   */
    uint32_t sendq_cap;        /* send-FIFO packets per node, power of 2, <= 1024 */
    uint32_t hist_bins;        /* NB, 1..65536; last bin = overflow (R31)         */
    uint64_t seed;             /* Philox key (R25)                                */
    const noc_sim_event *script; /* optional host array, copied at create       */
    uint64_t n_script;
    int32_t  device;           /* CUDA device ordinal                             */
    int32_t  world_size;       /* row bands across processes (1 = single GPU)     */
    int32_t  rank;             /* this process's band, 0..world_size-1            */
    uint32_t engine;           /* NOC_ENGINE_*                                     */
    uint8_t  nccl_id[128];     /* ncclUniqueId from rank 0 (world_size > 1)       */
    uint32_t bands;            /* world_size == 1 only: simulate the mesh as this
                                  many row bands on one GPU ("virtual bands", the
                                  multi-GPU partition on one device); 0/1 = none.
                                  Results are identical for every value.         */
    uint32_t route;            /* NOC_ROUTE_* (0 = the paper's reading)           */
    uint32_t dir_mode;         /* NOC_DIR_* (LSPD): where the location array lives */
    uint32_t dir_node;         /* NOC_DIR_CENTRAL: the node holding the whole
                                  directory (0..N-1); ignored otherwise          */
    uint32_t l1_sets;          /* LSPD, NEXT-f1 private write-through L1 (R42):
                                  0 = none (the base model), else 1..65536      */
    uint32_t l1_ways;          /* 1..16 (Table III: 32 sets x 2 ways)            */
    uint32_t l1_miss_lat;      /* "L1 miss cycle" countdown, 1 .. 2^29-1 */
    uint32_t inject_mode;      /* 0: R7 (inject only into a free input port);
                                  1: NEXT-f4, a flit that will eject frees its
                                  input port for the same cycle;
                                  2: NEXT-f4 fill-all, queued flits fill every
                                  free input port, oldest-queued first (SPEC
                                  S:L145; DESIGN R53).
                                  1 and 2 are not supported by NOC_ENGINE_TILED4 */
    uint32_t age_base;         /* test knob: injected flits start at this age
                                  instead of 0; 0 = the paper's model,
                                  <= 65535.  Shifts every age equally (ranking
                                  unchanged) so tests reach ages >= 2048 and the
                                  R32 age limit (NOC_EOVERFLOW)                  */
    uint32_t band_streams;     /* bands > 1 with the TILED engine: 1 = "virtual
                                  ranks": every band is advanced by its own
                                  launches on its own stream, with the
                                  multi-process sequence per launch (slot
                                  refresh, a cross-band barrier, the band's
                                  cooperative launch, a barrier) and events
                                  in place of the NCCL barrier; 0 = all bands
                                  in one launch.  Results are identical     */
    uint32_t mig_hist;         /* LSPD, NEXT-f2 migration + redirection (DESIGN
                                  R44-R52): length N of each L2 line's accessor
                                  history ("last N (say 10) accesses"),
                                  1..16; 0 = no migration (the base model).
                                  Needs tags_per_node*N <= 2^28              */
    uint32_t nfl_b2;           /* flits of a B2 block (Table I: 16), 1..16: a
                                  block migration (mig_hist > 0) and the memory
                                  fills / writebacks of mem_mode 1 and 2      */
    uint32_t mem_mode;         /* LSPD, where memory is (DESIGN R54-R55):
                                  NOC_MEM_OFFMESH, NOC_MEM_HOME, NOC_MEM_CTRLS.
                                  1 and 2 exclude migration (mig_hist = 0)    */
    uint32_t mem_ctrls;        /* NOC_MEM_CTRLS: number of controllers M,
                                  1..64, ceil(M/2) <= mesh_w (ignored otherwise) */
    uint32_t hub_sendq_cap;    /* send-FIFO packets at hub nodes -- the central
                                  directory node (NOC_DIR_CENTRAL) and the
                                  memory controllers (NOC_MEM_CTRLS); 0 =
                                  sendq_cap, else a power of two in
                                  sendq_cap..1024 (DESIGN R56)     */
} noc_sim_config;

/* Counters (DESIGN 3.6; Table II columns P:L303-304 and the statistics list
 * of P:L223).  Totals over all ranks. */
typedef struct noc_sim_counters {
    int64_t cycle;
    int64_t generated, packets_enqueued, injected, ejected, hops, deflections;
    int64_t probes_delivered, accesses, completed, l2_hits, l2_misses;
    int64_t dir_searches, requests_made, requests_received, replies_sent;
    int64_t replies_received, traps_sent, traps_received, mem_requests;
    int64_t installs, evictions, evs_sent, evs_received;
    int64_t drops[8];          /* by kind: PROBE DA DR NDR RQ RA TRAP EV           */
    int64_t l1_hits, l1_misses, wb_sent, wb_received;   /* NEXT-f1 L1 (R42)       */
    /* NEXT-f2 migration + redirection (R44-R52): requests to the directory,
     * refusals, blocks sent, blocks installed at the target, directory
     * updates, source invalidations, redirections sent / received */
    int64_t mig_requests, mig_nacks, migrations, mig_installs;
    int64_t dir_updates, invalidations, redirections, rr_received;
    /* memory nodes (R55): B2 fills sent by memory nodes / completed at the
     * requesters, B2 writebacks sent, writeback flits absorbed at memory nodes */
    int64_t mem_fills_sent, mem_fills_received, mem_wbs_sent, mem_wb_flits;
} noc_sim_counters;

/* Runtime facts about a handle (for measurement and the bench). */
typedef struct noc_sim_info {
    uint32_t engine;           /* engine actually used                             */
    uint32_t grid, block;      /* launch shape of the node-step kernel             */
    uint32_t nodes_local;      /* nodes owned by this rank                         */
    uint32_t row0, rows;       /* this rank's band                                 */
    uint64_t device_bytes;     /* device memory held                               */
    uint64_t loc_bytes;        /* of which: location array (4 B per tag, R36)      */
    uint64_t kernel_launches;  /* node-step launches issued so far                 */
    uint64_t cycles_run;       /* cycles advanced so far                           */
    int32_t  sm_count;
    uint32_t cluster;          /* TILED: > 0 = the band runs as one thread-block
                                  cluster of this many tiles (DSMEM links, no
                                  LL slots, no refresh launches)              */
    int32_t  reserved[6];
} noc_sim_info;

typedef struct noc_sim noc_sim;

/* ABI version of the loaded library (== NOC_SIM_ABI_VERSION). */
uint32_t noc_sim_abi_version(void);

/* Row bands (DESIGN 8).  Band g of P covers rows [g*H/P, (g+1)*H/P); it owns
 * those nodes' links, cores, FIFOs, L2 slices and the directory entries of the
 * tags homed on them (T mod N in the band).  With world_size = P processes
 * (one GPU each, torchrun), band = rank; the links crossing a band edge are
 * written by the sending GPU directly into the receiving GPU's boundary slots
 * (TILED) or link arrays (PERSIST, which also reads the neighbour's progress
 * counters) through CUDA IPC over NVLink; NCCL is used for setup and the
 * statistics / hash / drain reductions.  With the centralized directory the
 * whole location array lives in the directory node's band.  Fills out[128] with a fresh ncclUniqueId (rank 0 calls
 * this and broadcasts it).  Errors: NOC_ENCCL. */
int noc_sim_nccl_unique_id(uint8_t out[128]);

/* The rows [*row0, *row0 + *rows) of band `rank` of `world_size` on a mesh of
 * mesh_h rows: row0 = floor(rank * mesh_h / world_size) (the partition every
 * handle uses; host only, no device needed).  Errors: NOC_EINVAL. */
int noc_sim_band_rows(uint32_t mesh_h, int32_t world_size, int32_t rank, uint32_t *row0, uint32_t *rows);

/* Create a simulation at cycle 0 ("initialize" kernel): all links and
 * FIFOs empty, cores IDLE, L2 lines invalid, directory empty, counters 0.
 * cfg is copied (including the script).  When world_size > 1 this call is
 * collective over the ranks (NCCL communicator setup).
 * Errors: NOC_EINVAL (with the violated limit in the message), NOC_ENOMEM,
 * NOC_ECUDA, NOC_ENCCL.  On error *out = NULL. */
int noc_sim_create(const noc_sim_config *cfg, noc_sim **out);

/* NEXT-f3 streamed trace replay (DESIGN R57; SURVEY f3 "streamed with
 * double-buffered chunked H2D copies instead of the paper's per-cycle
 * cudaMemcpy"): append scripted generation events (the same
 * records as noc_sim_config.script) to the nodes' queues, so traces larger
 * than device memory are replayed chunk by chunk.  ev: host array of n events,
 * copied before the call returns (pinned staging; the host-to-device copy runs
 * asynchronously and overlaps the next noc_sim_run when none of the chunk's
 * events is due in it).  Per node the pushed events are ordered by cycle
 * (stable, as at create) and must not precede the node's earlier events.
 * Consumed events are dropped from device memory at the next merge.  Results
 * equal those of the whole script given at create as long as every event is
 * pushed before it is due.  With world_size > 1 every rank pushes the same
 * events (each keeps its band's).  Errors: NOC_EINVAL (range or order),
 * NOC_ECUDA, NOC_ESTATE (poisoned handle). */
int noc_sim_push_script(noc_sim *sim, const noc_sim_event *ev, uint64_t n);

/* Advance exactly n_cycles cycles (the while loop of P:L275-284 without its
 * per-cycle trace copy).  Resumable: run(a); run(b) == run(a+b).  Blocks until
 * the device finished.  Collective when world_size > 1.
 * Errors: NOC_ECUDA, NOC_ENCCL, NOC_EOVERFLOW. */
int noc_sim_run(noc_sim *sim, uint64_t n_cycles);

/* Like noc_sim_run and also returns the device time of the run in ms,
 * measured with CUDA events recorded on the library's stream around the
 * launches (this rank only). */
int noc_sim_run_timed(noc_sim *sim, uint64_t n_cycles, double *device_ms);

/* Stop generation and run until quiescent (no flit on a link, every FIFO
 * empty, every core IDLE) or max_cycles ("until ... no any outstanding
 * flit"; R30).  *used = cycles advanced, *drained = 1 if quiescent.  A cap is
 * reported, not an error.  Generation is re-enabled afterwards. */
int noc_sim_drain(noc_sim *sim, uint64_t max_cycles, uint64_t *used, int *drained);

/* Copy the counters (into *out, may be NULL) and the three histograms
 * (flit latency, deflections at eject, access latency; each nbins uint64
 * host words, may be NULL) -- "GetSimulationStatics".
 * Errors: NOC_EINVAL if nbins != hist_bins and a histogram pointer is given. */
int noc_sim_stats(noc_sim *sim, noc_sim_counters *out, uint64_t *hist_lat,
                  uint64_t *hist_defl, uint64_t *hist_acc, uint32_t nbins);

/* Canonical, layout-independent state hash (DESIGN 3.7): a pure function of
 * the model state; equal across engines and world sizes. */
int noc_sim_state_hash(noc_sim *sim, uint64_t *out);

/* Facts about the handle. */
int noc_sim_get_info(noc_sim *sim, noc_sim_info *out);

/* Free everything.  NULL-safe. */
void noc_sim_destroy(noc_sim *sim);

/* Thread-local message of the last error. */
const char *noc_sim_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
