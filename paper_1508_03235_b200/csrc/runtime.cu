// runtime.cu -- host runtime behind include/noc_sim.h: configuration
// validation, structure-of-arrays allocation in HBM (per row band), engine
// selection and launch control, drain, statistics and the canonical state
// hash, and the multi-GPU row-band plumbing (CUDA IPC + NCCL).
#include "../../include/noc_sim.h"
#include "kernels.h"

#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace noc;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

extern "C" const char *noc_sim_last_error(void) { return g_err.c_str(); }
extern "C" uint32_t noc_sim_abi_version(void) { return NOC_SIM_ABI_VERSION; }

#define CU(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(NOC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));           \
    } while (0)

#define NC(call)                                                                                  \
    do {                                                                                          \
        ncclResult_t r_ = (call);                                                                 \
        if (r_ != ncclSuccess)                                                                    \
            return fail(NOC_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));           \
    } while (0)

extern "C" int noc_sim_nccl_unique_id(uint8_t out[128])
{
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    memcpy(out, &id, 128);
    return NOC_OK;
}

struct noc_sim {
    noc_sim_config cfg;
    int nb = 1;                 // bands simulated by this process
    int P = 1;                  // bands in the whole mesh
    int g0 = 0;                 // global index of the first local band
    Dev D[MAX_BANDS];
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    uint64_t t = 0;             // next cycle to simulate
    uint32_t engine = NOC_ENGINE_STEP;
    // persistent engine
    uint32_t *progress = nullptr;
    uint32_t pbase = 0;
    uint32_t p_grid = 0, p_npc = 0, p_smem_hist = 0;
    // tiled engine
    DevSet set;
    uint32_t t_tpad = 0, t_smem_hist = 0;
    // shared by the bands of this process
    unsigned long long *cnt = nullptr, *hist = nullptr;
    uint32_t *err = nullptr;
    uint32_t *d_scratch = nullptr;          // [DRAIN_CHUNK + 2]
    unsigned long long *d_hash = nullptr;
    unsigned long long *d_red = nullptr;    // reduction buffer (NCCL)
    // multi-GPU
    int world = 1, rank = 0;
    ncclComm_t comm = nullptr;
    std::vector<void *> ipc_opened;
    // virtual ranks (band_streams): one stream, launch set and events per band
    int split = 0;
    cudaStream_t bst[MAX_BANDS] = {};
    cudaEvent_t bev[MAX_BANDS] = {};
    cudaEvent_t mev = nullptr;
    DevSet bset[MAX_BANDS];
    std::vector<void *> allocs;
    std::vector<size_t> alloc_bytes;
    uint64_t bytes = 0, loc_bytes = 0;
    // streamed scripts (NEXT-f3, R57): per node the cycle of its last event so
    // far; pushed chunks waiting to be merged (per band: device staging filled
    // by an asynchronous copy on cstream from pinned host memory)
    std::vector<uint64_t> script_last;
    std::vector<uint8_t> script_any;
    struct Pending {
        uint64_t min_cycle;
        uint32_t n[MAX_BANDS];
        uint4 *ev[MAX_BANDS];
        uint32_t *off[MAX_BANDS];
        void *host;
        cudaEvent_t done;
    };
    std::vector<Pending> pending;
    cudaStream_t cstream = nullptr;
    uint64_t launches = 0;
    int sm_count = 0;
    int poisoned = 0;
};

static const uint32_t DRAIN_CHUNK = 512;
static const uint32_t PERSIST_CHUNK = 1u << 20;

template <typename T>
static int dalloc(noc_sim *s, T **p, size_t count)
{
    size_t b = std::max<size_t>(count * sizeof(T), 16);
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, b);
    if (e != cudaSuccess) return fail(NOC_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    // the zeroing runs on the legacy default stream, which the library's
    // non-blocking streams are not ordered against: it must be complete
    // before the buffer is filled by a copy or kernel on those streams (a
    // late memset zeroed a merged script's offsets, losing a pushed piece).
    // Waits for this memset only; running kernels on the library's streams
    // are not waited for.
    e = cudaMemset(q, 0, b);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("cudaMemset: ") + cudaGetErrorString(e));
    s->allocs.push_back(q);
    s->alloc_bytes.push_back(b);
    s->bytes += b;
    *p = (T *)q;
    return NOC_OK;
}

// free one dalloc'ed buffer (streamed-script arrays that are replaced)
static void dfree(noc_sim *s, void *p)
{
    for (size_t i = 0; i < s->allocs.size(); ++i)
        if (s->allocs[i] == p) {
            cudaFree(p);
            s->bytes -= s->alloc_bytes[i];
            s->allocs.erase(s->allocs.begin() + (long)i);
            s->alloc_bytes.erase(s->alloc_bytes.begin() + (long)i);
            return;
        }
}

static int validate(const noc_sim_config *c)
{
    if (!c) return fail(NOC_EINVAL, "null config");
    const uint64_t N = (uint64_t)c->mesh_w * c->mesh_h;
    if (c->mesh_w < 2 || c->mesh_h < 2 || c->mesh_w > 2048 || c->mesh_h > 2048 || N > (1u << 21) - 1u)
        return fail(NOC_EINVAL, "mesh must be 2..2048 per side and at most 2^21-1 nodes (R9, R32)");
    if (c->mode > 1 || c->prio > 1 || c->route > 1) return fail(NOC_EINVAL, "mode/prio/route out of range");
    if (c->dir_mode > 1 || (c->dir_mode && c->dir_node >= N)) return fail(NOC_EINVAL, "dir_mode/dir_node out of range");
    if (c->sendq_cap == 0 || c->sendq_cap > 1024 || (c->sendq_cap & (c->sendq_cap - 1)))
        return fail(NOC_EINVAL, "sendq_cap must be a power of two in 1..1024");
    if (c->hist_bins == 0 || c->hist_bins > 65536) return fail(NOC_EINVAL, "hist_bins must be 1..65536");
    if (c->nfl_ra < 1 || c->nfl_ra > 8) return fail(NOC_EINVAL, "nfl_ra must be 1..8");
    if (c->mode == NOC_MODE_LSPD) {
        if (c->l2_sets < 1 || c->l2_sets > 65536 || c->l2_ways < 1 || c->l2_ways > 16)
            return fail(NOC_EINVAL, "l2 geometry: sets 1..65536, ways 1..16");
        if (c->tags_per_node < 2 || c->priv_tags < 1 || c->priv_tags >= c->tags_per_node)
            return fail(NOC_EINVAL, "need 1 <= priv_tags < tags_per_node");
        if ((uint64_t)c->tags_per_node * N > (1ull << 31)) return fail(NOC_EINVAL, "tag space TPN*N exceeds 2^31");
        if (c->mem_lat < 1 || c->mem_lat >= (1u << 29) || c->l2_hit_lat >= (1u << 29))
            return fail(NOC_EINVAL, "latencies must be < 2^29 (mem_lat >= 1)");
    }
    if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size)
        return fail(NOC_EINVAL, "bad world_size/rank");
    if (c->world_size > (int)MAX_BANDS || c->world_size > (int)c->mesh_h)
        return fail(NOC_EINVAL, "world_size must be <= 8 and <= mesh_h");
    if (c->bands > MAX_BANDS || c->bands > c->mesh_h) return fail(NOC_EINVAL, "bands must be <= 8 and <= mesh_h");
    if (c->bands > 1 && c->world_size > 1) return fail(NOC_EINVAL, "bands > 1 is for world_size == 1 only");
    if (c->engine > NOC_ENGINE_TILED4) return fail(NOC_EINVAL, "unknown engine");
    if (c->inject_mode > 2) return fail(NOC_EINVAL, "inject_mode out of range");
    if (c->age_base > AGE_MAX) return fail(NOC_EINVAL, "age_base > 65535 (R32)");
    if (c->band_streams > 1) return fail(NOC_EINVAL, "band_streams must be 0 or 1");
    if (c->mig_hist > 16) return fail(NOC_EINVAL, "mig_hist must be 0..16");
    if (c->mig_hist && (c->mode != NOC_MODE_LSPD || c->nfl_b2 < 1 || c->nfl_b2 > 16 ||
                        (uint64_t)c->tags_per_node * c->mesh_w * c->mesh_h > (1ull << 28)))
        return fail(NOC_EINVAL, "migration needs LSPD mode, nfl_b2 1..16 and a tag space <= 2^28 (R50)");
    if (c->band_streams && (c->bands < 2 || c->world_size > 1 ||
                            (c->engine != NOC_ENGINE_TILED && c->engine != NOC_ENGINE_AUTO)))
        return fail(NOC_EINVAL, "band_streams needs bands >= 2 in one process and the TILED engine");
    if (c->mem_mode > 2 || (c->mem_mode && (c->mode != NOC_MODE_LSPD || c->mig_hist || c->nfl_b2 < 1 || c->nfl_b2 > 16)))
        return fail(NOC_EINVAL, "memory nodes (mem_mode 1/2) need LSPD mode, no migration and nfl_b2 1..16 (R54)");
    if (c->mem_mode == 2 && (c->mem_ctrls < 1 || c->mem_ctrls > 64 || (c->mem_ctrls + 1) / 2 > c->mesh_w))
        return fail(NOC_EINVAL, "mem_ctrls must be 1..64 with ceil(M/2) <= mesh_w");
    if (c->hub_sendq_cap && (c->hub_sendq_cap < c->sendq_cap || c->hub_sendq_cap > 1024 ||
                             (c->hub_sendq_cap & (c->hub_sendq_cap - 1))))
        return fail(NOC_EINVAL, "hub_sendq_cap must be 0 or a power of two in sendq_cap..1024 (R56)");
    if (c->inject_mode && c->engine == NOC_ENGINE_TILED4)
        return fail(NOC_EINVAL, "inject_mode 1/2 (NEXT-f4) are not supported by the TILED4 engine");
    if (c->mode == NOC_MODE_LSPD && c->l1_sets &&
        (c->l1_sets > 65536 || c->l1_ways < 1 || c->l1_ways > 16 || c->l1_miss_lat < 1 || c->l1_miss_lat >= (1u << 29)))
        return fail(NOC_EINVAL, "l1 geometry: sets 0..65536, ways 1..16, miss latency 1..2^29-1");
    if (c->n_script && !c->script) return fail(NOC_EINVAL, "n_script > 0 with a null script");
    for (uint64_t i = 0; i < c->n_script; ++i) {
        const noc_sim_event &e = c->script[i];
        if (e.node >= N) return fail(NOC_EINVAL, "script node out of range");
        if (c->mode == NOC_MODE_UR && (e.value >= N || e.value == e.node))
            return fail(NOC_EINVAL, "script probe destination invalid");
        if (c->mode == NOC_MODE_LSPD && (uint64_t)e.value >= (uint64_t)c->tags_per_node * N)
            return fail(NOC_EINVAL, "script tag out of range");
    }
    return NOC_OK;
}

extern "C" void noc_sim_destroy(noc_sim *s)
{
    if (!s) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(s->device);
    if (s->stream) cudaStreamSynchronize(s->stream);
    for (void *p : s->ipc_opened) cudaIpcCloseMemHandle(p);
    if (s->comm) ncclCommDestroy(s->comm);
    for (void *p : s->allocs) cudaFree(p);
    for (auto &pd : s->pending) {
        if (pd.host) cudaFreeHost(pd.host);
        if (pd.done) cudaEventDestroy(pd.done);
    }
    if (s->cstream) { cudaStreamSynchronize(s->cstream); cudaStreamDestroy(s->cstream); }
    for (int k = 0; k < MAX_BANDS; ++k) {
        if (s->bst[k]) { cudaStreamSynchronize(s->bst[k]); cudaStreamDestroy(s->bst[k]); }
        if (s->bev[k]) cudaEventDestroy(s->bev[k]);
    }
    if (s->mev) cudaEventDestroy(s->mev);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    if (s->stream) cudaStreamDestroy(s->stream);
    cudaSetDevice(cur);
    delete s;
}

// rows of band g of P
static void band_rows(uint32_t H, int P, int g, uint32_t *row0, uint32_t *rows)
{
    uint32_t a = (uint32_t)((uint64_t)g * H / P), b = (uint32_t)((uint64_t)(g + 1) * H / P);
    *row0 = a;
    *rows = b - a;
}

extern "C" int noc_sim_band_rows(uint32_t mesh_h, int32_t world_size, int32_t rank, uint32_t *row0, uint32_t *rows)
{
    if (!row0 || !rows) return fail(NOC_EINVAL, "null argument");
    if (world_size < 1 || rank < 0 || rank >= world_size || (uint32_t)world_size > mesh_h)
        return fail(NOC_EINVAL, "bad world_size/rank");
    band_rows(mesh_h, world_size, rank, row0, rows);
    return NOC_OK;
}

// allocate and initialise the state of one band (DESIGN 6.1)
static int make_band(noc_sim *s, const noc_sim_config *cfg, int g, Dev &D)
{
    int rc;
    memset(&D, 0, sizeof D);
    D.W = cfg->mesh_w;
    D.H = cfg->mesh_h;
    D.N = D.W * D.H;
    band_rows(D.H, s->P, g, &D.row0, &D.rows);
    D.n0 = D.row0 * D.W;
    D.nloc = D.rows * D.W;
    D.mode = cfg->mode;
    D.prio = cfg->prio;
    D.route = cfg->route;
    D.dir_mode = cfg->mode == NOC_MODE_LSPD ? cfg->dir_mode : 0u;
    D.dir_node = cfg->dir_node;
    D.l1_sets = cfg->mode == NOC_MODE_LSPD ? cfg->l1_sets : 0u;
    D.l1_ways = cfg->l1_ways;
    D.l1_miss_lat = cfg->l1_miss_lat;
    D.inject_mode = cfg->inject_mode;
    D.age_base = cfg->age_base;
    D.mig_hist = cfg->mode == NOC_MODE_LSPD ? cfg->mig_hist : 0u;
    D.nfl_b2 = cfg->nfl_b2;
    D.mem_mode = cfg->mode == NOC_MODE_LSPD ? cfg->mem_mode : 0u;
    D.mem_ctrls = cfg->mem_ctrls;
    D.hub_cap = cfg->hub_sendq_cap;
    D.sets = cfg->mode == NOC_MODE_LSPD ? cfg->l2_sets : 1u;
    D.ways = cfg->mode == NOC_MODE_LSPD ? cfg->l2_ways : 1u;
    D.tpn = cfg->mode == NOC_MODE_LSPD ? cfg->tags_per_node : 0u;
    D.priv = cfg->priv_tags;
    D.thr_inj = cfg->thr_inj;
    D.thr_priv = cfg->thr_priv;
    D.l2_hit_lat = cfg->l2_hit_lat;
    D.mem_lat = cfg->mem_lat;
    D.nfl_ra = cfg->nfl_ra;
    D.qcap = cfg->sendq_cap;
    D.nb = cfg->hist_bins;
    D.seed_lo = (uint32_t)cfg->seed;
    D.seed_hi = (uint32_t)(cfg->seed >> 32);
    D.gen = 1;
    D.wmagic = (uint32_t)(((1ull << 32) + D.W - 1) / D.W);
    D.cnt = s->cnt;
    D.hist = s->hist;
    D.err = s->err;
    const size_t n = D.nloc;
    for (int b = 0; b < 2; ++b) {
        if ((rc = dalloc(s, &D.flit[b], 4 * n))) return rc;
        if ((rc = dalloc(s, &D.flag[b], n))) return rc;
    }
    if ((rc = dalloc(s, &D.fifo_ctl, n))) return rc;
    if ((rc = dalloc(s, &D.fifo_pkt, n * D.qcap))) return rc;
    if (D.hub_cap) {
        // hub nodes of this band (R56): the central directory node, the memory
        // controllers; each gets a FIFO of hub_cap packets
        std::vector<uint32_t> hubs;
        if (D.dir_mode == 1u) hubs.push_back(D.dir_node);
        if (D.mem_mode == 2u)
            for (uint32_t k = 0; k < D.mem_ctrls; ++k) hubs.push_back(mem_ctrl_node(D.W, D.H, D.mem_ctrls, k));
        std::vector<uint8_t> hub_of(n, 0);
        uint32_t nh = 0;
        for (uint32_t h : hubs)
            if (h >= D.n0 && h < D.n0 + D.nloc && !hub_of[h - D.n0]) hub_of[h - D.n0] = (uint8_t)++nh;
        if ((rc = dalloc(s, &D.hub_of, n))) return rc;
        if ((rc = dalloc(s, &D.hub_pkt, (size_t)std::max<uint32_t>(nh, 1u) * D.hub_cap))) return rc;
        CU(cudaMemcpy(D.hub_of, hub_of.data(), n, cudaMemcpyHostToDevice));
    }
    if (cfg->mode == NOC_MODE_LSPD) {
        if ((rc = dalloc(s, &D.core_hot, n))) return rc;
        if ((rc = dalloc(s, &D.core_cold, n))) return rc;
        if ((rc = dalloc(s, &D.l2, n * D.sets * D.ways))) return rc;
        if (D.l1_sets && (rc = dalloc(s, &D.l1, n * D.l1_sets * D.l1_ways))) return rc;
        uint64_t b0 = s->bytes;
        // distributed: the entries of the tags homed on this band's nodes;
        // centralized: the whole array in the directory node's band (R40)
        if (D.dir_mode) D.loc_n = (D.dir_node >= D.n0 && D.dir_node < D.n0 + D.nloc) ? (uint64_t)D.tpn * D.N : 0u;
        else D.loc_n = (uint64_t)D.tpn * n;
        if ((rc = dalloc(s, &D.loc, (size_t)D.loc_n))) return rc;
        if (D.mig_hist) {   // NEXT-f2 state: accessor rings, directory transit flags, inbound reassembly
            if ((rc = dalloc(s, &D.l2h, n * D.sets * D.ways * (size_t)D.mig_hist))) return rc;
            if ((rc = dalloc(s, &D.loc_mig, (size_t)D.loc_n))) return rc;
            if ((rc = dalloc(s, &D.migrx, n * 4u))) return rc;
        }
        s->loc_bytes += s->bytes - b0;
    }
    // script events of this band's nodes, per node ordered by (cycle, input order)
    std::vector<uint32_t> off(n + 1, 0);
    std::vector<uint4> ev;
    if (cfg->n_script) {
        std::vector<uint64_t> idx;
        for (uint64_t i = 0; i < cfg->n_script; ++i)
            if (cfg->script[i].node >= D.n0 && cfg->script[i].node < D.n0 + D.nloc) idx.push_back(i);
        std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
            const noc_sim_event &x = cfg->script[a], &y = cfg->script[b];
            if (x.node != y.node) return x.node < y.node;
            return x.cycle < y.cycle;
        });
        ev.resize(idx.size());
        for (size_t i = 0; i < idx.size(); ++i) {
            const noc_sim_event &x = cfg->script[idx[i]];
            ev[i] = make_uint4((uint32_t)x.cycle, (uint32_t)(x.cycle >> 32), x.value, 0u);
            off[x.node - D.n0 + 1] += 1;
        }
        for (size_t i = 0; i < n; ++i) off[i + 1] += off[i];
        D.has_script = 1;
    }
    uint4 *dev_ev = nullptr;
    uint32_t *dev_off = nullptr;
    if ((rc = dalloc(s, &dev_ev, ev.size()))) return rc;
    if ((rc = dalloc(s, &dev_off, n + 1))) return rc;
    if ((rc = dalloc(s, &D.script_pos, n))) return rc;
    if (!ev.empty()) CU(cudaMemcpy(dev_ev, ev.data(), ev.size() * sizeof(uint4), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dev_off, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    D.script = dev_ev;
    D.script_off = dev_off;
    return NOC_OK;
}

// stream-ordered barrier / reductions across ranks (no-ops when world == 1)
static int allreduce_u64(noc_sim *s, unsigned long long *buf, size_t count)
{
    if (s->world == 1) return NOC_OK;
    NC(ncclAllReduce(buf, buf, count, ncclUint64, ncclSum, s->comm, s->stream));
    return NOC_OK;
}
static int allreduce_u32(noc_sim *s, uint32_t *buf, size_t count)
{
    if (s->world == 1) return NOC_OK;
    NC(ncclAllReduce(buf, buf, count, ncclUint32, ncclSum, s->comm, s->stream));
    return NOC_OK;
}

// multi-GPU: map the neighbour bands' boundary slots (CUDA IPC over NVLink)
static int link_ranks(noc_sim *s)
{
    Dev &D = s->D[0];
    cudaIpcMemHandle_t mine;
    CU(cudaIpcGetMemHandle(&mine, D.ll));
    uint8_t *dev_h = nullptr;
    int rc;
    if ((rc = dalloc(s, &dev_h, (size_t)64 * s->world))) return rc;
    CU(cudaMemcpy(dev_h + 64 * s->rank, &mine, 64, cudaMemcpyHostToDevice));
    NC(ncclAllGather(dev_h + 64 * s->rank, dev_h, 64, ncclUint8, s->comm, s->stream));
    std::vector<uint8_t> all((size_t)64 * s->world);
    CU(cudaMemcpyAsync(all.data(), dev_h, all.size(), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (int side = 0; side < 2; ++side) {
        const int r = side == 0 ? s->rank - 1 : s->rank + 1;
        if (r < 0 || r >= s->world) continue;
        cudaIpcMemHandle_t h;
        memcpy(&h, all.data() + 64 * r, 64);
        void *p = nullptr;
        CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        s->ipc_opened.push_back(p);
        uint32_t row0, rows;
        band_rows(D.H, s->P, r, &row0, &rows);
        D.ll_nb[side] = (unsigned long long *)p;
        D.nloc_nb[side] = rows * D.W;
    }
    return NOC_OK;
}

// multi-GPU, PERSIST engine: map the neighbour bands' flit / flag arrays (both
// parities) and progress counters, and learn their nodes per CTA
static int link_ranks_persist(noc_sim *s)
{
    Dev &D = s->D[0];
    const int NH = 5;   // flit[0], flit[1], flag[0], flag[1], progress
    void *mine_p[NH] = {D.flit[0], D.flit[1], D.flag[0], D.flag[1], D.progress};
    uint8_t rec[NH * 64 + 8];
    memset(rec, 0, sizeof rec);
    for (int i = 0; i < NH; ++i) {
        cudaIpcMemHandle_t h;
        CU(cudaIpcGetMemHandle(&h, mine_p[i]));
        memcpy(rec + 64 * i, &h, 64);
    }
    memcpy(rec + NH * 64, &D.npc, 4);
    const size_t R = sizeof rec;
    uint8_t *dev_h = nullptr;
    int rc;
    if ((rc = dalloc(s, &dev_h, R * s->world))) return rc;
    CU(cudaMemcpy(dev_h + R * s->rank, rec, R, cudaMemcpyHostToDevice));
    NC(ncclAllGather(dev_h + R * s->rank, dev_h, R, ncclUint8, s->comm, s->stream));
    std::vector<uint8_t> all(R * s->world);
    CU(cudaMemcpyAsync(all.data(), dev_h, all.size(), cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    for (int side = 0; side < 2; ++side) {
        const int r = side == 0 ? s->rank - 1 : s->rank + 1;
        if (r < 0 || r >= s->world) continue;
        void *p[NH];
        for (int i = 0; i < NH; ++i) {
            cudaIpcMemHandle_t h;
            memcpy(&h, all.data() + R * r + 64 * i, 64);
            CU(cudaIpcOpenMemHandle(&p[i], h, cudaIpcMemLazyEnablePeerAccess));
            s->ipc_opened.push_back(p[i]);
        }
        uint32_t row0, rows;
        band_rows(D.H, s->P, r, &row0, &rows);
        D.flit_nb[side][0] = (uint4 *)p[0];
        D.flit_nb[side][1] = (uint4 *)p[1];
        D.flag_nb[side][0] = (uint32_t *)p[2];
        D.flag_nb[side][1] = (uint32_t *)p[3];
        D.prog_nb[side] = (uint32_t *)p[4];
        memcpy(&D.npc_nb[side], all.data() + R * r + NH * 64, 4);
        D.nloc_nb[side] = rows * D.W;
    }
    return NOC_OK;
}

extern "C" int noc_sim_create(const noc_sim_config *cfg, noc_sim **out)
{
    if (!out) return fail(NOC_EINVAL, "null out");
    *out = nullptr;
    int rc = validate(cfg);
    if (rc) return rc;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(NOC_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (cfg->device < 0 || cfg->device >= ndev) return fail(NOC_EINVAL, "device ordinal out of range");

    noc_sim *s = new noc_sim();
    s->cfg = *cfg;
    s->cfg.script = nullptr;
    s->device = cfg->device;
    s->world = cfg->world_size;
    s->rank = cfg->rank;
    if (s->world > 1) { s->nb = 1; s->P = s->world; s->g0 = s->rank; }
    else { s->nb = cfg->bands > 1 ? (int)cfg->bands : 1; s->P = s->nb; s->g0 = 0; }
    auto bail = [&](int code) { noc_sim_destroy(s); return code; };
    if (cudaSetDevice(s->device) != cudaSuccess) return bail(fail(NOC_ECUDA, "cudaSetDevice failed"));
    cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, s->device);
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&s->ev0) != cudaSuccess || cudaEventCreate(&s->ev1) != cudaSuccess)
        return bail(fail(NOC_ECUDA, "stream/event creation failed"));
    if (s->world > 1) {
        ncclUniqueId id;
        memcpy(&id, cfg->nccl_id, 128);
        ncclResult_t r = ncclCommInitRank(&s->comm, s->world, id, s->rank);
        if (r != ncclSuccess) return bail(fail(NOC_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
    }

    if ((rc = dalloc(s, &s->cnt, NCOUNTERS))) return bail(rc);
    if ((rc = dalloc(s, &s->hist, 3 * (size_t)cfg->hist_bins))) return bail(rc);
    if ((rc = dalloc(s, &s->err, 1))) return bail(rc);
    if ((rc = dalloc(s, &s->d_scratch, DRAIN_CHUNK + 2))) return bail(rc);
    if ((rc = dalloc(s, &s->d_hash, 1))) return bail(rc);
    if ((rc = dalloc(s, &s->d_red, NCOUNTERS + 3 * (size_t)cfg->hist_bins + 2))) return bail(rc);
    for (int k = 0; k < s->nb; ++k)
        if ((rc = make_band(s, cfg, s->g0 + k, s->D[k]))) return bail(rc);

    // engine: TILED when every band's tiles fit one CTA of <= TILE_BLOCK_MAX
    // threads per SM, else PERSIST (DESIGN 6.2); bands need TILED or PERSIST
    s->engine = cfg->engine;
    if (s->P > 1 && s->engine == NOC_ENGINE_STEP) return bail(fail(NOC_EINVAL, "row bands need the TILED or PERSIST engine"));
    // AUTO tries TILED (one thread per node), then TILED4 (4 lanes per node,
    // 2 CTAs per SM), then PERSIST: TILED is the fastest at the bench size
    // (DESIGN 6.4, profiles/r01_ab_engines.txt)
    // opt-in (NOCSIM_CLUSTER=1): a single band of up to TILE_CLUSTER_MAX tiles
    // runs as ONE thread-block cluster -- cross-tile links are DSMEM stores and
    // the cycle barrier is the cluster barrier (tile_kernel.cuh, FEAT bit 3).
    // Parity-green, but not the default: at C2 it is faster only without load
    // (1.01 vs 1.79 us per cycle idle, 4.2 vs 3.2 at lambda 0.05: 16 CTAs of 256
    // nodes wait for the slowest of 128 warps every cycle, profiles/r02_cluster_c2.txt)
    if ((s->engine == NOC_ENGINE_AUTO || s->engine == NOC_ENGINE_TILED) && s->nb == 1 && s->world == 1 &&
        cfg->route == 0 && cfg->inject_mode == 0 && getenv("NOCSIM_CLUSTER")) {
        const uint64_t nodes = (uint64_t)s->D[0].W * s->D[0].rows;
        uint32_t tiles = 0, np = 0;
        if (nodes > TILE_BLOCK_MAX && nodes <= (uint64_t)TILE_CLUSTER_MAX * TILE_BLOCK_MAX &&
            tiled_plan(s->D[0], TILE_CLUSTER_MAX, &tiles, &np) && tiles > 1 &&
            tiled_prepare_cluster(tiled_kernel_mode(s->D[0]), cfg->hist_bins, np, tiles, &s->t_smem_hist) ==
                cudaSuccess) {
            s->engine = NOC_ENGINE_TILED;
            s->t_tpad = np;
            s->set.nbands = 1;
            s->set.general = 0;
            s->set.cluster = tiles;
            s->set.tile0[0] = 0;
            s->set.tile0[1] = tiles;
            s->set.d[0] = s->D[0];
        }
        cudaGetLastError();
    }
    for (uint32_t cand : {NOC_ENGINE_TILED, NOC_ENGINE_TILED4}) {
        if (s->set.cluster) break;
        if (!(s->engine == NOC_ENGINE_AUTO || s->engine == cand)) continue;
        if (cand == NOC_ENGINE_TILED4 && cfg->inject_mode) continue;   // four lanes per router (R43)
        const bool four = cand == NOC_ENGINE_TILED4;
        bool ok = true;
        uint32_t np = four ? 8 : 32, total = 0;
        const uint32_t per_sm = four ? TILE4_MIN_BLOCKS : TILE_MIN_BLOCKS;
        const uint32_t budget = std::max<uint32_t>(1u, (uint32_t)s->sm_count * per_sm / (uint32_t)s->nb);
        s->set.nbands = (uint32_t)s->nb;
        s->set.general = s->nb > 1 || s->world > 1;
        s->set.tile0[0] = 0;
        for (int k = 0; k < s->nb && ok; ++k) {
            uint32_t tiles = 0, npk = 0;
            ok = four ? tiled4_plan(s->D[k], budget, &tiles, &npk) : tiled_plan(s->D[k], budget, &tiles, &npk);
            np = std::max(np, npk);
            total += tiles;
            s->set.tile0[k + 1] = total;
        }
        cudaError_t ce = cudaErrorInvalidConfiguration;
        if (ok) ce = four ? tiled4_prepare(cfg->mode, cfg->hist_bins, np, total, s->device, &s->t_smem_hist)
                          : tiled_prepare(tiled_kernel_mode(s->D[0]),
                                          cfg->route | (cfg->inject_mode ? 2u : 0u) | (s->nb > 1 || s->world > 1 ? 4u : 0u),
                                          cfg->hist_bins, np, total, s->device, &s->t_smem_hist);
        if (ce == cudaSuccess) {
            s->engine = cand;
            s->t_tpad = np;
            break;
        }
        cudaGetLastError();
        if (s->engine == cand)
            return bail(fail(NOC_EINVAL, std::string("TILED engine does not fit this mesh: ") + cudaGetErrorString(ce)));
    }
    if (s->engine == NOC_ENGINE_AUTO) s->engine = NOC_ENGINE_PERSIST;
    if ((s->engine == NOC_ENGINE_TILED || s->engine == NOC_ENGINE_TILED4) && !s->set.cluster) {
        for (int k = 0; k < s->nb; ++k)
            if ((rc = dalloc(s, &s->D[k].ll, (size_t)32u * s->D[k].nloc))) return bail(rc);
        // neighbour bands' boundary slots
        if (s->world > 1) {
            if ((rc = link_ranks(s))) return bail(rc);
        } else {
            for (int k = 0; k < s->nb; ++k) {
                if (k > 0) { s->D[k].ll_nb[0] = s->D[k - 1].ll; s->D[k].nloc_nb[0] = s->D[k - 1].nloc; }
                if (k + 1 < s->nb) { s->D[k].ll_nb[1] = s->D[k + 1].ll; s->D[k].nloc_nb[1] = s->D[k + 1].nloc; }
            }
        }
        for (int k = 0; k < s->nb; ++k) {
            if (launch_ll_reset(s->D[k], 0, s->stream) != cudaSuccess) return bail(fail(NOC_ECUDA, "ll reset failed"));
            s->set.d[k] = s->D[k];
        }
        if (cfg->band_streams) {
            if (s->engine != NOC_ENGINE_TILED) return bail(fail(NOC_EINVAL, "band_streams needs the TILED engine"));
            // each band alone in its launch (like one rank's band), on its own stream
            s->split = 1;
            if (cudaEventCreateWithFlags(&s->mev, cudaEventDisableTiming) != cudaSuccess)
                return bail(fail(NOC_ECUDA, "event creation failed"));
            for (int k = 0; k < s->nb; ++k) {
                if (cudaStreamCreateWithFlags(&s->bst[k], cudaStreamNonBlocking) != cudaSuccess ||
                    cudaEventCreateWithFlags(&s->bev[k], cudaEventDisableTiming) != cudaSuccess)
                    return bail(fail(NOC_ECUDA, "band stream creation failed"));
                DevSet &B = s->bset[k];
                B = s->set;
                B.d[0] = s->D[k];
                B.nbands = 1;
                B.tile0[0] = 0;
                B.tile0[1] = s->set.tile0[k + 1] - s->set.tile0[k];
                B.general = 1;
            }
        }
    }
    if (s->engine == NOC_ENGINE_PERSIST) {
        // each band: its CTAs, nodes per CTA and progress counters; then the
        // neighbour bands' link arrays and progress (in-process, or CUDA IPC)
        s->set.nbands = (uint32_t)s->nb;
        s->set.tile0[0] = 0;
        for (int k = 0; k < s->nb; ++k) {
            uint32_t g = 0, npc = 0;
            cudaError_t ce = persist_configure(s->D[k], s->device, (uint32_t)s->nb, &g, &npc, &s->p_smem_hist);
            if (ce != cudaSuccess) return bail(fail(NOC_ECUDA, std::string("persist_configure: ") + cudaGetErrorString(ce)));
            s->D[k].npc = npc;
            if ((rc = dalloc(s, &s->D[k].progress, g))) return bail(rc);
            s->set.tile0[k + 1] = s->set.tile0[k] + g;
        }
        s->p_grid = s->set.tile0[s->nb];
        s->p_npc = s->D[0].npc;
        s->progress = s->D[0].progress;
        if (s->world > 1) {
            if ((rc = link_ranks_persist(s))) return bail(rc);
        } else {
            for (int k = 0; k < s->nb; ++k)
                for (int side = 0; side < 2; ++side) {
                    const int j = side == 0 ? k - 1 : k + 1;
                    if (j < 0 || j >= s->nb) continue;
                    Dev &D = s->D[k], &E = s->D[j];
                    for (int b = 0; b < 2; ++b) { D.flit_nb[side][b] = E.flit[b]; D.flag_nb[side][b] = E.flag[b]; }
                    D.prog_nb[side] = E.progress;
                    D.npc_nb[side] = E.npc;
                    D.nloc_nb[side] = E.nloc;
                }
        }
        for (int k = 0; k < s->nb; ++k) s->set.d[k] = s->D[k];
    }
    // streamed scripts (R57): the last create-time event cycle of every node
    {
        const uint64_t N = (uint64_t)cfg->mesh_w * cfg->mesh_h;
        s->script_last.assign(N, 0);
        s->script_any.assign(N, 0);
        for (uint64_t i = 0; i < cfg->n_script; ++i) {
            const noc_sim_event &x = cfg->script[i];
            if (!s->script_any[x.node] || x.cycle > s->script_last[x.node]) s->script_last[x.node] = x.cycle;
            s->script_any[x.node] = 1;
        }
        if (cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(NOC_ECUDA, "copy stream creation failed"));
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(NOC_ECUDA, "init sync failed"));
    if (s->world > 1) {   // every rank has mapped its neighbours before anyone runs
        if ((rc = allreduce_u32(s, s->d_scratch, 1))) return bail(rc);
        if (cudaStreamSynchronize(s->stream) != cudaSuccess) return bail(fail(NOC_ECUDA, "init barrier failed"));
    }
    *out = s;
    return NOC_OK;
}

static int check_err(noc_sim *s)
{
    uint32_t err = 0;
    CU(cudaMemcpyAsync(&err, s->err, 4, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    if (err) {
        s->poisoned = 1;
        if (err & 0x80000000u) {
            char b[96];
            snprintf(b, sizeof b, "boundary / neighbour wait timed out (flags 0x%08x)", err);
            return fail(NOC_ECUDA, b);
        }
        if (err & ERR_DROP) return fail(NOC_EOVERFLOW, "send FIFO overflow in LSPD mode (R21: a dropped protocol message)");
        if (err & ERR_MIGRX) return fail(NOC_EOVERFLOW, "more than 4 inbound migrations at one node (R52)");
        if (err & (ERR_AGE | ERR_PEND)) return fail(NOC_EOVERFLOW, "field width exceeded (flit age, lifetime or pend)");
        return fail(NOC_ECUDA, "model assertion failed on device (protocol / EV holder)");
    }
    return NOC_OK;
}

// Refresh the launch sets' copies of band k's view after a host-side change
static void sync_band_views(noc_sim *s, int k)
{
    s->set.d[k] = s->D[k];
    if (s->split) s->bset[k].d[0] = s->D[k];
}

// Merge the pushed script chunks into the bands' event queues (R57): per node
// the events not consumed yet, then the pushed ones; consumed events are
// dropped, so device memory holds only what is still to come.
static int merge_scripts(noc_sim *s)
{
    for (auto &pd : s->pending) {
        CU(cudaStreamWaitEvent(s->stream, pd.done, 0));
        for (int k = 0; k < s->nb; ++k) {
            Dev &D = s->D[k];
            const size_t n = D.nloc;
            uint32_t *cnt = nullptr, *new_off = nullptr, *new_base = nullptr;
            int rc;
            if ((rc = dalloc(s, &cnt, n))) return rc;
            CU(launch_script_count(D, pd.off[k], cnt, s->stream));
            std::vector<uint32_t> h(n), off(n + 1, 0);
            CU(cudaMemcpyAsync(h.data(), cnt, n * 4, cudaMemcpyDeviceToHost, s->stream));
            CU(cudaStreamSynchronize(s->stream));
            for (size_t l = 0; l < n; ++l) off[l + 1] = off[l] + h[l];
            uint4 *new_ev = nullptr;
            if ((rc = dalloc(s, &new_off, n + 1))) return rc;
            if ((rc = dalloc(s, &new_base, n))) return rc;
            if ((rc = dalloc(s, &new_ev, off[n]))) return rc;
            CU(cudaMemcpyAsync(new_off, off.data(), (n + 1) * 4, cudaMemcpyHostToDevice, s->stream));
            CU(launch_script_merge(D, pd.off[k], pd.ev[k], new_off, new_ev, new_base, s->stream));
            CU(cudaStreamSynchronize(s->stream));
            dfree(s, (void *)D.script);
            dfree(s, (void *)D.script_off);
            if (D.script_base) dfree(s, D.script_base);
            dfree(s, cnt);
            dfree(s, pd.ev[k]);
            dfree(s, pd.off[k]);
            D.script = new_ev;
            D.script_off = new_off;
            D.script_base = new_base;
            D.has_script = 1;
            sync_band_views(s, k);
        }
        cudaFreeHost(pd.host);
        cudaEventDestroy(pd.done);
    }
    s->pending.clear();
    return NOC_OK;
}

static void set_gen(noc_sim *s, uint32_t gen)
{
    for (int k = 0; k < s->nb; ++k) {
        s->D[k].gen = gen;
        s->set.d[k].gen = gen;
        s->bset[k].d[0].gen = gen;   // virtual ranks: each band's own launch set
    }
}

// Advance n cycles with the handle's engine; activity (device, may be null)
// receives per-cycle busy-CTA counts when draining (n <= DRAIN_CHUNK).
static int advance_launches(noc_sim *s, uint64_t n, uint32_t *activity);

static int advance(noc_sim *s, uint64_t n, uint32_t *activity)
{
    // pushed script chunks (R57): merged before the launches if any of their
    // events may be due in this run, else after them (their copy overlaps it)
    if (!s->pending.empty()) {
        uint64_t due = ~0ull;
        for (auto &pd : s->pending) due = std::min(due, pd.min_cycle);
        if (due < s->t + n) {
            int rc = merge_scripts(s);
            if (rc) return rc;
        } else {
            int rc = advance_launches(s, n, activity);
            if (rc) return rc;
            return merge_scripts(s);
        }
    }
    return advance_launches(s, n, activity);
}

static int advance_launches(noc_sim *s, uint64_t n, uint32_t *activity)
{
    cudaError_t e;
    if (s->split) {
        // virtual ranks: per band, the launch sequence of one rank (DESIGN 8)
        // -- refresh its boundary slots, barrier with the other bands, its own
        // cooperative launch, barrier -- each band on its own stream; the
        // barriers are events every band stream waits for
        auto barrier = [&]() -> int {
            for (int b = 0; b < s->nb; ++b) CU(cudaEventRecord(s->bev[b], s->bst[b]));
            for (int b = 0; b < s->nb; ++b)
                for (int j = 0; j < s->nb; ++j)
                    if (j != b) CU(cudaStreamWaitEvent(s->bst[b], s->bev[j], 0));
            return NOC_OK;
        };
        CU(cudaEventRecord(s->mev, s->stream));
        for (int b = 0; b < s->nb; ++b) CU(cudaStreamWaitEvent(s->bst[b], s->mev, 0));
        uint64_t done = 0;
        int rc;
        while (done < n) {
            uint32_t k = (uint32_t)std::min<uint64_t>(n - done, PERSIST_CHUNK);
            for (int b = 0; b < s->nb; ++b) CU(launch_ll_refresh(s->D[b], s->t + done, s->bst[b]));
            if ((rc = barrier())) return rc;
            uint32_t *act = activity ? activity + done : nullptr;
            for (int b = 0; b < s->nb; ++b) {
                e = launch_tiled(s->bset[b], s->t + done, k, s->t_tpad, s->t_smem_hist, act, s->bst[b]);
                if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("tiled band launch: ") + cudaGetErrorString(e));
            }
            if ((rc = barrier())) return rc;
            done += k;
            s->launches += 1;
        }
        for (int b = 0; b < s->nb; ++b) CU(cudaStreamWaitEvent(s->stream, s->bev[b], 0));
    } else if (s->engine == NOC_ENGINE_TILED || s->engine == NOC_ENGINE_TILED4) {
        uint64_t done = 0;
        while (done < n) {
            uint32_t k = (uint32_t)std::min<uint64_t>(n - done, PERSIST_CHUNK);
            if (!s->set.cluster)
                for (int b = 0; b < s->nb; ++b) CU(launch_ll_refresh(s->D[b], s->t + done, s->stream));
            // ranks: every rank's refresh completes before any rank's kernel
            // starts, else a fast neighbour's first boundary stores (stamp t0+1)
            // could be re-stamped t0-1 by this rank's late refresh (a stream-
            // ordered barrier: the all-reduce completes only once every rank
            // enqueued it after its own refresh)
            if (s->world > 1) {
                int rc0 = allreduce_u32(s, s->d_scratch + DRAIN_CHUNK + 1, 1);
                if (rc0) return rc0;
            }
            uint32_t *act = activity ? activity + done : nullptr;
            e = s->engine == NOC_ENGINE_TILED4
                    ? launch_tiled4(s->set, s->t + done, k, s->t_tpad, s->t_smem_hist, act, s->stream)
                    : launch_tiled(s->set, s->t + done, k, s->t_tpad, s->t_smem_hist, act, s->stream);
            if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("tiled launch: ") + cudaGetErrorString(e));
            // ranks: the next refresh may only run once the neighbours stopped
            // writing into this band's boundary slots
            int rc = allreduce_u32(s, s->d_scratch + DRAIN_CHUNK, 1);
            if (rc) return rc;
            done += k;
            s->launches += 1;
        }
    } else if (s->engine == NOC_ENGINE_PERSIST) {
        uint64_t done = 0;
        while (done < n) {
            uint32_t k = (uint32_t)std::min<uint64_t>(n - done, PERSIST_CHUNK);
            e = launch_persist(s->set, s->t + done, k, s->pbase, s->p_smem_hist, activity ? activity + done : nullptr,
                               s->stream);
            if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("persistent launch: ") + cudaGetErrorString(e));
            s->pbase += k;
            done += k;
            s->launches += 1;
        }
    } else {
        for (uint64_t i = 0; i < n; ++i) {
            e = launch_step(s->D[0], s->t + i, activity ? activity + i : nullptr, s->stream);
            if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("step launch: ") + cudaGetErrorString(e));
            s->launches += 1;
        }
    }
    s->t += n;
    return NOC_OK;
}

extern "C" int noc_sim_push_script(noc_sim *s, const noc_sim_event *ev, uint64_t n)
{
    if (!s) return fail(NOC_EINVAL, "null handle");
    if (s->poisoned) return fail(NOC_ESTATE, "handle poisoned by an earlier error");
    if (n && !ev) return fail(NOC_EINVAL, "null events");
    if (!n) return NOC_OK;
    const noc_sim_config *c = &s->cfg;
    const uint64_t N = (uint64_t)c->mesh_w * c->mesh_h;
    std::vector<uint64_t> idx(n);
    for (uint64_t i = 0; i < n; ++i) {
        const noc_sim_event &e = ev[i];
        if (e.node >= N) return fail(NOC_EINVAL, "script node out of range");
        if (c->mode == NOC_MODE_UR && (e.value >= N || e.value == e.node))
            return fail(NOC_EINVAL, "script probe destination invalid");
        if (c->mode == NOC_MODE_LSPD && (uint64_t)e.value >= (uint64_t)c->tags_per_node * N)
            return fail(NOC_EINVAL, "script tag out of range");
        idx[i] = i;
    }
    std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
        if (ev[a].node != ev[b].node) return ev[a].node < ev[b].node;
        return ev[a].cycle < ev[b].cycle;
    });
    for (uint64_t i = 0; i < n; ++i) {   // each node's queue stays ordered by cycle
        const noc_sim_event &e = ev[idx[i]];
        if ((i == 0 || ev[idx[i - 1]].node != e.node) && s->script_any[e.node] && e.cycle < s->script_last[e.node])
            return fail(NOC_EINVAL, "pushed events of a node must not precede its earlier events");
    }
    CU(cudaSetDevice(s->device));
    noc_sim::Pending pd{};
    pd.min_cycle = ~0ull;
    // pinned staging: per band the events (by node) and the per-node offsets
    size_t host_bytes = 0;
    std::vector<std::vector<uint4>> bev(s->nb);
    std::vector<std::vector<uint32_t>> boff(s->nb);
    for (int k = 0; k < s->nb; ++k) {
        const Dev &D = s->D[k];
        boff[k].assign(D.nloc + 1, 0);
        for (uint64_t i = 0; i < n; ++i) {
            const noc_sim_event &e = ev[idx[i]];
            if (e.node < D.n0 || e.node >= D.n0 + D.nloc) continue;
            bev[k].push_back(make_uint4((uint32_t)e.cycle, (uint32_t)(e.cycle >> 32), e.value, 0u));
            boff[k][e.node - D.n0 + 1] += 1;
        }
        for (uint32_t l = 0; l < D.nloc; ++l) boff[k][l + 1] += boff[k][l];
        host_bytes += bev[k].size() * sizeof(uint4) + boff[k].size() * 4;
    }
    CU(cudaMallocHost(&pd.host, std::max<size_t>(host_bytes, 16)));
    CU(cudaEventCreateWithFlags(&pd.done, cudaEventDisableTiming));
    uint8_t *hp = (uint8_t *)pd.host;
    for (int k = 0; k < s->nb; ++k) {
        int rc;
        pd.n[k] = (uint32_t)bev[k].size();
        if ((rc = dalloc(s, &pd.ev[k], bev[k].size()))) return rc;
        if ((rc = dalloc(s, &pd.off[k], boff[k].size()))) return rc;
        memcpy(hp, bev[k].data(), bev[k].size() * sizeof(uint4));
        CU(cudaMemcpyAsync(pd.ev[k], hp, bev[k].size() * sizeof(uint4), cudaMemcpyHostToDevice, s->cstream));
        hp += bev[k].size() * sizeof(uint4);
        memcpy(hp, boff[k].data(), boff[k].size() * 4);
        CU(cudaMemcpyAsync(pd.off[k], hp, boff[k].size() * 4, cudaMemcpyHostToDevice, s->cstream));
        hp += boff[k].size() * 4;
    }
    CU(cudaEventRecord(pd.done, s->cstream));
    for (uint64_t i = 0; i < n; ++i) {
        const noc_sim_event &e = ev[idx[i]];
        s->script_last[e.node] = e.cycle;     // ordered by cycle within a node
        s->script_any[e.node] = 1;
        pd.min_cycle = std::min(pd.min_cycle, e.cycle);
    }
    for (int k = 0; k < s->nb; ++k) {
        s->D[k].has_script = 1;
        sync_band_views(s, k);
    }
    s->pending.push_back(pd);
    return NOC_OK;
}

extern "C" int noc_sim_run(noc_sim *s, uint64_t n_cycles)
{
    if (!s) return fail(NOC_EINVAL, "null handle");
    if (s->poisoned) return fail(NOC_ESTATE, "handle poisoned by an earlier error");
    CU(cudaSetDevice(s->device));
    int rc = advance(s, n_cycles, nullptr);
    if (rc) return rc;
    CU(cudaStreamSynchronize(s->stream));
    return check_err(s);
}

extern "C" int noc_sim_run_timed(noc_sim *s, uint64_t n_cycles, double *device_ms)
{
    if (!s) return fail(NOC_EINVAL, "null handle");
    if (s->poisoned) return fail(NOC_ESTATE, "handle poisoned by an earlier error");
    CU(cudaSetDevice(s->device));
    CU(cudaEventRecord(s->ev0, s->stream));
    int rc = advance(s, n_cycles, nullptr);
    if (rc) return rc;
    CU(cudaEventRecord(s->ev1, s->stream));
    CU(cudaEventSynchronize(s->ev1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    if (device_ms) *device_ms = ms;
    return check_err(s);
}

extern "C" int noc_sim_drain(noc_sim *s, uint64_t max_cycles, uint64_t *used, int *drained)
{
    if (!s) return fail(NOC_EINVAL, "null handle");
    if (s->poisoned) return fail(NOC_ESTATE, "handle poisoned by an earlier error");
    CU(cudaSetDevice(s->device));
    uint64_t t0 = s->t, k = 0;
    int q = 0, rc;
    set_gen(s, 0);
    // generation is re-enabled on every exit path (a scope guard)
    struct GenGuard {
        noc_sim *s;
        ~GenGuard() { set_gen(s, 1); }
    } guard{s};
    // quiescent already?
    CU(cudaMemsetAsync(s->d_scratch, 0, 4, s->stream));
    for (int b = 0; b < s->nb; ++b) CU(launch_busy_count(s->D[b], s->t, s->d_scratch, s->stream));
    if ((rc = allreduce_u32(s, s->d_scratch, 1))) return rc;
    uint32_t busy = 0;
    CU(cudaMemcpyAsync(&busy, s->d_scratch, 4, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    q = busy == 0;
    std::vector<uint32_t> act(DRAIN_CHUNK);
    while (!q && k < max_cycles) {
        uint32_t chunk = (uint32_t)std::min<uint64_t>(DRAIN_CHUNK, max_cycles - k);
        CU(cudaMemsetAsync(s->d_scratch, 0, sizeof(uint32_t) * chunk, s->stream));
        rc = advance(s, chunk, s->d_scratch);
        if (rc) return rc;
        if ((rc = allreduce_u32(s, s->d_scratch, chunk))) return rc;
        CU(cudaMemcpyAsync(act.data(), s->d_scratch, sizeof(uint32_t) * chunk, cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        uint32_t i = 0;
        while (i < chunk && act[i] != 0) ++i;
        if (i < chunk) {
            // quiescent at the end of cycle (base + i): nothing changed after it,
            // so the cycle counter is rewound to the first quiescent cycle
            q = 1;
            k += i + 1;
            s->t = t0 + k;
            // boundary slots were stamped up to the end of the chunk: re-stamp
            // them EMPTY for the rewound cycle (nothing is in flight)
            if ((s->engine == NOC_ENGINE_TILED || s->engine == NOC_ENGINE_TILED4) && !s->set.cluster)
                for (int b = 0; b < s->nb; ++b) CU(launch_ll_reset(s->D[b], s->t, s->stream));
            if ((rc = allreduce_u32(s, s->d_scratch + DRAIN_CHUNK, 1))) return rc;
        } else {
            k += chunk;
        }
    }
    if (used) *used = k;
    if (drained) *drained = q;
    return check_err(s);
}

static const int NC_NAMED = 23;

// counters and histograms summed over ranks, on the host
static int gather_stats(noc_sim *s, std::vector<unsigned long long> &c, std::vector<unsigned long long> &h)
{
    const size_t nh = 3 * (size_t)s->cfg.hist_bins;
    c.resize(NCOUNTERS);
    h.resize(nh);
    if (s->world > 1) {
        CU(cudaMemcpyAsync(s->d_red, s->cnt, NCOUNTERS * 8, cudaMemcpyDeviceToDevice, s->stream));
        CU(cudaMemcpyAsync(s->d_red + NCOUNTERS, s->hist, nh * 8, cudaMemcpyDeviceToDevice, s->stream));
        int rc = allreduce_u64(s, s->d_red, NCOUNTERS + nh);
        if (rc) return rc;
        CU(cudaMemcpyAsync(c.data(), s->d_red, NCOUNTERS * 8, cudaMemcpyDeviceToHost, s->stream));
        CU(cudaMemcpyAsync(h.data(), s->d_red + NCOUNTERS, nh * 8, cudaMemcpyDeviceToHost, s->stream));
    } else {
        CU(cudaMemcpyAsync(c.data(), s->cnt, NCOUNTERS * 8, cudaMemcpyDeviceToHost, s->stream));
        CU(cudaMemcpyAsync(h.data(), s->hist, nh * 8, cudaMemcpyDeviceToHost, s->stream));
    }
    CU(cudaStreamSynchronize(s->stream));
    return NOC_OK;
}

extern "C" int noc_sim_stats(noc_sim *s, noc_sim_counters *out, uint64_t *hl, uint64_t *hd, uint64_t *ha, uint32_t nbins)
{
    if (!s) return fail(NOC_EINVAL, "null handle");
    if ((hl || hd || ha) && nbins != s->cfg.hist_bins) return fail(NOC_EINVAL, "nbins != hist_bins");
    CU(cudaSetDevice(s->device));
    std::vector<unsigned long long> c, h;
    int rc = gather_stats(s, c, h);
    if (rc) return rc;
    if (out) {
        int64_t *dst = &out->generated;
        out->cycle = (int64_t)s->t;
        for (int i = 0; i < NC_NAMED; ++i) dst[i] = (int64_t)c[i];
        for (int k = 0; k < 8; ++k) out->drops[k] = (int64_t)c[C_DROPS + k];
        out->l1_hits = (int64_t)c[C_L1HIT];
        out->l1_misses = (int64_t)c[C_L1MISS];
        out->wb_sent = (int64_t)c[C_WBSENT];
        out->wb_received = (int64_t)c[C_WBRCVD];
        int64_t *mg = &out->mig_requests;
        for (int k = 0; k < 8; ++k) mg[k] = (int64_t)c[C_MIGREQ + k];
        int64_t *mm = &out->mem_fills_sent;
        for (int k = 0; k < 4; ++k) mm[k] = (int64_t)c[C_MEMFILLSENT + k];
    }
    uint64_t *hs[3] = {hl, hd, ha};
    for (int k = 0; k < 3; ++k)
        if (hs[k]) memcpy(hs[k], h.data() + (size_t)k * s->cfg.hist_bins, sizeof(uint64_t) * s->cfg.hist_bins);
    return NOC_OK;
}

extern "C" int noc_sim_state_hash(noc_sim *s, uint64_t *out)
{
    if (!s || !out) return fail(NOC_EINVAL, "null argument");
    CU(cudaSetDevice(s->device));
    CU(cudaMemsetAsync(s->d_hash, 0, 8, s->stream));
    for (int b = 0; b < s->nb; ++b) CU(launch_hash(s->D[b], s->t, s->d_hash, s->stream));
    int rc = allreduce_u64(s, s->d_hash, 1);
    if (rc) return rc;
    unsigned long long H = 0;
    CU(cudaMemcpyAsync(&H, s->d_hash, 8, cudaMemcpyDeviceToHost, s->stream));
    std::vector<unsigned long long> c, hist;
    if ((rc = gather_stats(s, c, hist))) return rc;
    uint64_t h = H;
    const uint32_t nb = s->cfg.hist_bins;
    for (uint32_t i = 0; i < NCOUNTERS; ++i) h += hterm(D_CNT, i, TupleHash(1).add(c[i]).h);
    for (uint32_t k = 0; k < 3; ++k)
        for (uint32_t b = 0; b < nb; ++b)
            if (hist[(size_t)k * nb + b])
                h += hterm(D_HIST, ((uint64_t)k << 32) + b, TupleHash(1).add(hist[(size_t)k * nb + b]).h);
    h += hterm(D_CYCLE, 0, TupleHash(1).add(s->t).h);
    *out = h;
    return NOC_OK;
}

extern "C" int noc_sim_get_info(noc_sim *s, noc_sim_info *o)
{
    if (!s || !o) return fail(NOC_EINVAL, "null argument");
    memset(o, 0, sizeof *o);
    o->engine = s->engine;
    if (s->engine == NOC_ENGINE_TILED || s->engine == NOC_ENGINE_TILED4) {
        o->grid = s->set.tile0[s->set.nbands];
        o->block = s->engine == NOC_ENGINE_TILED4 ? 4u * s->t_tpad : s->t_tpad;
        o->reserved[0] = (int32_t)s->D[0].TX;
        o->reserved[1] = (int32_t)s->D[0].TY;
    } else if (s->engine == NOC_ENGINE_PERSIST) {
        o->grid = s->p_grid;
        o->block = PERSIST_BLOCK;
    } else {
        o->grid = (s->D[0].nloc + 255u) / 256u;
        o->block = 256;
    }
    uint32_t nl = 0;
    for (int k = 0; k < s->nb; ++k) nl += s->D[k].nloc;
    o->nodes_local = nl;
    o->row0 = s->D[0].row0;
    o->rows = nl / s->D[0].W;
    o->device_bytes = s->bytes;
    o->loc_bytes = s->loc_bytes;
    o->kernel_launches = s->launches;
    o->cluster = s->set.cluster;
    o->cycles_run = s->t;
    o->sm_count = s->sm_count;
    o->reserved[2] = s->P;
    return NOC_OK;
}
