// runtime.cu -- host runtime behind include/noc_sim.h: configuration
// validation, structure-of-arrays allocation in HBM, engine selection and
// launch control, drain, statistics and the canonical state hash.
#include "../../include/noc_sim.h"
#include "kernels.h"

#include <algorithm>
#include <cstdio>
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

struct noc_sim {
    noc_sim_config cfg;
    Dev D;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    uint64_t t = 0;               // next cycle to simulate
    uint32_t engine = NOC_ENGINE_STEP;
    // persistent engine
    uint32_t *progress = nullptr;
    uint32_t pbase = 0;
    uint32_t p_grid = 0, p_npc = 0, p_smem_hist = 0;
    // tiled engine
    uint32_t t_grid = 0, t_tpad = 0, t_smem_hist = 0;
    // scratch
    uint32_t *d_scratch = nullptr;          // [DRAIN_CHUNK + 2]
    unsigned long long *d_hash = nullptr;
    std::vector<void *> allocs;
    uint64_t bytes = 0, loc_bytes = 0;
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
    e = cudaMemset(q, 0, b);
    if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("cudaMemset: ") + cudaGetErrorString(e));
    s->allocs.push_back(q);
    s->bytes += b;
    *p = (T *)q;
    return NOC_OK;
}

static int validate(const noc_sim_config *c)
{
    if (!c) return fail(NOC_EINVAL, "null config");
    const uint64_t N = (uint64_t)c->mesh_w * c->mesh_h;
    if (c->mesh_w < 2 || c->mesh_h < 2 || c->mesh_w > 2048 || c->mesh_h > 2048 || N > (1u << 21) - 1u)
        return fail(NOC_EINVAL, "mesh must be 2..2048 per side and at most 2^21-1 nodes (R9, R32)");
    if (c->mode > 1 || c->prio > 1) return fail(NOC_EINVAL, "mode/prio out of range");
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
    if (c->world_size > 1) return fail(NOC_EINVAL, "world_size > 1 is not built into this library version");
    if (c->engine > NOC_ENGINE_TILED) return fail(NOC_EINVAL, "unknown engine");
    for (int i = 0; i < 8; ++i)
        if (c->reserved[i]) return fail(NOC_EINVAL, "reserved fields must be 0");
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
    for (void *p : s->allocs) cudaFree(p);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    if (s->stream) cudaStreamDestroy(s->stream);
    cudaSetDevice(cur);
    delete s;
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
    auto bail = [&](int code) { noc_sim_destroy(s); return code; };
    if (cudaSetDevice(s->device) != cudaSuccess) return bail(fail(NOC_ECUDA, "cudaSetDevice failed"));
    cudaDeviceGetAttribute(&s->sm_count, cudaDevAttrMultiProcessorCount, s->device);
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&s->ev0) != cudaSuccess || cudaEventCreate(&s->ev1) != cudaSuccess)
        return bail(fail(NOC_ECUDA, "stream/event creation failed"));

    Dev &D = s->D;
    memset(&D, 0, sizeof D);
    D.W = cfg->mesh_w;
    D.H = cfg->mesh_h;
    D.N = D.W * D.H;
    D.row0 = 0;
    D.rows = D.H;
    D.n0 = 0;
    D.nloc = D.N;
    D.mode = cfg->mode;
    D.prio = cfg->prio;
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
    const size_t n = D.nloc;

    for (int b = 0; b < 2; ++b) {
        if ((rc = dalloc(s, &D.flit[b], 4 * n))) return bail(rc);
        if ((rc = dalloc(s, &D.flag[b], n))) return bail(rc);
    }
    if ((rc = dalloc(s, &D.fifo_ctl, n))) return bail(rc);
    if ((rc = dalloc(s, &D.fifo_pkt, n * D.qcap))) return bail(rc);
    if ((rc = dalloc(s, &D.cnt, NCOUNTERS))) return bail(rc);
    if ((rc = dalloc(s, &D.hist, 3 * (size_t)D.nb))) return bail(rc);
    if ((rc = dalloc(s, &D.err, 1))) return bail(rc);
    if (cfg->mode == NOC_MODE_LSPD) {
        if ((rc = dalloc(s, &D.core_hot, n))) return bail(rc);
        if ((rc = dalloc(s, &D.core_cold, n))) return bail(rc);
        if ((rc = dalloc(s, &D.l2, n * D.sets * D.ways))) return bail(rc);
        uint64_t b0 = s->bytes;
        if ((rc = dalloc(s, &D.loc, (size_t)D.tpn * n))) return bail(rc);
        s->loc_bytes = s->bytes - b0;
    }
    // script: per node, ordered by (cycle, input order)
    {
        std::vector<uint32_t> off(n + 1, 0);
        std::vector<uint4> ev;
        if (cfg->n_script) {
            std::vector<uint64_t> idx(cfg->n_script);
            for (uint64_t i = 0; i < cfg->n_script; ++i) idx[i] = i;
            std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
                const noc_sim_event &x = cfg->script[a], &y = cfg->script[b];
                if (x.node != y.node) return x.node < y.node;
                return x.cycle < y.cycle;
            });
            ev.resize(cfg->n_script);
            for (uint64_t i = 0; i < cfg->n_script; ++i) {
                const noc_sim_event &x = cfg->script[idx[i]];
                ev[i] = make_uint4((uint32_t)x.cycle, (uint32_t)(x.cycle >> 32), x.value, 0u);
                off[x.node + 1] += 1;
            }
            for (size_t i = 0; i < n; ++i) off[i + 1] += off[i];
            D.has_script = 1;
        }
        uint4 *dev_ev = nullptr;
        uint32_t *dev_off = nullptr;
        if ((rc = dalloc(s, &dev_ev, ev.size()))) return bail(rc);
        if ((rc = dalloc(s, &dev_off, n + 1))) return bail(rc);
        if ((rc = dalloc(s, &D.script_pos, n))) return bail(rc);
        if (!ev.empty() && cudaMemcpy(dev_ev, ev.data(), ev.size() * sizeof(uint4), cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(fail(NOC_ECUDA, "script upload failed"));
        if (cudaMemcpy(dev_off, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(fail(NOC_ECUDA, "script upload failed"));
        D.script = dev_ev;
        D.script_off = dev_off;
    }
    if ((rc = dalloc(s, &s->d_scratch, DRAIN_CHUNK + 2))) return bail(rc);
    if ((rc = dalloc(s, &s->d_hash, 1))) return bail(rc);

    // engine: TILED when every tile fits one CTA of <= TILE_MAX_THREADS
    // threads on its own SM, else PERSIST (DESIGN 6)
    s->engine = cfg->engine;
    if (s->engine == NOC_ENGINE_AUTO || s->engine == NOC_ENGINE_TILED) {
        Dev trial = D;
        uint32_t g = 0, tp = 0, sh = 0;
        cudaError_t ce = tiled_configure(trial, s->device, &g, &tp, &sh);
        if (ce == cudaSuccess) {
            s->engine = NOC_ENGINE_TILED;
            D.TX = trial.TX;
            D.TY = trial.TY;
            s->t_grid = g;
            s->t_tpad = tp;
            s->t_smem_hist = sh;
        } else if (s->engine == NOC_ENGINE_TILED) {
            cudaGetLastError();
            return bail(fail(NOC_EINVAL, std::string("TILED engine does not fit this mesh: ") + cudaGetErrorString(ce)));
        } else {
            cudaGetLastError();
            s->engine = NOC_ENGINE_PERSIST;
        }
    }
    if (s->engine == NOC_ENGINE_TILED) {
        if ((rc = dalloc(s, &D.ll, (size_t)32u * n))) return bail(rc);
        if (launch_ll_reset(D, 0, s->stream) != cudaSuccess) return bail(fail(NOC_ECUDA, "ll reset failed"));
    }
    if (s->engine == NOC_ENGINE_PERSIST) {
        cudaError_t ce = persist_configure(D, s->device, &s->p_grid, &s->p_npc, &s->p_smem_hist);
        if (ce != cudaSuccess) return bail(fail(NOC_ECUDA, std::string("persist_configure: ") + cudaGetErrorString(ce)));
        if ((rc = dalloc(s, &s->progress, s->p_grid))) return bail(rc);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(NOC_ECUDA, "init sync failed"));
    *out = s;
    return NOC_OK;
}

static int check_err(noc_sim *s)
{
    uint32_t err = 0;
    CU(cudaMemcpyAsync(&err, s->D.err, 4, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    if (err) {
        s->poisoned = 1;
        if (err & 0x80000000u) return fail(NOC_ECUDA, "persistent kernel: neighbour wait timed out");
        if (err & (ERR_AGE | ERR_PEND)) return fail(NOC_EOVERFLOW, "field width exceeded (flit age > 65535 or pend > 1023)");
        return fail(NOC_ECUDA, "model assertion failed on device (protocol / EV holder)");
    }
    return NOC_OK;
}

// Advance n cycles with the handle's engine; activity (device, may be null)
// receives per-cycle busy-CTA counts when draining (n <= DRAIN_CHUNK).
static int advance(noc_sim *s, uint64_t n, uint32_t *activity)
{
    cudaError_t e;
    if (s->engine == NOC_ENGINE_TILED) {
        uint64_t done = 0;
        while (done < n) {
            uint32_t k = (uint32_t)std::min<uint64_t>(n - done, PERSIST_CHUNK);
            e = launch_tiled(s->D, s->t + done, k, s->t_grid, s->t_tpad, s->t_smem_hist,
                             activity ? activity + done : nullptr, s->stream);
            if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("tiled launch: ") + cudaGetErrorString(e));
            done += k;
            s->launches += 1;
        }
    } else if (s->engine == NOC_ENGINE_PERSIST) {
        uint64_t done = 0;
        while (done < n) {
            uint32_t k = (uint32_t)std::min<uint64_t>(n - done, PERSIST_CHUNK);
            e = launch_persist(s->D, s->t + done, k, s->progress, s->pbase, s->p_grid, s->p_npc, s->p_smem_hist,
                               activity ? activity + done : nullptr, s->stream);
            if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("persistent launch: ") + cudaGetErrorString(e));
            s->pbase += k;
            done += k;
            s->launches += 1;
        }
    } else {
        for (uint64_t i = 0; i < n; ++i) {
            e = launch_step(s->D, s->t + i, activity ? activity + i : nullptr, s->stream);
            if (e != cudaSuccess) return fail(NOC_ECUDA, std::string("step launch: ") + cudaGetErrorString(e));
            s->launches += 1;
        }
    }
    s->t += n;
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
    int q = 0;
    s->D.gen = 0;
    // quiescent already?
    CU(cudaMemsetAsync(s->d_scratch, 0, 4, s->stream));
    CU(launch_busy_count(s->D, s->t, s->d_scratch, s->stream));
    uint32_t busy = 0;
    CU(cudaMemcpyAsync(&busy, s->d_scratch, 4, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    q = busy == 0;
    std::vector<uint32_t> act(DRAIN_CHUNK);
    while (!q && k < max_cycles) {
        uint32_t chunk = (uint32_t)std::min<uint64_t>(DRAIN_CHUNK, max_cycles - k);
        CU(cudaMemsetAsync(s->d_scratch, 0, sizeof(uint32_t) * chunk, s->stream));
        int rc = advance(s, chunk, s->d_scratch);
        if (rc) { s->D.gen = 1; return rc; }
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
            if (s->engine == NOC_ENGINE_TILED) CU(launch_ll_reset(s->D, s->t, s->stream));
        } else {
            k += chunk;
        }
    }
    s->D.gen = 1;
    if (used) *used = k;
    if (drained) *drained = q;
    return check_err(s);
}

static const int NC_NAMED = 23;

extern "C" int noc_sim_stats(noc_sim *s, noc_sim_counters *out, uint64_t *hl, uint64_t *hd, uint64_t *ha, uint32_t nbins)
{
    if (!s) return fail(NOC_EINVAL, "null handle");
    if ((hl || hd || ha) && nbins != s->D.nb) return fail(NOC_EINVAL, "nbins != hist_bins");
    CU(cudaSetDevice(s->device));
    if (out) {
        unsigned long long c[NCOUNTERS];
        CU(cudaMemcpyAsync(c, s->D.cnt, sizeof c, cudaMemcpyDeviceToHost, s->stream));
        CU(cudaStreamSynchronize(s->stream));
        int64_t *dst = &out->generated;
        out->cycle = (int64_t)s->t;
        for (int i = 0; i < NC_NAMED; ++i) dst[i] = (int64_t)c[i];
        for (int k = 0; k < 8; ++k) out->drops[k] = (int64_t)c[C_DROPS + k];
    }
    uint64_t *hs[3] = {hl, hd, ha};
    for (int h = 0; h < 3; ++h)
        if (hs[h]) CU(cudaMemcpyAsync(hs[h], s->D.hist + (size_t)h * s->D.nb, sizeof(uint64_t) * s->D.nb,
                                      cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    return NOC_OK;
}

extern "C" int noc_sim_state_hash(noc_sim *s, uint64_t *out)
{
    if (!s || !out) return fail(NOC_EINVAL, "null argument");
    CU(cudaSetDevice(s->device));
    CU(cudaMemsetAsync(s->d_hash, 0, 8, s->stream));
    CU(launch_hash(s->D, s->t, s->d_hash, s->stream));
    unsigned long long H = 0;
    CU(cudaMemcpyAsync(&H, s->d_hash, 8, cudaMemcpyDeviceToHost, s->stream));
    unsigned long long c[NCOUNTERS];
    CU(cudaMemcpyAsync(c, s->D.cnt, sizeof c, cudaMemcpyDeviceToHost, s->stream));
    std::vector<unsigned long long> hist(3 * (size_t)s->D.nb);
    CU(cudaMemcpyAsync(hist.data(), s->D.hist, hist.size() * 8, cudaMemcpyDeviceToHost, s->stream));
    CU(cudaStreamSynchronize(s->stream));
    uint64_t h = H;
    for (uint32_t i = 0; i < NCOUNTERS; ++i) h += hterm(D_CNT, i, TupleHash(1).add(c[i]).h);
    for (uint32_t k = 0; k < 3; ++k)
        for (uint32_t b = 0; b < s->D.nb; ++b)
            if (hist[(size_t)k * s->D.nb + b])
                h += hterm(D_HIST, ((uint64_t)k << 32) + b, TupleHash(1).add(hist[(size_t)k * s->D.nb + b]).h);
    h += hterm(D_CYCLE, 0, TupleHash(1).add(s->t).h);
    *out = h;
    return NOC_OK;
}

extern "C" int noc_sim_get_info(noc_sim *s, noc_sim_info *o)
{
    if (!s || !o) return fail(NOC_EINVAL, "null argument");
    memset(o, 0, sizeof *o);
    o->engine = s->engine;
    if (s->engine == NOC_ENGINE_TILED) {
        o->grid = s->t_grid;
        o->block = s->t_tpad;
        o->reserved[0] = (int32_t)s->D.TX;
        o->reserved[1] = (int32_t)s->D.TY;
    } else if (s->engine == NOC_ENGINE_PERSIST) {
        o->grid = s->p_grid;
        o->block = PERSIST_BLOCK;
    } else {
        o->grid = (s->D.nloc + 255u) / 256u;
        o->block = 256;
    }
    o->nodes_local = s->D.nloc;
    o->row0 = s->D.row0;
    o->rows = s->D.rows;
    o->device_bytes = s->bytes;
    o->loc_bytes = s->loc_bytes;
    o->kernel_launches = s->launches;
    o->cycles_run = s->t;
    o->sm_count = s->sm_count;
    return NOC_OK;
}
