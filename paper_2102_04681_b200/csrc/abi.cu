// abi.cu — network object, memory plan, CUDA-graph step loop and the C ABI of
// include/spice.h.  Host-side runtime of the B200 Spice hot path.
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <chrono>
#include <thread>
#include <vector>

#include "spice.h"
#include "spice_internal.cuh"
#include "spice_launch.h"

using namespace spice;

namespace {

thread_local std::string g_err;

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void *h = nullptr;
    const char *env = getenv("SPICE_NCCL_LIB");
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllGather && api.AllReduce &&
             api.CommDestroy && api.GetErrorString;
    return api;
}

// gathered bitmaps -> ascending global IDs (host side of the exchange, Fig. 2 union)
void decode_into(const uint32_t *bm, uint32_t G, uint32_t W, uint32_t S, std::vector<uint32_t> &L) {
    L.clear();
    for (uint32_t r = 0; r < G; ++r)
        for (uint32_t w = 0; w < W; ++w) {
            uint32_t bits = bm[(uint64_t)r * W + w];
            while (bits) {
                const uint32_t b = __builtin_ctz(bits);
                bits &= bits - 1;
                L.push_back((uint32_t)local_to_global((uint64_t)w * 32 + b, r, G, S));
            }
        }
    if (G > 1) std::sort(L.begin(), L.end());
}

// Decode nsteps consecutive steps of gathered bitmaps (words per step each) into per[q];
// independent steps are decoded on up to 8 host threads (the host side of a streaming
// read-out would otherwise be slower than the GPU steps it reads, at 1e6+ neurons).
uint64_t decode_steps(const uint32_t *bm, uint64_t nsteps, uint64_t words, uint32_t G, uint32_t W,
                      uint32_t S, std::vector<std::vector<uint32_t>> &per) {
    per.resize(nsteps);
    const uint64_t work = nsteps * words;
    unsigned nt = std::thread::hardware_concurrency();
    nt = std::max(1u, std::min<unsigned>(nt ? nt : 1, 8));
    if (work < (1u << 16) || nsteps < 2) nt = 1;
    nt = (unsigned)std::min<uint64_t>(nt, nsteps);
    auto body = [&](unsigned id) {
        for (uint64_t q = id; q < nsteps; q += nt) decode_into(bm + q * words, G, W, S, per[q]);
    };
    if (nt == 1) body(0);
    else {
        std::vector<std::thread> th;
        for (unsigned id = 1; id < nt; ++id) th.emplace_back(body, id);
        body(0);
        for (auto &x : th) x.join();
    }
    uint64_t tot = 0;
    for (auto &L : per) tot += L.size();
    return tot;
}

uint64_t owned_count(uint64_t n, uint32_t g, uint32_t G, uint32_t S) {
    const uint64_t full = n / ((uint64_t)S * G);           // complete rounds of G slices
    uint64_t c = full * S;
    const uint64_t rem = n - full * S * G;                 // neurons in the last round
    const uint64_t start = (uint64_t)g * S;
    if (rem > start) c += std::min<uint64_t>(S, rem - start);
    return c;
}

uint64_t prob_threshold(double p) {
    if (p <= 0.0) return 0;
    if (p >= 1.0) return 1ull << 32;
    return (uint64_t)std::floor(p * 4294967296.0);
}

// Poisson inversion table T_k = floor(2^32 F(k)) (reading R12; same formula as the
// oracle, written independently): p0 = exp(-lambda), p_k = p_{k-1} lambda / k.
std::vector<uint64_t> poisson_table(double lambda) {
    std::vector<uint64_t> t;
    double pk = std::exp(-lambda), F = pk;
    for (uint32_t k = 0; k < 4096; ++k) {
        const double T = std::floor(F * 4294967296.0);
        if (T >= 4294967295.0) { t.push_back(1ull << 32); return t; }
        t.push_back((uint64_t)T);
        pk = pk * lambda / (double)(k + 1);
        F = F + pk;
    }
    return {};
}

}  // namespace

struct spice_net {
    // configuration
    uint32_t model = 0, N = 0, n_exc = 0, delay = 0, D = 0, rank = 0, G = 1, S = 32, flags = 0;
    uint32_t R = 1;   // record steps
    double dt = 0.1, activity = 0;
    uint64_t seed = 0;
    std::vector<double> prm;
    std::vector<spice_rule> rules;
    int device = 0, n_sm = 148;
    cudaStream_t stream = nullptr;      // execution stream (library-owned or the caller's)
    bool own_stream = true;
    cudaStream_t cap_stream = nullptr;  // library-owned capture stream (graphs are captured here)
    void *(*dev_alloc)(size_t, void *) = nullptr;   // caller's device allocator (or cudaMalloc)
    void (*dev_free)(void *, void *) = nullptr;
    void *alloc_ctx = nullptr;
    bool poisoned = false;
    bool external = false;
    // PEER exchange: receive window (cudaMalloc: IPC-exportable), the G windows' addresses
    // (device array), the mappings opened here, and the device error flag of the wait kernel
    bool peer = false, connected = true;
    uint32_t *win = nullptr;
    uint32_t **peers_dev = nullptr;
    std::vector<void *> opened;
    uint32_t *xerr = nullptr;
    uint32_t *gbar = nullptr;           // persistent step kernel: grid-barrier slots + timeout flag
    // geometry
    uint64_t n_own = 0, n_own_max = 0;
    uint32_t W = 0, TW = 32, NT = 1, C = 1, TWs = 32;
    uint64_t ring_stride = 0;
    uint64_t nnz = 0;        // stored entries (incl. padding sentinels)
    uint64_t n_syn = 0;      // synapses (owned targets)
    bool pad8 = false;       // segments padded to 8-entry windows (window-stream delivery)
    uint32_t eshift = 0;     // entries hold (tile offset << eshift); 2 when padded
    uint32_t *deg = nullptr; // pad8: true out-degree of every source on this rank
    bool mixed_delays = false;   // synapses of more than one delay (reading R19)
    bool procedural = false;     // SPICE_FLAG_PROCEDURAL: rows regenerated per spike, none stored
    uint8_t *dly = nullptr;      // per-entry delay (mixed delays only), aligned with ent
    double mean_seg = 0;
    double gen_ms = 0, create_ms = 0;   // setup: generator kernels (device), create (host wall)
    bool small = false;                 // one-CTA persistent step kernel (k_small)
    uint32_t *hbm = nullptr;            // pinned host staging of recorded bitmaps (read_spikes)
    uint64_t hbm_words = 0;
    struct Slot {                       // double-buffered read-out (spikes_prefetch/collect)
        uint32_t *h = nullptr;          // pinned: the chunk's packed IDs
        uint64_t words = 0, t_begin = 0, t_end = 0;
        uint32_t *d_ids = nullptr, *d_cnt = nullptr, *h_cnt = nullptr;   // device IDs / counts, pinned counts
        uint64_t dcap = 0, ccap = 0, copied = 0, guess = 0;
        bool full = false, compact = false, guarded = false;
        cudaEvent_t done = nullptr, ready = nullptr;
    } slot[2];
    cudaStream_t xfer = nullptr;        // read-out: copies that must not queue behind later steps
    std::vector<std::vector<uint32_t>> hdec;   // decoded per-step lists (reused)
    uint32_t NR = 1, RS = 32;    // spike-list regions
    uint32_t prod_words = 0;     // synth fast path: producer-warp shared memory (words)
    unsigned long long *ptimes = nullptr;   // SPICE_PHASES diagnostics
    bool fused = true, global_atomics = false;
    // device memory
    std::vector<void *> allocs;
    uint64_t device_bytes = 0;
    uint64_t *row_ptr = nullptr;
    uint32_t *bnd = nullptr;
    uint16_t *ent_alloc = nullptr, *ent = nullptr;
    float *v = nullptr, *ge = nullptr, *gi = nullptr;
    uint32_t *ref = nullptr, *acc = nullptr, *ring = nullptr;
    uint32_t *sl_ids = nullptr, *sl_counts = nullptr;
    uint64_t *sl_rows = nullptr;
    uint64_t *desc = nullptr;
    uint32_t *dcount = nullptr;
    uint32_t *record = nullptr, *sendbuf = nullptr, *gather = nullptr;
    unsigned long long *fired_cta = nullptr, *delivered_cta = nullptr;
    uint64_t *t0 = nullptr;
    uint32_t *force_bits = nullptr;
    uint64_t *force_ctl = nullptr;
    uint64_t *ptab = nullptr;
    // Brunel+
    float *w = nullptr;
    uint32_t *pre_ts = nullptr, *post = nullptr, *post_mask = nullptr;   // event-driven STDP state
    float *pre_c = nullptr, *tab_p = nullptr, *tab_m = nullptr;
    std::vector<float> htab_p, htab_m;     // host copies (trace read-out)
    long long *pring = nullptr;
    ModelConst mc{};
    SimArgs args{};
    // host progress
    uint64_t t_host = 0;
    // step graphs: graphs[k] runs 2^k steps (k < kGraphLevels)
    static constexpr uint32_t kGraphLevels = 9;
    cudaGraphExec_t graphs[kGraphLevels] = {};
    // nccl
    ncclComm_t comm = nullptr;
    cudaEvent_t ev = nullptr;
};

namespace {

spice_status fail(spice_net *n, spice_status st, const char *fmt, ...) {
    char buf[768];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    char head[96];
    snprintf(head, sizeof head, "spice rank %u step %llu: ", n ? n->rank : 0u,
             (unsigned long long)(n ? n->t_host : 0ull));
    g_err = std::string(head) + buf;
    if (n && (st == SPICE_ECUDA || st == SPICE_ENCCL)) n->poisoned = true;
    return st;
}

#define CU(net, x)                                                                           \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess)                                                               \
            return fail(net, SPICE_ECUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                 \
    } while (0)

#define CHECK_NET(net)                                                                       \
    do {                                                                                     \
        if (!(net)) return fail(nullptr, SPICE_EINVAL, "null handle");                       \
        if ((net)->poisoned) return fail(net, SPICE_ESTATE, "handle poisoned by an earlier error"); \
    } while (0)

spice_status dalloc(spice_net *n, void **p, size_t bytes, const char *what) {
    *p = nullptr;
    if (n->dev_alloc) {
        *p = n->dev_alloc(bytes ? bytes : 16, n->alloc_ctx);
        if (!*p) return fail(n, SPICE_ENOMEM, "dev_alloc of %zu bytes for %s failed", bytes, what);
    } else {
        cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(n, SPICE_ENOMEM, "cudaMalloc of %zu bytes for %s failed: %s", bytes, what,
                        cudaGetErrorString(e));
        }
    }
    n->allocs.push_back(*p);
    n->device_bytes += bytes;
    return SPICE_OK;
}
void release(spice_net *n, void *p) {
    if (n->dev_free) n->dev_free(p, n->alloc_ctx);
    else if (!n->dev_alloc) cudaFree(p);
}
template <typename T>
spice_status dalloc_t(spice_net *n, T **p, size_t count, const char *what) {
    return dalloc(n, reinterpret_cast<void **>(p), count * sizeof(T), what);
}
void dfree(spice_net *n, void *p) {
    if (!p) return;
    auto it = std::find(n->allocs.begin(), n->allocs.end(), p);
    if (it != n->allocs.end()) n->allocs.erase(it);
    release(n, p);
}

spice_status validate(const spice_config *c) {
    if (!c) return fail(nullptr, SPICE_EINVAL, "null config");
    if (c->abi_version != SPICE_ABI_VERSION) return fail(nullptr, SPICE_EINVAL, "abi_version %u != %u", c->abi_version, SPICE_ABI_VERSION);
    if (c->model < SPICE_VOGELS || c->model > SPICE_SYNTH)
        return fail(nullptr, SPICE_EINVAL, "model %u not supported by this build", c->model);
    if (c->n_neurons == 0) return fail(nullptr, SPICE_EINVAL, "n_neurons must be > 0");
    if (c->n_exc > c->n_neurons) return fail(nullptr, SPICE_EINVAL, "n_exc > n_neurons");
    if (c->delay_steps == 0) return fail(nullptr, SPICE_EINVAL, "delay_steps must be >= 1");
    if (!(c->dt_ms > 0)) return fail(nullptr, SPICE_EINVAL, "dt_ms must be > 0");
    if (c->world_size == 0 || c->rank >= c->world_size) return fail(nullptr, SPICE_EINVAL, "rank %u / world_size %u", c->rank, c->world_size);
    if (c->slice_width % 32) return fail(nullptr, SPICE_EINVAL, "slice_width must be a multiple of 32");
    if (c->record_steps == 0) return fail(nullptr, SPICE_EINVAL, "record_steps must be >= 1");
    if (c->tile_width && (c->tile_width % 32 || c->tile_width > kMaxTileWidth))
        return fail(nullptr, SPICE_EINVAL, "tile_width must be a multiple of 32 and <= %u", kMaxTileWidth);
    const uint32_t need = c->model == SPICE_VOGELS ? 17 : c->model == SPICE_BRUNEL ? 10
                        : c->model == SPICE_BRUNEL_PLUS ? 16 : 0;
    if (c->model == SPICE_BRUNEL_PLUS && c->ctas_per_tile > 1)
        return fail(nullptr, SPICE_EINVAL, "Brunel+ needs one CTA per tile (ctas_per_tile = 1)");
    uint32_t nplastic = 0;
    if (c->n_model_params < need || (need && !c->model_params))
        return fail(nullptr, SPICE_EINVAL, "model %u needs %u parameters, got %u", c->model, need, c->n_model_params);
    if (c->model == SPICE_SYNTH && !(c->activity >= 0 && c->activity <= 1))
        return fail(nullptr, SPICE_EINVAL, "activity outside [0,1]");
    if (c->n_rules && !c->rules) return fail(nullptr, SPICE_EINVAL, "rules is NULL");
    if (c->n_rules > 16) return fail(nullptr, SPICE_EINVAL, "at most 16 rules");
    for (uint32_t r = 0; r < c->n_rules; ++r) {
        const spice_rule &R = c->rules[r];
        if (R.src_begin > R.src_end || R.src_end > c->n_neurons || R.dst_begin > R.dst_end || R.dst_end > c->n_neurons)
            return fail(nullptr, SPICE_EINVAL, "rule %u: ranges outside [0, N)", r);
        if (R.kind == SPICE_FIXED_PROB && !(R.p >= 0 && R.p <= 1)) return fail(nullptr, SPICE_EINVAL, "rule %u: p outside [0,1]", r);
        if (R.kind != SPICE_FIXED_PROB && R.kind != SPICE_FIXED_INDEGREE) return fail(nullptr, SPICE_EINVAL, "rule %u: unknown kind", r);
        if (R.plastic && c->model != SPICE_BRUNEL_PLUS) return fail(nullptr, SPICE_EINVAL, "rule %u: plastic synapses need model BRUNEL_PLUS", r);
        if (R.plastic && ++nplastic > kMaxPlasticRules) return fail(nullptr, SPICE_EINVAL, "at most %d plastic rules", kMaxPlasticRules);
        if (R.delay_min && (R.delay_max > 255 || (R.delay_max && R.delay_max < R.delay_min)))
            return fail(nullptr, SPICE_EINVAL, "rule %u: delay range [%u, %u] (1 <= min <= max <= 255)", r, R.delay_min, R.delay_max);
        for (uint32_t q = 0; q < r; ++q) {
            const spice_rule &Q = c->rules[q];
            const bool src_overlap = R.src_begin < Q.src_end && Q.src_begin < R.src_end;
            const bool dst_overlap = R.dst_begin < Q.dst_end && Q.dst_begin < R.dst_end;
            if (src_overlap && dst_overlap && R.src_begin < R.src_end && R.dst_begin < R.dst_end &&
                Q.src_begin < Q.src_end && Q.dst_begin < Q.dst_end)
                return fail(nullptr, SPICE_EINVAL, "rules %u and %u overlap in both ranges", q, r);
        }
    }
    return SPICE_OK;
}

void build_model_const(spice_net *n) {
    ModelConst &m = n->mc;
    const double *P = n->prm.data();
    const double dt = n->dt;
    if (n->model == SPICE_VOGELS) {
        m.h = (float)(dt / P[0]); m.EL = (float)P[1]; m.Vt = (float)P[2]; m.Vr = (float)P[3];
        m.R = (uint32_t)std::llround(P[4] / dt); m.Ee = (float)P[5]; m.Ei = (float)P[6];
        m.ke = (float)(dt / P[7]); m.ki = (float)(dt / P[8]); m.dge = (float)P[9]; m.dgi = (float)P[10];
    } else if (n->model == SPICE_BRUNEL || n->model == SPICE_BRUNEL_PLUS) {
        m.h = (float)(dt / P[0]); m.EL = (float)P[1]; m.theta = (float)P[2]; m.Vr = (float)P[3];
        m.R = (uint32_t)std::llround(P[4] / dt);
        m.JE = (float)P[5]; m.JI = (float)(-P[6] * P[5]);
        if (n->model == SPICE_BRUNEL_PLUS) {
            m.ap = (float)std::exp(-dt / P[10]); m.am = (float)std::exp(-dt / P[11]);
            m.Ap = (float)P[12]; m.Am = (float)P[13]; m.wmax = (float)P[14];
        }
    } else {
        m.thr_fire = prob_threshold(n->activity);
    }
}

// Enqueue steps k = 0..steps-1 of one replay (each kernel reads t = *t0 + k) on stream s.
spice_status enqueue_steps(spice_net *n, uint32_t steps, cudaStream_t s) {
    const SimArgs &a = n->args;
    if (n->small) {                                        // one launch for the whole chunk
        CU(n, launch_small(a, 0, steps, s));
    } else if (n->G == 1 && n->fused && !n->global_atomics) {
        CU(n, launch_update(a, 0, s));
        if (a.persist) CU(n, launch_run(a, 0, steps - 1, s));          // one persistent launch
        else for (uint32_t k = 0; k + 1 < steps; ++k) CU(n, launch_fused(a, k, s));   // deliver(k)+update(k+1)
        CU(n, launch_deliver(a, steps - 1, false, n->n_sm, s));
    } else {
        // G > 1: the exchange of step k's bitmaps (NCCL all-gather, or the PEER flags wait:
        // the bitmap words were stored into every window by the update) and bitmap->list
        const bool peer = n->peer;
        auto xchg = [&](uint32_t k) -> spice_status {
            if (peer) CU(n, launch_peer_wait(a, k, s));
            else {
                ncclResult_t r = nccl().AllGather(n->sendbuf, n->gather, n->W, ncclUint32, n->comm, s);
                if (r != ncclSuccess) return fail(n, SPICE_ENCCL, "ncclAllGather: %s", nccl().GetErrorString(r));
            }
            CU(n, launch_bitmap_to_list(a, k, s));
            return SPICE_OK;
        };
        auto publish = [&](uint32_t k) -> spice_status {   // after the update of step k (PEER)
            if (peer) CU(n, launch_peer_signal(a, k, s));
            return SPICE_OK;
        };
        spice_status st;
        if (n->G > 1 && n->fused && !n->global_atomics) {
            // padded layout: update(0), then per step exchange(t) -> bitmap->list + descriptors(t)
            // -> fused deliver(t)+update(t+1); the last step delivers unfused
            CU(n, launch_update(a, 0, s));
            if ((st = publish(0))) return st;
            for (uint32_t k = 0; k < steps; ++k) {
                if ((st = xchg(k))) return st;
                if (k + 1 < steps) {
                    CU(n, launch_fused(a, k, s));
                    if ((st = publish(k + 1))) return st;
                } else {
                    CU(n, launch_deliver(a, k, false, n->n_sm, s));
                }
            }
        } else {
            for (uint32_t k = 0; k < steps; ++k) {
                CU(n, launch_update(a, k, s));
                if (n->G > 1) {
                    if ((st = publish(k))) return st;
                    if ((st = xchg(k))) return st;
                }
                CU(n, launch_deliver(a, k, n->global_atomics, n->n_sm, s));
            }
        }
    }
    CU(n, launch_advance(n->t0, steps, s, n->gbar));
    return SPICE_OK;
}

spice_status capture_graph(spice_net *n, uint32_t steps, cudaGraphExec_t *out) {
    cudaGraph_t g = nullptr;
    CU(n, cudaStreamBeginCapture(n->cap_stream, cudaStreamCaptureModeThreadLocal));
    spice_status st = enqueue_steps(n, steps, n->cap_stream);
    cudaError_t e2 = cudaStreamEndCapture(n->cap_stream, &g);
    if (st != SPICE_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (e2 != cudaSuccess) return fail(n, SPICE_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(e2));
    cudaError_t err = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (err != cudaSuccess) return fail(n, SPICE_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(err));
    return SPICE_OK;
}

void destroy(spice_net *n) {
    if (!n) return;
    if (n->stream) cudaStreamSynchronize(n->stream);
    if (n->xfer) cudaStreamSynchronize(n->xfer);
    for (cudaGraphExec_t &g : n->graphs) if (g) cudaGraphExecDestroy(g);
    for (void *p : n->opened) cudaIpcCloseMemHandle(p);
    if (n->win) cudaFree(n->win);
    if (n->comm) nccl().CommDestroy(n->comm);
    for (void *p : n->allocs) release(n, p);
    n->allocs.clear();
    if (n->ev) cudaEventDestroy(n->ev);
    if (n->hbm) cudaFreeHost(n->hbm);
    for (auto &sl : n->slot) {
        if (sl.h) cudaFreeHost(sl.h);
        if (sl.h_cnt) cudaFreeHost(sl.h_cnt);
        if (sl.done) cudaEventDestroy(sl.done);
        if (sl.ready) cudaEventDestroy(sl.ready);
    }
    if (n->xfer) cudaStreamDestroy(n->xfer);
    if (n->stream && n->own_stream) cudaStreamDestroy(n->stream);
    if (n->cap_stream) cudaStreamDestroy(n->cap_stream);
    delete n;
}

// Exact post-generation check that packed 16-bit receptor counts cannot overflow:
// the number of excitatory (inhibitory) in-synapses of any owned target is < 65535.
__global__ void indegree_kernel(const uint64_t *row_ptr, const uint32_t *bnd, const uint16_t *ent,
                                uint32_t N, uint32_t NT, uint32_t TW, uint32_t n_exc, uint32_t eshift, uint32_t *deg) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); w < (uint64_t)N * NT; w += nwarps) {
        const uint32_t s = (uint32_t)(w / NT), b = (uint32_t)(w % NT);
        const uint32_t *bp = bnd + (uint64_t)s * (NT + 1) + b;
        const uint64_t st = row_ptr[s] + bp[0];
        const uint32_t len = bp[1] - bp[0];
        const uint32_t q = s >= n_exc ? 65536u : 1u;
        for (uint32_t e = lane; e < len; e += 32) {
            const uint32_t x = (uint32_t)ent[st + e] >> eshift;
            if (x < TW) atomicAdd(&deg[(uint64_t)b * TW + x], q);     // skip padding sentinels
        }
    }
}
__global__ void max_halves_kernel(const uint32_t *deg, uint64_t n, uint32_t *out) {
    uint32_t me = 0, mi = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        me = max(me, deg[i] & 0xFFFFu); mi = max(mi, deg[i] >> 16);
    }
    atomicMax(&out[0], me); atomicMax(&out[1], mi);
}

spice_status generate(spice_net *n) {
    GenGeom g{};
    g.N = n->N; g.n_own = (uint32_t)n->n_own; g.rank = n->rank; g.G = n->G; g.S = n->S;
    g.TW = n->TW; g.NT = n->NT; g.key0 = (uint32_t)n->seed; g.key1 = (uint32_t)(n->seed >> 32);
    g.pad8 = n->pad8 ? 1u : 0u;
    g.eshift = n->eshift;
    const uint64_t nb = (uint64_t)n->N * (n->NT + 1);
    uint32_t *cursor = nullptr;
    spice_status st;
    if ((st = dalloc_t(n, &n->row_ptr, (size_t)n->N + 1, "row_ptr"))) return st;
    // generator device time (P:443 quotes the setup kernel's synapses per ms): count,
    // scan, fill, pad and sort kernels, excluding allocations and host round trips
    cudaEvent_t eg[4] = {};
    for (cudaEvent_t &e : eg) cudaEventCreate(&e);
    struct EvFree { cudaEvent_t *e; ~EvFree() { for (int q = 0; q < 4; ++q) if (e[q]) cudaEventDestroy(e[q]); } } evf{eg};
    if ((st = dalloc_t(n, &n->bnd, nb + 4, "segment bounds"))) return st;   // + 16-byte tail pad
    CU(n, cudaMemsetAsync(n->bnd, 0, (nb + 4) * 4, n->stream));
    // rules in ascending destination order so that per-segment appends stay sorted
    std::vector<uint32_t> order(n->rules.size());
    for (uint32_t r = 0; r < order.size(); ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        return n->rules[a].dst_begin < n->rules[b].dst_begin;
    });
    std::vector<GenRule> gr;
    bool any_indeg = false;
    for (uint32_t r : order) {
        const spice_rule &R = n->rules[r];
        GenRule x{R.src_begin, R.src_end, R.dst_begin, R.dst_end, R.kind, R.k, r, prob_threshold(R.p)};
        gr.push_back(x);
        any_indeg |= R.kind == SPICE_FIXED_INDEGREE && R.k > 0;
    }
    CU(n, cudaEventRecord(eg[0], n->stream));
    for (const GenRule &x : gr) CU(n, gen_count(g, x, n->bnd, n->stream));
    CU(n, cudaEventRecord(eg[1], n->stream));
    uint64_t nnz = 0;
    if (n->pad8 && (st = dalloc_t(n, &n->deg, n->N, "out-degrees"))) return st;
    CU(n, gen_scan(g, n->bnd, n->row_ptr, &nnz, n->deg, n->stream));
    n->nnz = nnz;
    if (n->pad8 && nnz / kWin >= (1ull << 31) - 1)
        return fail(n, SPICE_EINVAL, "%llu synapse windows per rank exceed the 32-bit window index", (unsigned long long)(nnz / kWin));
    if ((st = dalloc_t(n, &n->ent_alloc, (size_t)nnz + 2 * kEntPad, "synapse entries"))) return st;
    n->ent = n->ent_alloc + kEntPad;
    CU(n, cudaMemsetAsync(n->ent_alloc, 0, ((size_t)nnz + 2 * kEntPad) * 2, n->stream));
    if ((st = dalloc_t(n, &cursor, nb, "fill cursors"))) return st;
    CU(n, cudaMemsetAsync(cursor, 0, nb * 4, n->stream));
    CU(n, cudaEventRecord(eg[2], n->stream));
    for (const GenRule &x : gr) CU(n, gen_fill(g, x, n->row_ptr, n->bnd, cursor, n->ent, n->stream));
    if (n->pad8) CU(n, gen_pad_segments(g, n->row_ptr, n->bnd, cursor, n->ent, n->stream));
    if (any_indeg) CU(n, gen_sort_segments(g, n->row_ptr, n->bnd, n->ent, n->stream));   // sentinels (>= TW) sort last
    CU(n, cudaEventRecord(eg[3], n->stream));
    CU(n, cudaStreamSynchronize(n->stream));
    {
        float m01 = 0, m23 = 0;
        cudaEventElapsedTime(&m01, eg[0], eg[1]);
        cudaEventElapsedTime(&m23, eg[2], eg[3]);
        n->gen_ms = (double)m01 + (double)m23;
    }
    if (n->pad8) CU(n, gen_sum_u32(n->deg, n->N, &n->n_syn, n->stream));
    else n->n_syn = nnz;
    dfree(n, cursor);
    n->device_bytes -= nb * 4;
    n->mean_seg = n->N ? (double)nnz / ((double)n->N * n->NT) : 0;
    // receptor packing check: exc counts in bits 0-15 and inh counts in bits 16-31 (two
    // populations), or one 32-bit count (one population: only the synth accumulator reads
    // it as a whole; the other models unpack the low half, so it must stay < 65535 too)
    if (n->n_own && (n->n_exc < n->N || n->model != SPICE_SYNTH)) {
        uint32_t *deg = nullptr, *mx = nullptr;
        if ((st = dalloc_t(n, &deg, n->ring_stride, "in-degree check"))) return st;
        if ((st = dalloc_t(n, &mx, 2, "in-degree max"))) return st;
        CU(n, cudaMemsetAsync(deg, 0, n->ring_stride * 4, n->stream));
        CU(n, cudaMemsetAsync(mx, 0, 8, n->stream));
        indegree_kernel<<<n->n_sm * 8, 256, 0, n->stream>>>(n->row_ptr, n->bnd, n->ent, n->N, n->NT, n->TW, n->n_exc, n->eshift, deg);
        max_halves_kernel<<<n->n_sm * 4, 256, 0, n->stream>>>(deg, n->ring_stride, mx);
        uint32_t h[2] = {0, 0};
        CU(n, cudaMemcpyAsync(h, mx, 8, cudaMemcpyDeviceToHost, n->stream));
        CU(n, cudaStreamSynchronize(n->stream));
        dfree(n, deg); dfree(n, mx);
        n->device_bytes -= n->ring_stride * 4 + 8;
        if (h[0] >= 65535u || h[1] >= 65535u)
            return fail(n, SPICE_EINVAL, "a target has >= 65535 in-synapses of one receptor type; packed counts could overflow");
    }
    return SPICE_OK;
}

}  // namespace

// =========================================================================== ABI
extern "C" {

const char *spice_last_error(void) { return g_err.c_str(); }

uint32_t spice_partition_owner(uint64_t j, uint32_t G, uint32_t S) {
    return (G && S) ? (uint32_t)((j / S) % G) : 0u;
}
uint64_t spice_partition_local_to_global(uint64_t i, uint32_t g, uint32_t G, uint32_t S) {
    return local_to_global(i, g, G, S);
}
uint64_t spice_partition_owned_count(uint64_t n, uint32_t g, uint32_t G, uint32_t S) {
    if (!G || !S || g >= G) return 0;
    return owned_count(n, g, G, S);
}
uint32_t spice_default_slice_width(uint64_t n, uint32_t G) {
    if (G <= 1) return 32;
    const uint64_t s = n / (256ull * G);      // ~256 slices per rank ("hundreds")
    const uint64_t r = (s / 32) * 32;
    return (uint32_t)std::max<uint64_t>(32, std::min<uint64_t>(r, 1u << 20));
}

spice_status spice_decode_bitmaps(const uint32_t *words, uint32_t G, uint32_t W, uint32_t S,
                                  uint32_t *ids, uint64_t cap, uint64_t *total) {
    if (!words || !G || !S || S % 32) return fail(nullptr, SPICE_EINVAL, "bad bitmap geometry");
    std::vector<uint32_t> L;
    decode_into(words, G, W, S, L);
    if (total) *total = L.size();
    if (L.size() > cap || (!ids && !L.empty())) return fail(nullptr, SPICE_ETRUNC, "need %zu ids", L.size());
    if (!L.empty()) memcpy(ids, L.data(), L.size() * 4);
    return SPICE_OK;
}

spice_status spice_nccl_unique_id(void *out128) {
    if (!out128) return fail(nullptr, SPICE_EINVAL, "null output");
    if (!nccl().ok) return fail(nullptr, SPICE_ENCCL, "libnccl.so.2 not found (set SPICE_NCCL_LIB)");
    ncclUniqueId id;
    ncclResult_t r = nccl().GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, SPICE_ENCCL, "ncclGetUniqueId: %s", nccl().GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out128, &id, 128);
    return SPICE_OK;
}

spice_status spice_create_network(const spice_config *c, spice_net **out) {
    if (!out) return fail(nullptr, SPICE_EINVAL, "null output handle");
    *out = nullptr;
    spice_status st = validate(c);
    if (st) return st;
    const auto t_create = std::chrono::steady_clock::now();
    spice_net *n = new spice_net();
    n->model = c->model; n->N = c->n_neurons; n->n_exc = c->n_exc; n->delay = c->delay_steps;
    n->D = c->delay_steps + 1; n->rank = c->rank; n->G = c->world_size;
    // per-synapse delays (reading R19): the fast path keeps the minimum delay of all rules;
    // synapses with longer delays carry a delay byte; the ring spans the longest delay
    {
        uint32_t dmin = ~0u, dmax = 0;
        for (uint32_t r = 0; r < c->n_rules; ++r) {
            const spice_rule &R = c->rules[r];
            if (R.src_begin >= R.src_end || R.dst_begin >= R.dst_end) continue;
            const uint32_t lo = R.delay_min ? R.delay_min : c->delay_steps;
            const uint32_t hi = R.delay_min && R.delay_max > lo ? R.delay_max : lo;
            dmin = std::min(dmin, lo);
            dmax = std::max(dmax, hi);
        }
        if (dmax == 0) dmin = dmax = c->delay_steps;        // no synapses
        n->mixed_delays = dmin != dmax;
        n->delay = dmin;
        n->D = dmax + 1;
    }
    n->S = c->slice_width ? c->slice_width : spice_default_slice_width(c->n_neurons, c->world_size);
    n->flags = c->flags; n->R = c->record_steps; n->dt = c->dt_ms; n->activity = c->activity;
    // Brunel+ reads step t's bitmap while the same launch writes step t + 1's: two slots
    if (n->model == SPICE_BRUNEL_PLUS && n->R < 2) n->R = 2;
    n->seed = c->seed; n->device = c->device;
    n->dev_alloc = c->dev_alloc; n->dev_free = c->dev_free; n->alloc_ctx = c->alloc_ctx;
    n->external = (c->flags & SPICE_FLAG_EXTERNAL_EXCHANGE) != 0;
    n->prm.assign(c->model_params, c->model_params + c->n_model_params);
    n->rules.assign(c->rules, c->rules + c->n_rules);
    auto bail = [&](spice_status s) { destroy(n); return s; };
    if (c->exchange != SPICE_EXCHANGE_NCCL && c->exchange != SPICE_EXCHANGE_PEER)
        return bail(fail(n, SPICE_EINVAL, "unknown exchange %u", c->exchange));
    n->peer = n->G > 1 && !n->external && c->exchange == SPICE_EXCHANGE_PEER;
    if (n->G > 1 && !n->external && !n->peer && !c->nccl_unique_id)
        return bail(fail(n, SPICE_EINVAL, "world_size > 1 needs nccl_unique_id, SPICE_EXCHANGE_PEER or EXTERNAL_EXCHANGE"));
    {
        cudaError_t e = cudaSetDevice(n->device);
        if (e) return bail(fail(n, SPICE_ECUDA, "cudaSetDevice(%d): %s", n->device, cudaGetErrorString(e)));
        cudaDeviceGetAttribute(&n->n_sm, cudaDevAttrMultiProcessorCount, n->device);
        if (c->flags & SPICE_FLAG_USER_STREAM) {
            n->stream = (cudaStream_t)c->stream;
            n->own_stream = false;
        } else {
            e = cudaStreamCreateWithFlags(&n->stream, cudaStreamNonBlocking);
            if (e) return bail(fail(n, SPICE_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e)));
        }
        e = cudaStreamCreateWithFlags(&n->cap_stream, cudaStreamNonBlocking);
        if (e) return bail(fail(n, SPICE_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e)));
        cudaEventCreateWithFlags(&n->ev, cudaEventDisableTiming);
    }
    // ---- partition (a0) ----
    n->n_own = owned_count(n->N, n->rank, n->G, n->S);
    n->n_own_max = owned_count(n->N, 0, n->G, n->S);
    n->W = (uint32_t)((n->n_own_max + 31) / 32);
    // ---- delivery tiles ----
    // padded segments (every (row, tile) segment a whole number of 16-byte windows) for all
    // models but Brunel+ (whose plastic weights are aligned with the unpadded entries).
    // Padded entries are byte offsets up to kMaxPadTile targets per tile, counter indices
    // (one more shift per entry) up to kMaxPadTileWord.
    // C CTAs per tile (ctas_per_tile): the tile is cut into C slices of TWs = TW / C targets
    // (multiples of 32); CTA x updates slice x.  On the fused G = 1 path the C CTAs form a
    // thread-block cluster that reduces the tile's counters through distributed shared memory.
    // (G > 1: the bitmap->list kernel writes the descriptors of the gathered spikes)
    n->procedural = (n->flags & SPICE_FLAG_PROCEDURAL) != 0;
    if (n->procedural) {
        if (n->model == SPICE_BRUNEL_PLUS)
            return bail(fail(n, SPICE_EINVAL, "procedural connectivity needs stored weights for STDP (Brunel+)"));
        if (n->flags & (SPICE_FLAG_GLOBAL_ATOMICS | SPICE_FLAG_EXTERNAL_EXCHANGE))
            return bail(fail(n, SPICE_EINVAL, "procedural connectivity: no global-atomics or external-exchange mode"));
        for (const spice_rule &R : n->rules)
            if (R.kind != SPICE_FIXED_PROB)
                return bail(fail(n, SPICE_EINVAL, "procedural connectivity regenerates FIXED_PROB rules only"));
        if (n->rules.size() > 16) return bail(fail(n, SPICE_EINVAL, "procedural connectivity: at most 16 rules"));
    }
    n->pad8 = n->model != SPICE_BRUNEL_PLUS && !n->procedural;
    // auto: 2-CTA cluster tiles for large padded networks (half the spike x tile visits per
    // CTA; measured -4 % step time on synth 3e9, DESIGN.md delivery log; at G > 1 the rows
    // are G times shorter and the threshold is halved: -26 % on the G = 8 weak-scaling slice,
    // tools/g_proxy.py), else one CTA per tile
    n->C = n->procedural ? 1u : c->ctas_per_tile ? c->ctas_per_tile
         : (n->pad8 && !c->tile_width && n->n_own >= (uint64_t)n->n_sm * (n->G > 1 ? 2048u : 4096u) ? 2u : 1u);
    if (n->C > kMaxCluster) return bail(fail(n, SPICE_EINVAL, "ctas_per_tile %u > %u", n->C, kMaxCluster));
    // small networks: one tile of all owned neurons, one CTA runs whole graph chunks
    // (k_small); auto only, SPICE_NOSMALL=1 disables (A/B)
    {
        const uint64_t tw = (n->n_own + 31) / 32 * 32;
        n->small = n->G == 1 && n->pad8 && !c->tile_width && !c->ctas_per_tile && n->C == 1 &&
                   n->delay == 1 && !n->mixed_delays && (n->model == SPICE_VOGELS || n->model == SPICE_BRUNEL || n->model == SPICE_SYNTH) &&
                   !(n->flags & (SPICE_FLAG_GLOBAL_ATOMICS | SPICE_FLAG_EXTERNAL_EXCHANGE | SPICE_FLAG_UNFUSED)) &&
                   tw >= 32 && tw <= kMaxPadTileWord && small_smem_bytes((uint32_t)tw, n->model) <= 227 * 1024 - 2048 &&
                   !getenv("SPICE_NOSMALL");
    }
    // G > 1 (rows G times shorter: more, shorter segments per spike): 4-CTA cluster tiles,
    // as many as are co-resident (one wave), when a tile's counters fit shared memory --
    // half the spike x tile visits of 2-CTA tiles (tools/g_proxy.py, G = 8 rank slice of
    // the 24e9 network: 53.5 -> 40.9 us/step; G = 4 42.6 -> 36.4; G = 2 35.4 -> 33.2)
    if (!n->small && !c->tile_width && !c->ctas_per_tile && n->pad8 && n->G > 1 && n->C == 2) {
        const uint32_t ncl = max_active_clusters(4);
        if (ncl) {
            const uint64_t tw4 = ((n->n_own + ncl - 1) / ncl + 127) / 128 * 128;
            const size_t smem_cap = 227 * 1024 - 2048 - 6 * 1024;
            if (tw4 <= kMaxPadTileWord && tile_smem_bytes((uint32_t)tw4, 1024, 0) <= smem_cap) {
                n->C = 4;
                n->TW = (uint32_t)tw4;
            }
        }
    }
    if (n->small) {
        n->TW = (uint32_t)((n->n_own + 31) / 32 * 32);
    } else if (n->C == 4 && !c->tile_width && !c->ctas_per_tile && n->G > 1 && n->pad8) {
        // (set above)
    } else if (c->tile_width) {
        const uint32_t q = 32u * n->C;
        n->TW = (c->tile_width + q - 1) / q * q;
    } else {
        const uint64_t want = (uint64_t)std::max(1, n->n_sm / (int)n->C) * n->C;   // one CTA per SM
        uint64_t tws = (n->n_own + want - 1) / want;
        tws = (tws + 31) / 32 * 32;
        const uint64_t cap = (n->pad8 ? (n->C > 1 ? kMaxPadTileWord : kMaxPadTile) : kMaxTileWidth) / (32u * n->C) * 32u;
        n->TW = (uint32_t)(std::min<uint64_t>(std::max<uint64_t>(tws, 32), cap) * n->C);
    }
    n->TWs = n->TW / n->C;
    n->eshift = n->pad8 && n->TW <= kMaxPadTile ? 2u : 0u;
    n->NT = (uint32_t)std::max<uint64_t>(1, (n->n_own + n->TW - 1) / n->TW);

    n->ring_stride = (uint64_t)n->NT * n->TW;
    n->global_atomics = (n->flags & SPICE_FLAG_GLOBAL_ATOMICS) != 0;
    n->fused = !(n->flags & SPICE_FLAG_UNFUSED) && (n->C == 1 || n->pad8);
    // spike-list regions: one per CTA slice (G = 1, written by the slice's update) or one per
    // kB2LWords gathered bitmap words (G > 1, written by bitmap->list)
    if (n->G == 1) { n->NR = n->NT * n->C; n->RS = n->TWs; }
    else {      // about one region per SM: bitmap->list (and its descriptor writes) in one wave
        const uint64_t gw = (uint64_t)n->G * n->W;
        uint64_t bw = (gw + n->n_sm - 1) / n->n_sm;
        bw = std::max<uint64_t>(kB2LWords, (bw + 31) / 32 * 32);
        n->NR = (uint32_t)((gw + bw - 1) / bw);
        n->RS = (uint32_t)(bw * 32);
    }
    if (n->NR > kMaxRegions) return bail(fail(n, SPICE_EINVAL, "%u spike-list regions > %u: use a wider tile_width", n->NR, kMaxRegions));
    const size_t smem_max = 227 * 1024 - 2048 - 6 * 1024;  // dynamic; static shared variables need the rest
    if (n->model == SPICE_SYNTH && n->G == 1 && n->pad8 && tile_smem_bytes(n->TW, n->NR, kSynthProdWordsHost) <= smem_max)
        n->prod_words = kSynthProdWordsHost;
    if (n->pad8 && tile_smem_bytes(n->TW, n->NR, n->prod_words) > smem_max) return bail(fail(n, SPICE_EINVAL, "tile_width %u too wide for shared memory", n->TW));
    if (n->model == SPICE_BRUNEL_PLUS && plastic_smem_bytes(n->TW, n->NR) > smem_max)
        return bail(fail(n, SPICE_EINVAL, "tile_width %u too wide for the Brunel+ tile kernels", n->TW));
    // ---- NCCL communicator ----
    if (n->G > 1 && !n->external && !n->peer) {
        if (!nccl().ok) return bail(fail(n, SPICE_ENCCL, "libnccl.so.2 not found (set SPICE_NCCL_LIB)"));
        ncclUniqueId id;
        memcpy(&id, c->nccl_unique_id, sizeof id);
        ncclResult_t r = nccl().CommInitRank(&n->comm, (int)n->G, id, (int)n->rank);
        if (r != ncclSuccess) return bail(fail(n, SPICE_ENCCL, "ncclCommInitRank: %s", nccl().GetErrorString(r)));
    }
    // ---- connectivity (a0') ----
    if (!n->procedural) {
        if ((st = generate(n))) return bail(st);
    }
    if (n->mixed_delays && !n->procedural) {
        DelayRules dr{};
        for (uint32_t r = 0; r < c->n_rules; ++r) {
            const spice_rule &R = c->rules[r];
            dr.box[dr.n][0] = R.src_begin; dr.box[dr.n][1] = R.src_end;
            dr.box[dr.n][2] = R.dst_begin; dr.box[dr.n][3] = R.dst_end;
            dr.lo[dr.n] = R.delay_min ? R.delay_min : c->delay_steps;
            dr.hi[dr.n] = R.delay_min && R.delay_max > dr.lo[dr.n] ? R.delay_max : dr.lo[dr.n];
            dr.index[dr.n] = r;
            ++dr.n;
        }
        GenGeom gd{};
        gd.N = n->N; gd.n_own = (uint32_t)n->n_own; gd.rank = n->rank; gd.G = n->G; gd.S = n->S;
        gd.TW = n->TW; gd.NT = n->NT; gd.key0 = (uint32_t)n->seed; gd.key1 = (uint32_t)(n->seed >> 32);
        gd.eshift = n->eshift;
        if ((st = dalloc_t(n, &n->dly, (size_t)n->nnz + 16, "synapse delays"))) return bail(st);
        CU(n, cudaMemsetAsync(n->dly, (int)n->delay, (size_t)n->nnz + 16, n->stream));
        CU(n, gen_delays(gd, dr, n->delay, n->row_ptr, n->bnd, n->ent, n->dly, n->stream));
    }
    // ---- state, ring, spike buffers (state padded to NT*TW for 16-byte vector access) ----
    const uint64_t no = n->ring_stride;
    const uint64_t nctas = (uint64_t)n->NT * n->C;
    if ((st = dalloc_t(n, &n->ring, (size_t)n->D * n->ring_stride, "input ring"))) return bail(st);
    // (three copies by step mod 3: sim.cu lslot)
    if ((st = dalloc_t(n, &n->sl_ids, 3ull * n->NR * n->RS, "spike lists"))) return bail(st);
    if ((st = dalloc_t(n, &n->sl_rows, 3ull * n->NR * n->RS, "spike list rows"))) return bail(st);
    if ((st = dalloc_t(n, &n->sl_counts, 3ull * n->NR, "spike list counts"))) return bail(st);

    if ((st = dalloc_t(n, &n->record, (size_t)n->R * n->G * n->W, "spike record"))) return bail(st);
    if ((st = dalloc_t(n, &n->sendbuf, std::max<uint32_t>(n->W, 1), "send bitmap"))) return bail(st);
    if ((st = dalloc_t(n, &n->gather, (size_t)n->G * std::max<uint32_t>(n->W, 1), "gathered bitmaps"))) return bail(st);
    if ((st = dalloc_t(n, &n->fired_cta, nctas, "fired counters"))) return bail(st);
    if ((st = dalloc_t(n, &n->delivered_cta, nctas, "delivered counters"))) return bail(st);
    if ((st = dalloc_t(n, &n->t0, 1, "step counter"))) return bail(st);
    if ((st = dalloc_t(n, &n->force_bits, std::max<uint32_t>(n->W, 1), "force bits"))) return bail(st);
    if ((st = dalloc_t(n, &n->force_ctl, 2, "force control"))) return bail(st);
    if ((st = dalloc_t(n, &n->v, no, "v"))) return bail(st);
    if ((st = dalloc_t(n, &n->ref, no, "ref"))) return bail(st);
    if (n->model == SPICE_VOGELS) {
        if ((st = dalloc_t(n, &n->ge, no, "ge"))) return bail(st);
        if ((st = dalloc_t(n, &n->gi, no, "gi"))) return bail(st);
    }
    if (n->model == SPICE_SYNTH && (st = dalloc_t(n, &n->acc, no, "acc"))) return bail(st);
    cudaStream_t s = n->stream;
    CU(n, cudaMemsetAsync(n->ring, 0, (size_t)n->D * n->ring_stride * 4, s));
    CU(n, cudaMemsetAsync(n->sl_counts, 0, 3ull * n->NR * 4, s));
    CU(n, cudaMemsetAsync(n->sendbuf, 0, std::max<uint32_t>(n->W, 1) * 4, s));   // words past the last tile stay 0
    CU(n, cudaMemsetAsync(n->gather, 0, (size_t)n->G * std::max<uint32_t>(n->W, 1) * 4, s));
    CU(n, cudaMemsetAsync(n->record, 0, (size_t)n->R * n->G * n->W * 4, s));
    CU(n, cudaMemsetAsync(n->fired_cta, 0, nctas * 8, s));
    CU(n, cudaMemsetAsync(n->delivered_cta, 0, nctas * 8, s));
    CU(n, cudaMemsetAsync(n->t0, 0, 8, s));
    CU(n, cudaMemsetAsync(n->force_bits, 0, std::max<uint32_t>(n->W, 1) * 4, s));
    CU(n, cudaMemsetAsync(n->force_ctl, 0xFF, 16, s));
    CU(n, cudaMemsetAsync(n->v, 0, no * 4, s));
    CU(n, cudaMemsetAsync(n->ref, 0, no * 4, s));
    if (n->ge) CU(n, cudaMemsetAsync(n->ge, 0, no * 4, s));
    if (n->gi) CU(n, cudaMemsetAsync(n->gi, 0, no * 4, s));
    if (n->acc) CU(n, cudaMemsetAsync(n->acc, 0, no * 4, s));
    PlasticBoxes pbx{};
    for (const spice_rule &R : n->rules)
        if (R.plastic) { uint32_t *bx = pbx.box[pbx.n++]; bx[0] = R.src_begin; bx[1] = R.src_end; bx[2] = R.dst_begin; bx[3] = R.dst_end; }
    if (n->model == SPICE_BRUNEL_PLUS) {
        GenGeom g2{};
        g2.N = n->N; g2.n_own = (uint32_t)n->n_own; g2.rank = n->rank; g2.G = n->G; g2.S = n->S;
        g2.TW = n->TW; g2.NT = n->NT; g2.key0 = (uint32_t)n->seed; g2.key1 = (uint32_t)(n->seed >> 32);
        if (n->nnz >= (1ull << 32))
            return bail(fail(n, SPICE_EINVAL, "Brunel+ slices hold < 2^32 synapses per rank (32-bit entry starts); got %llu",
                             (unsigned long long)n->nnz));
        if (n->N / 1024 + 1 > 1486)                        // (flush-row list of one step, sim.cu kPlFlush)
            return bail(fail(n, SPICE_EINVAL, "Brunel+ supports up to 1.5M neurons"));
        if ((st = dalloc_t(n, &n->w, n->nnz + 8, "plastic weights"))) return bail(st);
        if ((st = dalloc_t(n, &n->pring, (size_t)n->D * n->ring_stride, "plastic input ring"))) return bail(st);
        if ((st = dalloc_t(n, &n->pre_ts, 3ull * n->N, "pre spike steps"))) return bail(st);   // (by step mod 3)
        if ((st = dalloc_t(n, &n->pre_c, 3ull * n->N, "pre traces"))) return bail(st);
        if ((st = dalloc_t(n, &n->post, 2ull * 4 * no, "post spike history"))) return bail(st);
        if ((st = dalloc_t(n, &n->post_mask, 64ull * no, "post spike bit rings"))) return bail(st);
        if ((st = dalloc_t(n, &n->tab_p, 8192, "pre trace table"))) return bail(st);
        if ((st = dalloc_t(n, &n->tab_m, 8192, "post trace table"))) return bail(st);
        CU(n, cudaMemsetAsync(n->pring, 0, (size_t)n->D * n->ring_stride * 8, s));
        CU(n, cudaMemsetAsync(n->pre_ts, 0xFF, 3ull * n->N * 4, s));          // no spike yet
        CU(n, cudaMemsetAsync(n->pre_c, 0, 3ull * n->N * 4, s));
        {
            std::vector<uint32_t> init(4 * no);
            for (uint64_t i = 0; i < no; ++i) { init[4 * i] = init[4 * i + 1] = init[4 * i + 2] = 0xFFFFFFFFu; init[4 * i + 3] = 0u; }
            CU(n, cudaMemcpy(n->post, init.data(), init.size() * 4, cudaMemcpyHostToDevice));
            CU(n, cudaMemcpy(n->post + 4 * no, init.data(), init.size() * 4, cudaMemcpyHostToDevice));
        }
        CU(n, cudaMemsetAsync(n->post_mask, 0, 64ull * no * 4, s));
        // closed-form trace tables (reading R13): exp(-k dt / tau) in double, rounded once
        n->htab_p.resize(8192); n->htab_m.resize(8192);
        for (uint32_t k = 0; k < 8192; ++k) {
            n->htab_p[k] = (float)std::exp(-(double)k * n->dt / n->prm[10]);
            n->htab_m[k] = (float)std::exp(-(double)k * n->dt / n->prm[11]);
        }
        CU(n, cudaMemcpy(n->tab_p, n->htab_p.data(), 8192 * 4, cudaMemcpyHostToDevice));
        CU(n, cudaMemcpy(n->tab_m, n->htab_m.data(), 8192 * 4, cudaMemcpyHostToDevice));
        CU(n, gen_plastic_weights(g2, pbx, n->row_ptr, n->bnd, n->ent, n->w, (float)n->prm[15], s));
        CU(n, cudaStreamSynchronize(s));
    }
    build_model_const(n);
    GenGeom g{};
    g.N = n->N; g.n_own = (uint32_t)n->n_own; g.rank = n->rank; g.G = n->G; g.S = n->S;
    g.TW = n->TW; g.NT = n->NT; g.key0 = (uint32_t)n->seed; g.key1 = (uint32_t)(n->seed >> 32);
    const double *P = n->prm.data();
    if (n->model == SPICE_VOGELS) {
        CU(n, gen_init_uniform(g, 0, (float)P[11], (float)P[12], n->v, s));
        CU(n, gen_init_uniform(g, 1, (float)P[13], (float)P[14], n->ge, s));
        CU(n, gen_init_uniform(g, 2, (float)P[15], (float)P[16], n->gi, s));
    } else if (n->model == SPICE_BRUNEL || n->model == SPICE_BRUNEL_PLUS) {
        CU(n, gen_init_uniform(g, 0, (float)P[8], (float)P[9], n->v, s));
        std::vector<uint64_t> tab = poisson_table(P[7]);
        if (tab.empty()) return bail(fail(n, SPICE_EINVAL, "lambda_ext %g too large for the Poisson table", P[7]));
        if ((st = dalloc_t(n, &n->ptab, tab.size(), "Poisson table"))) return bail(st);
        CU(n, cudaMemcpyAsync(n->ptab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, s));
        n->mc.ptab = n->ptab;
        n->mc.ptab_len = (uint32_t)tab.size();
        uint32_t p2 = 1;
        while (p2 < n->mc.ptab_len) p2 <<= 1;
        n->mc.ptab_half = p2 >> 1;
    }
    CU(n, cudaStreamSynchronize(s));
    // padded-layout delivery structures: per-tile segment-descriptor lists (written by the
    // producers of the step's spikes, consumed through per-warp window rings).  Not with the
    // paper-style global-atomics delivery: it walks the spike lists itself.
    if (n->pad8 && !n->global_atomics) {
        // a tile's list holds every spike of the step: the rank's own (G = 1) or all N (G > 1)
        const uint64_t dstride = ((n->G == 1 ? n->n_own : (uint64_t)n->N) + 1) & ~1ull;
        // three step buffers: the producers of step t + 1 (synth fast path: in the prologue
        // of the kernel delivering t, which may overlap the kernel delivering t - 1)
        if ((st = dalloc_t(n, &n->desc, 3ull * n->NT * dstride, "segment descriptors"))) return bail(st);
        if ((st = dalloc_t(n, &n->dcount, 4, "descriptor counters"))) return bail(st);
        CU(n, cudaMemset(n->dcount, 0, 16));
    }
    if (n->C > 1 && !n->desc) n->fused = false;           // cluster tiles: descriptor path only
    if (n->G > 1 && !n->desc) n->fused = false;           // G > 1: fused only on the padded layout
    if (n->procedural) n->fused = false;                   // update + procedural delivery per step
    // ---- kernel arguments ----
    SimArgs &a = n->args;
    a.pdl = getenv("SPICE_NO_PDL") ? 0u : 1u;             // (A/B switch for measurements)
    a.model = n->model; a.N = n->N; a.n_exc = n->n_exc; a.delay = n->delay; a.D = n->D; a.dly = n->dly;
    a.rank = n->rank; a.G = n->G; a.S = n->S; a.n_own = (uint32_t)n->n_own; a.W = n->W;
    a.TW = n->TW; a.NT = n->NT; a.C = n->C; a.TWs = n->TWs; a.ring_stride = n->ring_stride; a.record_steps = n->R;
    a.mD = ~0ull / a.D + 1; a.mR = ~0ull / a.record_steps + 1;
    if (n->model == SPICE_BRUNEL_PLUS) {
        // every plastic weight stays in [0, max(w0, w_max)] (clamped potentiation, depression
        // floored at 0), so q = rint(w 2^32) <= qmax; a target receives at most N events per
        // step: the split sums cannot wrap when N (2^16 - 1) < 2^32 and N (qmax >> 16) < 2^32
        const double wtop = std::max(n->prm.size() > 15 ? n->prm[15] : 0.0, n->prm.size() > 14 ? n->prm[14] : 0.0);
        const double qmax = std::ceil(std::max(wtop, 0.0) * 4294967296.0);
        a.pl_split = (uint64_t)n->N * 65535ull < (1ull << 32) && qmax < 9.0e15 &&
                     (double)n->N * std::floor(qmax / 65536.0) < 4294967296.0 ? 1u : 0u;
    }
    a.prod_words = n->prod_words;
    if (getenv("SPICE_PHASES") && atoi(getenv("SPICE_PHASES"))) {     // diagnostics only
        if ((st = dalloc_t(n, &n->ptimes, (size_t)n->NT * n->C * 16, "phase clocks"))) return bail(st);
        CU(n, cudaMemset(n->ptimes, 0, (size_t)n->NT * n->C * 16 * 8));
        a.ptimes = n->ptimes;
    }
    a.key0 = (uint32_t)n->seed; a.key1 = (uint32_t)(n->seed >> 32);
    a.NR = n->NR; a.RS = n->RS;
    a.mc = n->mc;
    a.row_ptr = n->row_ptr; a.bnd = n->bnd; a.ent = n->ent; a.deg = n->deg; a.eshift = n->eshift; a.nnz = n->nnz;
    a.v = n->v; a.ge = n->ge; a.gi = n->gi; a.ref = n->ref; a.acc = n->acc; a.ring = n->ring;
    a.sl_ids = n->sl_ids; a.sl_rows = n->sl_rows; a.sl_counts = n->sl_counts; a.desc = n->desc;
    a.dstride = ((n->G == 1 ? n->n_own : (uint64_t)n->N) + 1) & ~1ull; a.dcount = n->dcount;
    a.record = n->record; a.sendbuf = n->sendbuf;
    a.gather = n->gather; a.fired_cta = n->fired_cta; a.delivered_cta = n->delivered_cta;
    a.t0 = n->t0; a.force_bits = n->force_bits; a.force_ctl = n->force_ctl;
    a.w = n->w; a.pring = n->pring;
    a.pre_ts = n->pre_ts; a.pre_c = n->pre_c; a.post = n->post; a.post_mask = n->post_mask;
    a.tab_p = n->tab_p; a.tab_m = n->tab_m;
    a.npl = pbx.n;
    if (n->procedural) {
        for (uint32_t r = 0; r < n->rules.size(); ++r) {
            const spice_rule &R = n->rules[r];
            const uint64_t thr = prob_threshold(R.p);
            const uint32_t lo = R.delay_min ? R.delay_min : n->delay, hi = R.delay_min && R.delay_max > lo ? R.delay_max : lo;
            uint32_t *P = a.proc[a.nproc++];
            P[0] = R.src_begin; P[1] = R.src_end; P[2] = R.dst_begin; P[3] = R.dst_end;
            P[4] = (uint32_t)thr; P[5] = (uint32_t)(thr >> 32); P[6] = r;
            P[7] = lo | (hi << 16);
        }
    }
    memcpy(a.pl, pbx.box, sizeof a.pl);
    CU(n, prepare_kernels(a));
    // G = 1 synth with delay 1: the steps of a graph replay in one persistent launch
    // (SPICE_NO_PERSIST=1: one fused kernel per step, the A/B baseline)
    if (n->G == 1 && n->fused && !n->global_atomics && !n->small && !n->procedural && !getenv("SPICE_NO_PERSIST") &&
        run_supported(a, n->n_sm)) {
        if ((st = dalloc_t(n, &n->gbar, 10, "grid barrier"))) return bail(st);   // 4 x u64 slots + flag
        CU(n, cudaMemset(n->gbar, 0, 40));
        a.gbar = n->gbar;
        a.persist = 1;
    }
    if (n->procedural) {            // exact synapse count and receptor-packing check (nothing stored)
        unsigned long long *cnt = nullptr;
        uint32_t *tc = nullptr, *mx = nullptr;
        if ((st = dalloc_t(n, &cnt, 1, "synapse count"))) return bail(st);
        if ((st = dalloc_t(n, &tc, 2 * std::max<uint64_t>(n->n_own, 1), "in-degree counts"))) return bail(st);
        if ((st = dalloc_t(n, &mx, 2, "in-degree max"))) return bail(st);
        CU(n, cudaMemsetAsync(cnt, 0, 8, s));
        CU(n, cudaMemsetAsync(tc, 0, 2 * std::max<uint64_t>(n->n_own, 1) * 4, s));
        CU(n, cudaMemsetAsync(mx, 0, 8, s));
        CU(n, launch_count_proc(a, cnt, tc, s));
        max_halves_kernel<<<n->n_sm * 4, 256, 0, s>>>(tc, 2 * n->n_own, mx);
        uint32_t h[2] = {0, 0};
        unsigned long long hc = 0;
        CU(n, cudaMemcpyAsync(&hc, cnt, 8, cudaMemcpyDeviceToHost, s));
        CU(n, cudaMemcpyAsync(h, mx, 8, cudaMemcpyDeviceToHost, s));
        CU(n, cudaStreamSynchronize(s));
        n->n_syn = hc;
        const uint64_t fb = 3ull * 8 + 2 * std::max<uint64_t>(n->n_own, 1) * 4;
        dfree(n, cnt); dfree(n, tc); dfree(n, mx);
        n->device_bytes -= fb;
        if (h[0] >= 65535u || h[1] > 0u)                   // (plain counts: any high half is >= 65536)
            return bail(fail(n, SPICE_EINVAL, "a target has >= 65535 in-synapses of one receptor type; packed counts could overflow"));
    }
    // the caller's stream may still be running work of its own: everything the library
    // enqueued on it so far (memsets, generator) is done; capture never touches it
    CU(n, cudaStreamSynchronize(s));
    if (n->peer) {
        // receive window: 2 parities x G x W bitmap words + G u64 flags; device memory from
        // cudaMalloc (exportable through CUDA IPC), released in destroy
        const size_t wb = (2ull * n->G * n->W + 2ull * n->G + 2) * 4;
        cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&n->win), wb);
        if (e != cudaSuccess) { cudaGetLastError(); return bail(fail(n, SPICE_ENOMEM, "cudaMalloc of the %zu-byte peer window failed", wb)); }
        CU(n, cudaMemset(n->win, 0, wb));
        if ((st = dalloc_t(n, &n->peers_dev, n->G, "peer window table"))) return bail(st);
        if ((st = dalloc_t(n, &n->xerr, 1, "exchange error flag"))) return bail(st);
        CU(n, cudaMemset(n->xerr, 0, 4));
        n->args.gather = n->win;
        n->args.peers = n->peers_dev;
        n->args.xerr = n->xerr;
        n->connected = false;                              // graphs are captured by spice_peer_connect
    }
    if (!n->external && !n->peer)
        for (uint32_t k = 0; k < spice_net::kGraphLevels; ++k)
            if ((st = capture_graph(n, 1u << k, &n->graphs[k]))) return bail(st);
    n->create_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_create).count();
    *out = n;
    return SPICE_OK;
}

spice_status spice_setup_times(spice_net *n, double *gen_ms, double *create_ms) {
    CHECK_NET(n);
    if (gen_ms) *gen_ms = n->gen_ms;
    if (create_ms) *create_ms = n->create_ms;
    return SPICE_OK;
}

// A compacted read-out still pending on the read-out stream holds ring slots
// [t_begin, t_end) until done: steps from t_begin + R on (which overwrite them) wait for it.
spice_status guard_readout(spice_net *n, uint64_t steps) {
    for (auto &sl : n->slot)
        if (sl.full && sl.compact && !sl.guarded && n->t_host + steps > sl.t_begin + n->R) {
            CU(n, cudaStreamWaitEvent(n->stream, sl.done, 0));
            sl.guarded = true;
        }
    return SPICE_OK;
}

spice_status spice_step(spice_net *n, uint64_t steps) {
    CHECK_NET(n);
    if (n->external) return fail(n, SPICE_ESTATE, "external-exchange networks step via spice_exchange_begin/end");
    if (!n->connected) return fail(n, SPICE_ESTATE, "PEER exchange: call spice_peer_connect first");
    if (spice_status st = guard_readout(n, steps)) return st;
    while (steps) {                                        // largest graph first
        uint32_t k = spice_net::kGraphLevels - 1;
        while ((1ull << k) > steps) --k;
        CU(n, cudaGraphLaunch(n->graphs[k], n->stream));
        steps -= 1ull << k;
        n->t_host += 1ull << k;
    }
    return SPICE_OK;
}

namespace {
struct PeerBlob {                 // spice_peer_handle's 128 bytes
    cudaIpcMemHandle_t ipc;       // 64
    uint64_t pid;
    uint64_t ptr;                 // the window's address in the exporting process
    int32_t device;
    uint32_t magic, rank, G, W, pad[7];
};
static_assert(sizeof(PeerBlob) == 128, "peer handle size");
constexpr uint32_t kPeerMagic = 0x45435053u;   // "SPCE"

// PEER exchange errors surface at the next host synchronisation
spice_status check_xerr(spice_net *n) {
    uint32_t e = 0;
    if (n->gbar) {                                 // (and the persistent kernel's grid barrier)
        CU(n, cudaMemcpy(&e, n->gbar + 8, 4, cudaMemcpyDeviceToHost));
        if (e) return fail(n, SPICE_ECUDA, "persistent step kernel: a grid barrier did not complete within 10 s");
    }
    if (!n->xerr) return SPICE_OK;
    CU(n, cudaMemcpy(&e, n->xerr, 4, cudaMemcpyDeviceToHost));
    if (e) return fail(n, SPICE_ENCCL, "PEER exchange: rank %u's bitmap did not arrive within 20 s", e - 1);
    return SPICE_OK;
}
}  // namespace

spice_status spice_peer_handle(spice_net *n, void *out128) {
    CHECK_NET(n);
    if (!n->peer || !out128) return fail(n, SPICE_EINVAL, "not a PEER-exchange network (or null output)");
    PeerBlob b{};
    CU(n, cudaIpcGetMemHandle(&b.ipc, n->win));
    b.pid = (uint64_t)getpid();
    b.ptr = (uint64_t)(uintptr_t)n->win;
    b.device = n->device;
    b.magic = kPeerMagic;
    b.rank = n->rank;
    b.G = n->G;
    b.W = n->W;
    memcpy(out128, &b, sizeof b);
    return SPICE_OK;
}

spice_status spice_peer_connect(spice_net *n, const void *handles) {
    CHECK_NET(n);
    if (!n->peer || !handles) return fail(n, SPICE_EINVAL, "not a PEER-exchange network (or null handles)");
    if (n->connected) return fail(n, SPICE_ESTATE, "already connected");
    std::vector<uint32_t *> ptrs(n->G, nullptr);
    for (uint32_t r = 0; r < n->G; ++r) {
        PeerBlob b;
        memcpy(&b, static_cast<const char *>(handles) + 128ull * r, sizeof b);
        if (b.magic != kPeerMagic || b.rank != r || b.G != n->G || b.W != n->W)
            return fail(n, SPICE_EINVAL, "peer handle %u is not rank %u of this %u-rank network", r, r, n->G);
        if (r == n->rank) { ptrs[r] = n->win; continue; }
        if (b.pid == (uint64_t)getpid()) { ptrs[r] = reinterpret_cast<uint32_t *>(b.ptr); continue; }   // same process
        void *p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, b.ipc, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(n, SPICE_ECUDA, "cudaIpcOpenMemHandle(rank %u): %s", r, cudaGetErrorString(e));
        n->opened.push_back(p);
        ptrs[r] = static_cast<uint32_t *>(p);
    }
    CU(n, cudaMemcpy(n->peers_dev, ptrs.data(), n->G * sizeof(uint32_t *), cudaMemcpyHostToDevice));
    for (uint32_t k = 0; k < spice_net::kGraphLevels; ++k) {
        spice_status st = capture_graph(n, 1u << k, &n->graphs[k]);
        if (st) return st;
    }
    n->connected = true;
    return SPICE_OK;
}

spice_status spice_exchange_begin(spice_net *n) {
    CHECK_NET(n);
    if (!n->external) return fail(n, SPICE_ESTATE, "not an external-exchange network");
    if (spice_status st = guard_readout(n, 2)) return st;
    CU(n, launch_update(n->args, 0, n->stream));
    CU(n, cudaEventRecord(n->ev, n->stream));
    return SPICE_OK;
}

spice_status spice_exchange_put(spice_net *dst, spice_net *src) {
    CHECK_NET(dst);
    CHECK_NET(src);
    if (dst->W != src->W || src->rank >= dst->G) return fail(dst, SPICE_EINVAL, "incompatible exchange peers");
    CU(dst, cudaStreamWaitEvent(dst->stream, src->ev, 0));
    CU(dst, cudaMemcpyAsync(dst->gather + (uint64_t)src->rank * src->W, src->sendbuf, (size_t)src->W * 4,
                            cudaMemcpyDeviceToDevice, dst->stream));
    // test hook: complete the copy so src may overwrite its send buffer next step
    CU(dst, cudaStreamSynchronize(dst->stream));
    return SPICE_OK;
}

spice_status spice_exchange_get_send(spice_net *n, uint32_t *out, int on_device) {
    CHECK_NET(n);
    if (!n->external) return fail(n, SPICE_ESTATE, "not an external-exchange network");
    if (!out) return fail(n, SPICE_EINVAL, "null buffer");
    const size_t bytes = (size_t)n->W * 4;
    if (on_device) {
        CU(n, cudaMemcpyAsync(out, n->sendbuf, bytes, cudaMemcpyDeviceToDevice, n->stream));
    } else {
        CU(n, cudaMemcpyAsync(out, n->sendbuf, bytes, cudaMemcpyDeviceToHost, n->stream));
        CU(n, cudaStreamSynchronize(n->stream));
    }
    return SPICE_OK;
}

spice_status spice_exchange_set_recv(spice_net *n, uint32_t rank, const uint32_t *words, int on_device) {
    CHECK_NET(n);
    if (!n->external) return fail(n, SPICE_ESTATE, "not an external-exchange network");
    if (!words || rank >= n->G) return fail(n, SPICE_EINVAL, "null buffer or rank out of range");
    const size_t bytes = (size_t)n->W * 4;
    uint32_t *dst = n->gather + (uint64_t)rank * n->W;
    if (on_device) {
        CU(n, cudaMemcpyAsync(dst, words, bytes, cudaMemcpyDeviceToDevice, n->stream));
    } else {
        CU(n, cudaMemcpyAsync(dst, words, bytes, cudaMemcpyHostToDevice, n->stream));
        CU(n, cudaStreamSynchronize(n->stream));
    }
    return SPICE_OK;
}

spice_status spice_exchange_end(spice_net *n) {
    CHECK_NET(n);
    if (!n->external) return fail(n, SPICE_ESTATE, "not an external-exchange network");
    if (spice_status st = guard_readout(n, 2)) return st;
    if (n->G > 1) CU(n, launch_bitmap_to_list(n->args, 0, n->stream));
    CU(n, launch_deliver(n->args, 0, n->global_atomics, n->n_sm, n->stream));
    CU(n, launch_advance(n->t0, 1, n->stream));
    CU(n, cudaEventRecord(n->ev, n->stream));
    n->t_host += 1;
    return SPICE_OK;
}

spice_status spice_exchange_end_fused(spice_net *n) {
    CHECK_NET(n);
    if (!n->external) return fail(n, SPICE_ESTATE, "not an external-exchange network");
    if (spice_status st = guard_readout(n, 2)) return st;
    if (!n->fused || n->global_atomics || n->G == 1) return fail(n, SPICE_ESTATE, "no fused G > 1 path on this network");
    CU(n, launch_bitmap_to_list(n->args, 0, n->stream));
    CU(n, launch_fused(n->args, 0, n->stream));        // deliver(t) + update(t+1): next bitmap
    CU(n, launch_advance(n->t0, 1, n->stream));
    CU(n, cudaEventRecord(n->ev, n->stream));
    n->t_host += 1;
    return SPICE_OK;
}

spice_status spice_read_spikes(spice_net *n, uint64_t t_begin, uint64_t t_end, uint32_t *ids,
                               uint64_t cap, uint64_t *offsets, uint64_t *total) {
    CHECK_NET(n);
    if (t_begin > t_end || t_end > n->t_host || (n->t_host > n->R && t_begin < n->t_host - n->R))
        return fail(n, SPICE_ERANGE, "steps [%llu, %llu) not in the record ring (have [%llu, %llu))",
                    (unsigned long long)t_begin, (unsigned long long)t_end,
                    (unsigned long long)(n->t_host > n->R ? n->t_host - n->R : 0), (unsigned long long)n->t_host);
    const uint64_t words = (uint64_t)n->G * n->W;
    const uint64_t nsteps = t_end - t_begin;
    // bitmaps of the requested steps -> a pinned host buffer (one async copy per contiguous
    // run of ring slots, one stream synchronisation), then decoded on the host
    if (n->hbm_words < nsteps * words) {
        if (n->hbm) cudaFreeHost(n->hbm);
        n->hbm = nullptr;
        n->hbm_words = 0;
        CU(n, cudaMallocHost(reinterpret_cast<void **>(&n->hbm), std::max<uint64_t>(nsteps * words, 1) * 4));
        n->hbm_words = nsteps * words;
    }
    for (uint64_t t = t_begin; t < t_end;) {
        const uint64_t slot = t % n->R;
        const uint64_t run = std::min<uint64_t>(t_end - t, n->R - slot);
        CU(n, cudaMemcpyAsync(n->hbm + (t - t_begin) * words, n->record + slot * words, run * words * 4,
                              cudaMemcpyDeviceToHost, n->stream));
        t += run;
    }
    CU(n, cudaStreamSynchronize(n->stream));
    if (spice_status xs = check_xerr(n)) return xs;
    std::vector<std::vector<uint32_t>> &per = n->hdec;
    const uint64_t tot = decode_steps(n->hbm, nsteps, words, n->G, n->W, n->S, per);
    if (total) *total = tot;
    if (tot > cap || (!ids && tot)) return fail(n, SPICE_ETRUNC, "need %llu ids", (unsigned long long)tot);
    uint64_t o = 0;
    for (uint64_t q = 0; q < per.size(); ++q) {
        if (offsets) offsets[q] = o;
        memcpy(ids + o, per[q].data(), per[q].size() * 4);
        o += per[q].size();
    }
    if (offsets) offsets[per.size()] = o;
    return SPICE_OK;
}

spice_status spice_spikes_prefetch(spice_net *n, uint64_t t_begin, uint64_t t_end, uint32_t slot) {
    CHECK_NET(n);
    if (slot > 1) return fail(n, SPICE_EINVAL, "slot must be 0 or 1");
    if (t_begin > t_end || t_end > n->t_host || (n->t_host > n->R && t_begin < n->t_host - n->R) ||
        t_end - t_begin > n->R)
        return fail(n, SPICE_ERANGE, "steps [%llu, %llu) not in the record ring (have [%llu, %llu))",
                    (unsigned long long)t_begin, (unsigned long long)t_end,
                    (unsigned long long)(n->t_host > n->R ? n->t_host - n->R : 0), (unsigned long long)n->t_host);
    spice_net::Slot &sl = n->slot[slot];
    if (sl.full) CU(n, cudaEventSynchronize(sl.done));    // (an uncollected earlier copy)
    const uint64_t words = (uint64_t)n->G * n->W, nsteps = t_end - t_begin;
    if (!sl.done) CU(n, cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    sl.t_begin = t_begin;
    sl.t_end = t_end;
    sl.compact = nsteps * words >= (1u << 16);
    if (!sl.compact) {         // small bitmaps: copy them as they are, collect decodes on the host
        const uint64_t need = std::max<uint64_t>(nsteps * words, 1);
        if (sl.words < need) {
            if (sl.h) cudaFreeHost(sl.h);
            sl.h = nullptr;
            sl.words = 0;
            CU(n, cudaMallocHost(reinterpret_cast<void **>(&sl.h), need * 4));
            sl.words = need;
        }
        for (uint64_t t = t_begin; t < t_end;) {        // one copy per contiguous run of ring slots
            const uint64_t rs = t % n->R;
            const uint64_t run = std::min<uint64_t>(t_end - t, n->R - rs);
            CU(n, cudaMemcpyAsync(sl.h + (t - t_begin) * words, n->record + rs * words, run * words * 4,
                                  cudaMemcpyDeviceToHost, n->stream));
            t += run;
        }
        CU(n, cudaEventRecord(sl.done, n->stream));
        sl.full = true;
        return SPICE_OK;
    }
    // the chunk's bitmaps are compacted on the device into per-step counts and packed
    // ascending IDs; the counts and a guess of the IDs (1.25x the previous chunk's total)
    // are copied now, collect fetches any remainder
    const uint64_t worst = std::max<uint64_t>(nsteps * n->N, 1);
    spice_status st;
    if (sl.dcap < worst) {
        dfree(n, sl.d_ids);
        sl.d_ids = nullptr;
        sl.dcap = 0;
        if ((st = dalloc_t(n, &sl.d_ids, worst, "read-out IDs"))) return st;
        sl.dcap = worst;
    }
    if (sl.ccap < nsteps + 1) {
        dfree(n, sl.d_cnt);
        sl.d_cnt = nullptr;
        if (sl.h_cnt) cudaFreeHost(sl.h_cnt);
        sl.h_cnt = nullptr;
        sl.ccap = 0;
        if ((st = dalloc_t(n, &sl.d_cnt, nsteps + 1, "read-out counts"))) return st;
        CU(n, cudaMallocHost(reinterpret_cast<void **>(&sl.h_cnt), (nsteps + 1) * 4));
        sl.ccap = nsteps + 1;
    }
    if (!sl.guess) sl.guess = nsteps * std::max<uint64_t>(1024, n->N / 32);
    const uint64_t guess = std::min<uint64_t>(sl.guess, worst);
    if (sl.words < guess) {
        if (sl.h) cudaFreeHost(sl.h);
        sl.h = nullptr;
        sl.words = 0;
        CU(n, cudaMallocHost(reinterpret_cast<void **>(&sl.h), guess * 4));
        sl.words = guess;
    }
    // on the read-out stream, after the steps enqueued so far (an event), concurrently with
    // the steps enqueued later; a step that would overwrite these ring slots (t_begin + R
    // onwards) waits for it (guard_readout)
    if (!n->xfer) CU(n, cudaStreamCreateWithFlags(&n->xfer, cudaStreamNonBlocking));
    if (!sl.ready) CU(n, cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
    CU(n, cudaEventRecord(sl.ready, n->stream));
    CU(n, cudaStreamWaitEvent(n->xfer, sl.ready, 0));
    CU(n, launch_compact(n->record, n->R, words, t_begin, (uint32_t)nsteps, n->G, n->W, n->S, n->N, sl.d_cnt,
                         sl.d_ids, n->xfer));
    CU(n, cudaMemcpyAsync(sl.h_cnt, sl.d_cnt, nsteps * 4, cudaMemcpyDeviceToHost, n->xfer));
    CU(n, cudaMemcpyAsync(sl.h, sl.d_ids, guess * 4, cudaMemcpyDeviceToHost, n->xfer));
    CU(n, cudaEventRecord(sl.done, n->xfer));
    sl.copied = guess;
    sl.guarded = false;
    sl.full = true;
    return SPICE_OK;
}

spice_status spice_spikes_collect(spice_net *n, uint32_t slot, uint32_t *ids, uint64_t cap,
                                  uint64_t *offsets, uint64_t *total) {
    CHECK_NET(n);
    if (slot > 1) return fail(n, SPICE_EINVAL, "slot must be 0 or 1");
    spice_net::Slot &sl = n->slot[slot];
    if (!sl.full) return fail(n, SPICE_ESTATE, "slot %u holds no prefetched steps", slot);
    CU(n, cudaEventSynchronize(sl.done));
    const uint64_t nsteps = sl.t_end - sl.t_begin;
    if (!sl.compact) {
        const uint64_t words = (uint64_t)n->G * n->W;
        std::vector<std::vector<uint32_t>> &per = n->hdec;
        const uint64_t tot = decode_steps(sl.h, nsteps, words, n->G, n->W, n->S, per);
        if (total) *total = tot;
        if (tot > cap || (!ids && tot)) return fail(n, SPICE_ETRUNC, "need %llu ids", (unsigned long long)tot);
        uint64_t o = 0;
        for (uint64_t q = 0; q < nsteps; ++q) {
            if (offsets) offsets[q] = o;
            if (!per[q].empty()) memcpy(ids + o, per[q].data(), per[q].size() * 4);
            o += per[q].size();
        }
        if (offsets) offsets[nsteps] = o;
        sl.full = false;
        return SPICE_OK;
    }
    uint64_t tot = 0;
    for (uint64_t q = 0; q < nsteps; ++q) tot += sl.h_cnt[q];
    if (total) *total = tot;
    if (tot > cap || (!ids && tot)) return fail(n, SPICE_ETRUNC, "need %llu ids", (unsigned long long)tot);
    if (tot > sl.copied) {                               // more than the guess: the rest now
        if (sl.words < tot) {
            uint32_t *h2 = nullptr;
            CU(n, cudaMallocHost(reinterpret_cast<void **>(&h2), tot * 4));
            memcpy(h2, sl.h, sl.copied * 4);
            cudaFreeHost(sl.h);
            sl.h = h2;
            sl.words = tot;
        }
        if (!n->xfer) CU(n, cudaStreamCreateWithFlags(&n->xfer, cudaStreamNonBlocking));
        CU(n, cudaMemcpyAsync(sl.h + sl.copied, sl.d_ids + sl.copied, (tot - sl.copied) * 4,
                              cudaMemcpyDeviceToHost, n->xfer));
        CU(n, cudaStreamSynchronize(n->xfer));
        sl.copied = tot;
    }
    sl.guess = tot + tot / 4 + 4096;
    uint64_t o = 0;
    for (uint64_t q = 0; q < nsteps; ++q) {
        if (offsets) offsets[q] = o;
        o += sl.h_cnt[q];
    }
    if (offsets) offsets[nsteps] = o;
    if (tot) memcpy(ids, sl.h, tot * 4);
    sl.full = false;
    return SPICE_OK;
}

namespace {
// Philox4x32-10 on the host (the same published algorithm as the device's, for regenerating
// procedural rows in the read-out hooks)
void philox_host(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
// Row s of a procedural network on this rank: (global target, delay) pairs, ascending.
void procedural_row(const spice_net *n, uint32_t s, std::vector<std::pair<uint32_t, uint8_t>> &row) {
    row.clear();
    const uint32_t k0 = (uint32_t)n->seed, k1 = (uint32_t)(n->seed >> 32);
    for (uint64_t i = 0; i < n->n_own; ++i) {
        const uint32_t j = (uint32_t)local_to_global(i, n->rank, n->G, n->S);
        for (uint32_t r = 0; r < n->rules.size(); ++r) {
            const spice_rule &R = n->rules[r];
            if (s < R.src_begin || s >= R.src_end || j < R.dst_begin || j >= R.dst_end) continue;
            const uint32_t ctr[4] = {s, j >> 2, r, kTagConn};
            uint32_t o[4];
            philox_host(ctr, k0, k1, o);
            if ((uint64_t)o[j & 3] >= prob_threshold(R.p)) continue;
            const uint32_t lo = R.delay_min ? R.delay_min : n->delay;
            const uint32_t hi = R.delay_min && R.delay_max > lo ? R.delay_max : lo;
            uint32_t d = lo;
            if (hi > lo) {
                const uint32_t cd[4] = {s, j >> 2, r, kTagDelay};
                philox_host(cd, k0, k1, o);
                d += (uint32_t)(((uint64_t)o[j & 3] * (hi - lo + 1)) >> 32);
            }
            row.emplace_back(j, (uint8_t)d);
        }
    }
    std::sort(row.begin(), row.end());
}
}  // namespace

spice_status spice_read_connectivity(spice_net *n, uint32_t row_begin, uint32_t row_end, uint32_t *tgt,
                                     uint64_t cap, uint64_t *row_offsets, uint64_t *total) {
    CHECK_NET(n);
    if (row_begin > row_end || row_end > n->N) return fail(n, SPICE_EINVAL, "rows outside [0, N)");
    if (n->procedural) {                       // regenerated (the device stores no rows)
        std::vector<std::pair<uint32_t, uint8_t>> row;
        uint64_t o = 0;
        for (uint32_t q = row_begin; q < row_end; ++q) {
            procedural_row(n, q, row);
            if (row_offsets) row_offsets[q - row_begin] = o;
            for (auto &e : row) { if (tgt && o < cap) tgt[o] = e.first; ++o; }
        }
        if (row_offsets) row_offsets[row_end - row_begin] = o;
        if (total) *total = o;
        if (o > cap || (!tgt && o)) return fail(n, SPICE_ETRUNC, "need %llu targets", (unsigned long long)o);
        return SPICE_OK;
    }
    CU(n, cudaStreamSynchronize(n->stream));
    const uint32_t nr = row_end - row_begin;
    std::vector<uint64_t> rp(nr + 1);
    CU(n, cudaMemcpy(rp.data(), n->row_ptr + row_begin, (nr + 1) * 8ull, cudaMemcpyDeviceToHost));
    const uint64_t stored = rp[nr] - rp[0];
    std::vector<uint64_t> off(nr + 1, 0);       // output offsets (padding sentinels excluded)
    if (n->pad8) {
        std::vector<uint32_t> dg(nr ? nr : 1);
        if (nr) CU(n, cudaMemcpy(dg.data(), n->deg + row_begin, nr * 4ull, cudaMemcpyDeviceToHost));
        for (uint32_t q = 0; q < nr; ++q) off[q + 1] = off[q] + dg[q];
    } else {
        for (uint32_t q = 0; q <= nr; ++q) off[q] = rp[q] - rp[0];
    }
    const uint64_t tot = off[nr];
    if (total) *total = tot;
    if (tot > cap || (!tgt && tot)) return fail(n, SPICE_ETRUNC, "need %llu targets", (unsigned long long)tot);
    std::vector<uint32_t> bd((uint64_t)nr * (n->NT + 1));
    std::vector<uint16_t> en(stored ? stored : 1);
    if (nr) CU(n, cudaMemcpy(bd.data(), n->bnd + (uint64_t)row_begin * (n->NT + 1), bd.size() * 4, cudaMemcpyDeviceToHost));
    if (stored) CU(n, cudaMemcpy(en.data(), n->ent + rp[0], stored * 2, cudaMemcpyDeviceToHost));
    for (uint32_t q = 0; q < nr; ++q) {
        if (row_offsets) row_offsets[q] = off[q];
        const uint32_t *B = bd.data() + (uint64_t)q * (n->NT + 1);
        uint64_t o = off[q];
        for (uint32_t b = 0; b < n->NT; ++b)
            for (uint32_t e = B[b]; e < B[b + 1]; ++e) {
                const uint32_t x = (uint32_t)en[rp[q] - rp[0] + e] >> n->eshift;
                if (x >= n->TW) continue;                       // padding sentinel
                tgt[o++] = (uint32_t)local_to_global((uint64_t)b * n->TW + x, n->rank, n->G, n->S);
            }
        if (o != off[q + 1]) return fail(n, SPICE_ECUDA, "row %u: %llu targets, out-degree %llu", row_begin + q,
                                         (unsigned long long)(o - off[q]), (unsigned long long)(off[q + 1] - off[q]));
    }
    if (row_offsets) row_offsets[nr] = tot;
    return SPICE_OK;
}

spice_status spice_read_delays(spice_net *n, uint32_t row_begin, uint32_t row_end, uint8_t *out,
                               uint64_t cap, uint64_t *total) {
    CHECK_NET(n);
    if (row_begin > row_end || row_end > n->N) return fail(n, SPICE_EINVAL, "rows outside [0, N)");
    if (n->procedural) {
        std::vector<std::pair<uint32_t, uint8_t>> row;
        uint64_t o = 0;
        for (uint32_t q = row_begin; q < row_end; ++q) {
            procedural_row(n, q, row);
            for (auto &e : row) { if (out && o < cap) out[o] = e.second; ++o; }
        }
        if (total) *total = o;
        if (o > cap || (!out && o)) return fail(n, SPICE_ETRUNC, "need %llu delays", (unsigned long long)o);
        return SPICE_OK;
    }
    CU(n, cudaStreamSynchronize(n->stream));
    const uint32_t nr = row_end - row_begin;
    std::vector<uint64_t> rp(nr + 1);
    CU(n, cudaMemcpy(rp.data(), n->row_ptr + row_begin, (nr + 1) * 8ull, cudaMemcpyDeviceToHost));
    const uint64_t stored = rp[nr] - rp[0];
    std::vector<uint32_t> bd((uint64_t)nr * (n->NT + 1));
    std::vector<uint16_t> en(stored ? stored : 1);
    std::vector<uint8_t> dl(stored ? stored : 1, (uint8_t)n->delay);
    if (nr) CU(n, cudaMemcpy(bd.data(), n->bnd + (uint64_t)row_begin * (n->NT + 1), bd.size() * 4, cudaMemcpyDeviceToHost));
    if (stored) CU(n, cudaMemcpy(en.data(), n->ent + rp[0], stored * 2, cudaMemcpyDeviceToHost));
    if (stored && n->dly) CU(n, cudaMemcpy(dl.data(), n->dly + rp[0], stored, cudaMemcpyDeviceToHost));
    uint64_t o = 0;                                       // connectivity order, sentinels removed
    for (uint32_t q = 0; q < nr; ++q) {
        const uint32_t *B = bd.data() + (uint64_t)q * (n->NT + 1);
        for (uint32_t b = 0; b < n->NT; ++b)
            for (uint32_t e = B[b]; e < B[b + 1]; ++e) {
                const uint64_t k = rp[q] - rp[0] + e;
                if (((uint32_t)en[k] >> n->eshift) >= n->TW) continue;
                if (out && o < cap) out[o] = dl[k];
                ++o;
            }
    }
    if (total) *total = o;
    if (o > cap || (!out && o)) return fail(n, SPICE_ETRUNC, "need %llu delays", (unsigned long long)o);
    return SPICE_OK;
}

static spice_status field_ptr(spice_net *n, uint32_t field, void **p) {
    *p = nullptr;
    switch (field) {
    case SPICE_FIELD_V: *p = n->model != SPICE_SYNTH ? n->v : nullptr; break;
    case SPICE_FIELD_GE: *p = n->ge; break;
    case SPICE_FIELD_GI: *p = n->gi; break;
    case SPICE_FIELD_REF: *p = n->model != SPICE_SYNTH ? n->ref : nullptr; break;
    case SPICE_FIELD_ACC: *p = n->acc; break;
    case SPICE_FIELD_XTR: *p = n->pre_c; break;
    case SPICE_FIELD_YTR: *p = n->post; break;
    default: break;
    }
    if (!*p) return fail(n, SPICE_EINVAL, "field %u not present for model %u", field, n->model);
    return SPICE_OK;
}

spice_status spice_read_state(spice_net *n, uint32_t field, void *out, uint64_t count) {
    CHECK_NET(n);
    void *p;
    spice_status st = field_ptr(n, field, &p);
    if (st) return st;
    if (count != n->n_own) return fail(n, SPICE_EINVAL, "n = %llu, owned = %llu", (unsigned long long)count, (unsigned long long)n->n_own);
    CU(n, cudaStreamSynchronize(n->stream));
    // traces in event-driven form (reading R13): X(t) = c P[t - ts], evaluated here at
    // t = steps done with the device's operation (one rounded float product)
    auto tr = [&](float c, uint32_t ts, const std::vector<float> &tab) -> float {
        if (ts == 0xFFFFFFFFu) return 0.0f;
        const uint64_t k = n->t_host - ts;
        return k < tab.size() ? c * tab[k] : 0.0f;
    };
    if (field == SPICE_FIELD_XTR) {           // pre traces of the owned neurons (global arrays)
        const uint64_t par = n->t_host % 3;             // (pre state copies by step mod 3)
        std::vector<float> c(n->N);
        std::vector<uint32_t> ts(n->N);
        CU(n, cudaMemcpy(c.data(), n->pre_c + par * n->N, n->N * 4ull, cudaMemcpyDeviceToHost));
        CU(n, cudaMemcpy(ts.data(), n->pre_ts + par * n->N, n->N * 4ull, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < count; ++i) {
            const uint64_t j = local_to_global(i, n->rank, n->G, n->S);
            ((float *)out)[i] = tr(c[j], ts[j], n->htab_p);
        }
        return SPICE_OK;
    }
    if (field == SPICE_FIELD_YTR) {           // post traces (post history, parity of t)
        std::vector<uint32_t> h(4 * count);
        if (count) CU(n, cudaMemcpy(h.data(), n->post + (n->t_host & 1) * 4 * n->ring_stride, count * 16, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < count; ++i) {
            float c;
            memcpy(&c, &h[4 * i + 3], 4);
            ((float *)out)[i] = tr(c, h[4 * i], n->htab_m);
        }
        return SPICE_OK;
    }
    if (count) CU(n, cudaMemcpy(out, p, count * 4, cudaMemcpyDeviceToHost));
    return SPICE_OK;
}

spice_status spice_write_state(spice_net *n, uint32_t field, const void *in, uint64_t count) {
    CHECK_NET(n);
    void *p;
    spice_status st = field_ptr(n, field, &p);
    if (st) return st;
    if (count != n->n_own) return fail(n, SPICE_EINVAL, "n = %llu, owned = %llu", (unsigned long long)count, (unsigned long long)n->n_own);
    CU(n, cudaStreamSynchronize(n->stream));
    if (field == SPICE_FIELD_XTR || field == SPICE_FIELD_YTR)
        return fail(n, SPICE_EINVAL, "STDP traces are event-driven state (last spike step + value): read-only");
    if (count) CU(n, cudaMemcpy(p, in, count * 4, cudaMemcpyHostToDevice));
    return SPICE_OK;
}

spice_status spice_read_input(spice_net *n, uint32_t rel, uint32_t *counts, int64_t *plastic, uint64_t count) {
    CHECK_NET(n);
    if (rel >= n->D) return fail(n, SPICE_EINVAL, "rel %u >= D %u", rel, n->D);
    if (count != n->n_own) return fail(n, SPICE_EINVAL, "n must equal the owned count");
    CU(n, cudaStreamSynchronize(n->stream));
    const uint64_t slot = (n->t_host + rel) % n->D;
    if (counts && count) CU(n, cudaMemcpy(counts, n->ring + slot * n->ring_stride, count * 4, cudaMemcpyDeviceToHost));
    if (plastic) {
        if (n->pring && count) CU(n, cudaMemcpy(plastic, n->pring + slot * n->ring_stride, count * 8, cudaMemcpyDeviceToHost));
        else memset(plastic, 0, count * 8);
    }
    return SPICE_OK;
}

spice_status spice_read_weights(spice_net *n, uint32_t row_begin, uint32_t row_end, float *w,
                                uint64_t cap, uint64_t *total) {
    CHECK_NET(n);
    if (!n->w) return fail(n, SPICE_EINVAL, "model %u has no plastic weights", n->model);
    if (row_begin > row_end || row_end > n->N) return fail(n, SPICE_EINVAL, "rows outside [0, N)");
    CU(n, cudaStreamSynchronize(n->stream));
    uint64_t rp[2];
    CU(n, cudaMemcpy(&rp[0], n->row_ptr + row_begin, 8, cudaMemcpyDeviceToHost));
    CU(n, cudaMemcpy(&rp[1], n->row_ptr + row_end, 8, cudaMemcpyDeviceToHost));
    const uint64_t tot = rp[1] - rp[0];
    if (total) *total = tot;
    if (tot > cap || (!w && tot)) return fail(n, SPICE_ETRUNC, "need %llu weights", (unsigned long long)tot);
    if (tot) {
        // the eager rule's weights: stored weights plus the rows' pending (lazy) potentiations
        float *dv = nullptr;
        spice_status st2 = dalloc_t(n, &dv, tot, "weight read-out");
        if (st2) return st2;
        CU(n, launch_settle_weights(n->args, n->t_host, row_begin, row_end, dv, n->stream));
        CU(n, cudaMemcpyAsync(w, dv, tot * 4, cudaMemcpyDeviceToHost, n->stream));
        CU(n, cudaStreamSynchronize(n->stream));
        dfree(n, dv);
        n->device_bytes -= tot * 4;
    }
    return SPICE_OK;
}

spice_status spice_force_spikes(spice_net *n, const uint32_t *ids, uint64_t count, int mode) {
    CHECK_NET(n);
    if (mode != 1 && mode != 2) return fail(n, SPICE_EINVAL, "mode must be 1 (replace) or 2 (add)");
    std::vector<uint32_t> bits(std::max<uint32_t>(n->W, 1), 0u);
    for (uint64_t q = 0; q < count; ++q) {
        const uint32_t j = ids[q];
        if (j >= n->N) return fail(n, SPICE_EINVAL, "id %u >= N", j);
        if ((j / n->S) % n->G != n->rank) continue;
        const uint64_t i = (uint64_t)(j / n->S / n->G) * n->S + j % n->S;   // inverse of Listing 1
        bits[i >> 5] |= 1u << (i & 31);
    }
    const uint64_t ctl[2] = {n->t_host, (uint64_t)mode};
    CU(n, cudaMemcpyAsync(n->force_bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice, n->stream));
    CU(n, cudaMemcpyAsync(n->force_ctl, ctl, 16, cudaMemcpyHostToDevice, n->stream));
    CU(n, cudaStreamSynchronize(n->stream));
    return SPICE_OK;
}

spice_status spice_stats(spice_net *n, uint64_t *steps, uint64_t *fired, uint64_t *delivered) {
    CHECK_NET(n);
    CU(n, cudaStreamSynchronize(n->stream));
    std::vector<unsigned long long> f((size_t)n->NT * n->C), d((size_t)n->NT * n->C);
    CU(n, cudaMemcpy(f.data(), n->fired_cta, f.size() * 8, cudaMemcpyDeviceToHost));
    CU(n, cudaMemcpy(d.data(), n->delivered_cta, d.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long sf = 0, sd = 0;
    for (auto x : f) sf += x;
    for (auto x : d) sd += x;
    if (steps) *steps = n->t_host;
    if (fired) *fired = sf;
    if (delivered) *delivered = sd;
    return SPICE_OK;
}

void *spice_stream(spice_net *n) { return n ? (void *)n->stream : nullptr; }

spice_status spice_sync(spice_net *n) {
    CHECK_NET(n);
    CU(n, cudaStreamSynchronize(n->stream));
    return check_xerr(n);
}

spice_status spice_info(spice_net *n, uint64_t *n_owned, uint64_t *n_syn, uint32_t *n_tiles,
                        uint32_t *tile_width, uint32_t *ctas, uint64_t *bytes) {
    CHECK_NET(n);
    if (n_owned) *n_owned = n->n_own;
    if (n_syn) *n_syn = n->n_syn;
    if (n_tiles) *n_tiles = n->NT;
    if (tile_width) *tile_width = n->TW;
    if (ctas) *ctas = n->C;
    if (bytes) *bytes = n->device_bytes;
    return SPICE_OK;
}

spice_status spice_profile(spice_net *n, uint64_t steps, double *ms, uint32_t cap, uint32_t *nk) {
    CHECK_NET(n);
    if (n->external) return fail(n, SPICE_ESTATE, "profiling needs an NCCL, PEER or single-GPU network");
    if (!n->connected) return fail(n, SPICE_ESTATE, "PEER exchange: call spice_peer_connect first");
    if (!ms || cap < 4) return fail(n, SPICE_EINVAL, "need room for 4 timings");
    cudaStream_t s = n->stream;
    const SimArgs &a = n->args;
    cudaEvent_t e0, e1;
    CU(n, cudaEventCreate(&e0));
    CU(n, cudaEventCreate(&e1));
    double acc[4] = {0, 0, 0, 0};
    uint64_t cnt[4] = {0, 0, 0, 0};
    auto timed = [&](int slot, auto &&fn) -> spice_status {
        CU(n, cudaEventRecord(e0, s));
        spice_status st = fn();
        if (st) return st;
        CU(n, cudaEventRecord(e1, s));
        CU(n, cudaEventSynchronize(e1));
        float x = 0;
        CU(n, cudaEventElapsedTime(&x, e0, e1));
        acc[slot] += x;
        cnt[slot] += 1;
        return SPICE_OK;
    };
    // G > 1 exchange pieces: publish = this rank's arrival flags after an update (PEER);
    // gather = NCCL all-gather or waiting for every rank's flags (PEER), then bitmap->list
    auto publish = [&](uint32_t k) -> spice_status {
        if (n->peer) CU(n, launch_peer_signal(a, k, s));
        return SPICE_OK;
    };
    auto gather = [&]() -> spice_status {
        if (n->peer) CU(n, launch_peer_wait(a, 0, s));
        else {
            ncclResult_t r = nccl().AllGather(n->sendbuf, n->gather, n->W, ncclUint32, n->comm, s);
            if (r != ncclSuccess) return fail(n, SPICE_ENCCL, "ncclAllGather: %s", nccl().GetErrorString(r));
        }
        CU(n, launch_bitmap_to_list(a, 0, s));
        return SPICE_OK;
    };
    // (1) unfused steps: update, [exchange], deliver
    for (uint64_t q = 0; q < steps; ++q) {
        spice_status st = timed(0, [&]() -> spice_status { CU(n, launch_update(a, 0, s)); return SPICE_OK; });
        if (st) return st;
        if (n->G > 1) {
            if ((st = publish(0))) return st;
            st = timed(3, gather);
            if (st) return st;
        }
        st = timed(1, [&]() -> spice_status { CU(n, launch_deliver(a, 0, n->global_atomics, n->n_sm, s)); return SPICE_OK; });
        if (st) return st;
        CU(n, launch_advance(n->t0, 1, s));
        n->t_host += 1;
    }
    // (2s) small networks: the one-CTA step kernel, one step per launch ("fused" slot)
    if (n->small && steps > 0) {
        for (uint64_t q = 0; q < steps; ++q) {
            spice_status st = timed(2, [&]() -> spice_status { CU(n, launch_small(a, 0, 1, s)); return SPICE_OK; });
            if (st) return st;
            CU(n, launch_advance(n->t0, 1, s));
            n->t_host += 1;
        }
    }
    // (2) the fused kernel (G = 1): update(t), then fused launches deliver(t)+update(t+1)
    if (!n->small && n->G == 1 && n->fused && !n->global_atomics && steps > 0) {
        CU(n, launch_update(a, 0, s));
        for (uint64_t q = 0; q < steps; ++q) {
            spice_status st = timed(2, [&]() -> spice_status { CU(n, launch_fused(a, 0, s)); return SPICE_OK; });
            if (st) return st;
            CU(n, launch_advance(n->t0, 1, s));
            n->t_host += 1;
        }
        CU(n, launch_deliver(a, 0, false, n->n_sm, s));
        CU(n, launch_advance(n->t0, 1, s));
        n->t_host += 1;
    }
    // (2') G > 1: update(0), then all-gather + bitmap->list (exchange) and the fused kernel
    if (n->G > 1 && !n->external && n->fused && !n->global_atomics && steps > 0) {
        CU(n, launch_update(a, 0, s));
        spice_status st0 = publish(0);
        if (st0) return st0;
        for (uint64_t q = 0; q < steps; ++q) {
            spice_status st = timed(3, gather);
            if (st) return st;
            st = timed(2, [&]() -> spice_status { CU(n, launch_fused(a, 0, s)); return SPICE_OK; });
            if (st) return st;
            if ((st = publish(1))) return st;                // (step t + 1's bitmap, before the advance)
            CU(n, launch_advance(n->t0, 1, s));
            n->t_host += 1;
        }
        if ((st0 = gather())) return st0;
        CU(n, launch_deliver(a, 0, false, n->n_sm, s));
        CU(n, launch_advance(n->t0, 1, s));
        n->t_host += 1;
    }
    // (3) the fused kernel as the timed region runs it: a captured graph of kProf back-to-
    //     back fused launches (the steady state), replayed and timed with events
    double in_graph = 0.0;
    if (cap >= 5 && n->G == 1 && n->fused && !n->global_atomics && steps > 0) {
        constexpr uint32_t kProf = 32;
        if (!n->small) CU(n, launch_update(a, 0, s));
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        CU(n, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        if (n->small) launch_small(a, 0, kProf, s);       // (per step: the chunk's time / kProf)
        else if (a.persist) launch_run(a, 0, kProf, s);   // (persistent: the launch's time / kProf)
        else for (uint32_t k = 0; k < kProf; ++k) launch_fused(a, k, s);
        launch_advance(n->t0, kProf, s, n->gbar);
        CU(n, cudaStreamEndCapture(s, &g));
        cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) return fail(n, SPICE_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
        const uint64_t reps = std::max<uint64_t>(1, steps / kProf);
        CU(n, cudaGraphLaunch(ge, s));                       // warm
        CU(n, cudaEventRecord(e0, s));
        for (uint64_t r = 0; r < reps; ++r) CU(n, cudaGraphLaunch(ge, s));
        CU(n, cudaEventRecord(e1, s));
        CU(n, cudaEventSynchronize(e1));
        float x = 0;
        CU(n, cudaEventElapsedTime(&x, e0, e1));
        in_graph = x / (double)(reps * kProf);
        cudaGraphExecDestroy(ge);
        n->t_host += (reps + 1) * kProf;
        if (!n->small) {                                   // close the fused sequence
            CU(n, launch_deliver(a, 0, false, n->n_sm, s));
            CU(n, launch_advance(n->t0, 1, s));
            n->t_host += 1;
        }
    }
    CU(n, cudaStreamSynchronize(s));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (int k = 0; k < 4; ++k) ms[k] = cnt[k] ? acc[k] / (double)cnt[k] : 0.0;
    if (cap >= 5) ms[4] = in_graph;
    if (nk) *nk = cap >= 5 ? 5 : 4;
    return SPICE_OK;
}

spice_status spice_debug_phases(spice_net *n, uint64_t *out, uint64_t cap, uint64_t *count) {
    CHECK_NET(n);
    const uint64_t m = n->ptimes ? (uint64_t)n->NT * n->C * 16 : 0;
    if (count) *count = m;
    if (!m) return SPICE_OK;
    if (!out || cap < m) return fail(n, SPICE_ETRUNC, "need %llu values", (unsigned long long)m);
    CU(n, cudaStreamSynchronize(n->stream));
    CU(n, cudaMemcpy(out, n->ptimes, m * 8, cudaMemcpyDeviceToHost));
    return SPICE_OK;
}

uint64_t spice_launches(spice_net *n, uint64_t steps) {
    if (!n) return 0;
    uint64_t total = 0;
    while (steps) {                                        // the decomposition spice_step uses
        uint32_t k = spice_net::kGraphLevels - 1;
        while ((1ull << k) > steps) --k;
        const uint64_t m = 1ull << k;
        if (n->small) total += 2;                          // k_small + k_advance per replay
        else if (n->args.persist) total += m > 1 ? 4 : 3;  // update, persistent steps, deliver, advance
        else {
            // + one k_advance per replay; the fused sequences open with an update (G = 1 and
            // G > 1) and close with a plain delivery
            total += spice_kernels_per_step(n) * m + 1 + (n->fused && !n->global_atomics ? 1 : 0);
        }
        steps -= m;
    }
    return total;
}

uint32_t spice_kernels_per_step(spice_net *n) {
    if (!n) return 0;
    if (n->G == 1 && n->fused && !n->global_atomics) return 1u;   // fused deliver(t)+update(t+1)
    const uint32_t px = n->peer ? 2u : 0u;                        // PEER: flag signal + wait kernels
    if (n->G > 1 && n->fused && !n->global_atomics) return 2u + px;   // bitmap_to_list, fused (+ NCCL's)
    return n->G == 1 ? 2u : 3u + px;   // update, [bitmap_to_list], deliver (+ NCCL's own kernel)
}

spice_status spice_free(spice_net *n) {
    if (!n) return SPICE_OK;
    destroy(n);
    return SPICE_OK;
}

}  // extern "C"
