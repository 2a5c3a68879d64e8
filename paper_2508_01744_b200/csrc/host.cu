// host.cu — the C-ABI entry points of include/agft.h: validation, workspace layout,
// launches, status codes.  No device allocation happens here: every device buffer
// is the caller's.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <new>
#include <vector>

#include "agft_internal.cuh"

using namespace agft;

struct agft_handle_s {
    agft_config cfg;
    Layout layout;
    Ws ws;
    cudaStream_t stream;
    cudaStream_t side[kNumCls];   // one stream per kernel class: classes of a sub-chunk overlap
    cudaEvent_t fork, join[kNumCls];
    uint32_t t;             // current global step (observe/apply alternate strictly)
    uint32_t sweep_t;       // next window of the offline sweep (ENV.md §5 accumulation order)
    uint32_t live_pending;  // 1 between agft_select and its agft_observe
    agft_status sticky;     // AGFT_OK or AGFT_E_CUDA
    // agft_profile_*: per-class launch events (timed, on the class's stream) while profiling is on
    struct ProfEv {
        int cls;
        cudaEvent_t a, b;
    };
    bool prof_on, prof_serial;
    std::vector<ProfEv> prof_ev;
    size_t prof_used;
    // agft_timeline: per-warp records of the replay-class launches (null = off)
    unsigned long long *tl = nullptr;
    uint64_t tl_cap = 0;
    uint32_t tl_seq = 0;
};

namespace agft {
static std::atomic<uint64_t> g_launches{0};
void note_launches(uint32_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace agft

namespace {

bool finite(double v) { return std::isfinite(v); }

// Sub-chunk length between re-classifications: short while the action spaces are still
// collapsing (most tuners reach K_act ≤ 32 within ~1,000 windows and K_act = 1 within
// ~1,400), long once the classes are stable.
uint32_t env_u32(const char *name, uint32_t def)
{
    const char *e = std::getenv(name);
    const long v = e ? std::atol(e) : 0;
    return v > 0 ? (uint32_t)v : def;
}

uint32_t sub_chunk(uint32_t t)
{
    // (round 2: 128 / 512 instead of 256 / 1,024 — +0.7% on the C4 day, profiles/r02_subchunk_ab/)
    static const uint32_t early = env_u32("AGFT_SUB_EARLY", 128), mid = env_u32("AGFT_SUB_MID", 512),
                          late = env_u32("AGFT_SUB_LATE", 4096);
    if (t < 2048) return early;
    if (t < 8192) return mid;
    return late;
}

cudaError_t launch_seg(const ReplayArgs &a, uint32_t D, int G, cudaStream_t s) { return launch_seg2(a, D, G, s); }

bool stream_prio_enabled()
{
    const char *e = std::getenv("AGFT_STREAM_PRIO");
    return !(e && e[0] == '0');
}

// rank[c] = position of class c in the priority order (0 = highest)
void prio_order(int (&rank)[kNumCls])
{
    // (round 2: the classes whose warps run longest first — G = 4, G = 32, WIDE, then G = 8, G = 16, SOLO;
    // +2% on the C4 day over the round-1 order 2,1,3,0,5,4; profiles/r02_prio_ab/)
    static const int def[kNumCls] = {kClsSeg8, kClsSeg64, kClsWide, kClsSeg16, kClsSeg32, kClsSolo};
    int order[kNumCls];
    for (int i = 0; i < kNumCls; ++i) order[i] = def[i];
    if (const char *e = std::getenv("AGFT_PRIO_ORDER")) {
        int n = 0, v = 0;
        bool any = false;
        for (const char *q = e;; ++q) {
            if (*q >= '0' && *q <= '9') { v = v * 10 + (*q - '0'); any = true; continue; }
            if (any && n < kNumCls && v < kNumCls) order[n++] = v;
            v = 0; any = false;
            if (!*q) break;
        }
    }
    for (int c = 0; c < kNumCls; ++c) rank[c] = kNumCls - 1;
    for (int i = kNumCls - 1; i >= 0; --i) rank[order[i]] = i;
}

void destroy_streams(agft_handle h)
{
    for (int c = 0; c < kNumCls; ++c) {
        if (h->side[c]) cudaStreamDestroy(h->side[c]);
        if (h->join[c]) cudaEventDestroy(h->join[c]);
    }
    if (h->fork) cudaEventDestroy(h->fork);
}

// Class streams by priority: the classes whose warps run longest get the SMs first, so the short
// classes pack around them (A/B).  AGFT_STREAM_PRIO=0 disables; AGFT_PRIO_ORDER="3,5,0,2,1,4"
// overrides the order (class ids of agft_internal.cuh, highest priority first).
cudaError_t create_streams(agft_handle h)
{
    cudaError_t e = cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming);
    int prio_lo = 0, prio_hi = 0;
    const bool prio = stream_prio_enabled() && cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi) == cudaSuccess;
    int rank[kNumCls];
    prio_order(rank);
    for (int c = 0; c < kNumCls && e == cudaSuccess; ++c) {
        int p = prio_lo;
        if (prio) {
            p = prio_hi + rank[c];
            if (p > prio_lo) p = prio_lo;
        }
        e = cudaStreamCreateWithPriority(&h->side[c], cudaStreamNonBlocking, p);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->join[c], cudaEventDisableTiming);
    }
    return e;
}

agft_status validate(const agft_config *c)
{
    if (!c) return AGFT_E_INVALID_ARG;
    if (c->abi_version != AGFT_ABI_VERSION) return AGFT_E_INVALID_ARG;
    if (c->n_tuners == 0 || c->n_traces == 0) return AGFT_E_INVALID_ARG;
    if (c->kernel_policy > AGFT_POLICY_WIDE) return AGFT_E_INVALID_ARG;
    const agft_grid &g = c->grid;
    if (g.n_arms == 0) return AGFT_E_EMPTY_ARMS;
    if (g.f_step_mhz == 0 || g.n_arms > AGFT_MAX_ARMS || g.f_min_mhz == 0) return AGFT_E_INVALID_GRID;
    if ((uint64_t)g.f_min_mhz + (uint64_t)(g.n_arms - 1) * g.f_step_mhz > g.f_max_hw_mhz) return AGFT_E_INVALID_GRID;
    if (c->d < 1 || c->d > AGFT_MAX_D) return AGFT_E_DIM;
    for (int i = 0; i < 7; ++i)
        if (!finite(c->norm_lo[i]) || !finite(c->norm_hi[i]) || c->norm_lo[i] > c->norm_hi[i]) return AGFT_E_NONFINITE;
    const agft_policy &p = c->policy;
    if (!finite(p.tau) || p.tau <= 0 || !finite(p.clip_lo) || !finite(p.clip_hi) || p.clip_lo > p.clip_hi ||
        !finite(p.tie_rel) || p.tie_rel < 0)
        return AGFT_E_NONFINITE;
    if (p.median_window < 1 || p.median_window > AGFT_MAX_WINDOW) return AGFT_E_INVALID_ARG;
    const agft_refine &rf = c->refine;               // ENV.md §4.11
    if (rf.enable > 1u) return AGFT_E_INVALID_ARG;
    if (rf.enable && (rf.period < 1u || rf.step_mhz < 1u)) return AGFT_E_INVALID_ARG;
    if (c->closed.enable > 2u) return AGFT_E_INVALID_ARG;   // 1: ENV-C (ENV.md §6), 2: ENV-S (§7)
    const agft_phase &ph = c->phase;                 // ENV.md §4.10
    if (ph.enable > 1u) return AGFT_E_INVALID_ARG;
    if (ph.enable && (ph.window < 1u || !finite(ph.delta) || !finite(ph.lambda) || ph.delta < 0 || ph.lambda < 0))
        return ph.window < 1u ? AGFT_E_INVALID_ARG : AGFT_E_NONFINITE;
    const agft_env &e = c->env;
    const double ev[] = {e.window_s, e.p_idle, e.k_lin, e.k_cube, e.u_floor, e.u_max, e.c_prefill,
                         e.c_decode, e.beta, e.sigma_e, e.sigma_t};
    for (double v : ev)
        if (!finite(v) || v < 0) return AGFT_E_NONFINITE;
    if (e.window_s <= 0 || e.u_max <= 0 || e.u_max >= 1 || e.sigma_e >= 1 || e.sigma_t >= 1 || e.c_decode <= 0 ||
        e.beta > 1)
        return AGFT_E_NONFINITE;
    const agft_trace_cfg &t = c->trace;
    if (t.seg_steps == 0 || t.steps_per_hour == 0 || t.burst_steps == 0 || t.cap == 0 || t.kv_total == 0 ||
        t.pattern_mode > 4)
        return AGFT_E_INVALID_ARG;
    if (!finite(t.lambda0) || t.lambda0 < 0 || !finite(t.t_iter0) || t.t_iter0 <= 0 || !finite(t.t_iter1) ||
        t.t_iter1 < 0 || !finite(t.e2e0) || !finite(t.tau_ref) || !finite(t.burst_mult))
        return AGFT_E_NONFINITE;
    uint32_t wsum = 0;
    for (int i = 0; i < 5; ++i) {
        wsum += t.weight[i];
        if (t.ctx_hi[i] < t.ctx_lo[i] || t.gen_hi[i] < t.gen_lo[i]) return AGFT_E_INVALID_ARG;
        if (!finite(t.conc_mult[i]) || t.conc_mult[i] < 0 || !finite(t.hit_rate[i]) || t.hit_rate[i] < 0 ||
            t.hit_rate[i] > 1)
            return AGFT_E_NONFINITE;
    }
    if (wsum != 256) return AGFT_E_INVALID_ARG;
    for (int i = 0; i < 24; ++i)
        if (!finite(t.knot[i]) || t.knot[i] < 0) return AGFT_E_NONFINITE;
    if (!finite(c->prune.cascade_fraction) || c->prune.cascade_fraction <= 0 || c->prune.cascade_fraction > 1)
        return AGFT_E_NONFINITE;
    return AGFT_OK;
}

// Per-tuner parameters: every index the kernels derive from them must be in range —
// trace_id selects a trace's records / raw rows, record_slot a row of d_traj / d_gap — and the
// sweep values must be finite (α0 ≥ 0, k_h ≥ 0).  Host copy of the array.
agft_status validate_params(const agft_config *c, const agft_tuner_params *p)
{
    for (uint32_t i = 0; i < c->n_tuners; ++i) {
        const agft_tuner_params &q = p[i];
        if (q.trace_id >= c->n_traces) return AGFT_E_INVALID_ARG;
        if (q.record_slot != AGFT_NO_RECORD && q.record_slot >= c->record_slots) return AGFT_E_INVALID_ARG;
        if (!finite(q.alpha0) || q.alpha0 < 0 || !finite(q.extreme_reward_threshold) || !finite(q.historical_k) ||
            q.historical_k < 0)
            return AGFT_E_INVALID_ARG;
    }
    return AGFT_OK;
}

// the workspace must live on the current device (kernels and side streams are created there)
agft_status check_device_ptr(const void *d_ptr, int dev)
{
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, d_ptr) != cudaSuccess) {
        cudaGetLastError();
        return AGFT_E_INVALID_ARG;
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return AGFT_E_INVALID_ARG;
    if (at.type == cudaMemoryTypeDevice && at.device != dev) return AGFT_E_DEVICE;
    return AGFT_OK;
}

// copy a device array of n agft_tuner_params to the host and validate it
agft_status validate_device_params(const agft_config *c, const agft_tuner_params *d_params, cudaStream_t s)
{
    agft_tuner_params *hp = static_cast<agft_tuner_params *>(std::malloc(sizeof(agft_tuner_params) * c->n_tuners));
    if (!hp) return AGFT_E_INVALID_ARG;
    agft_status st = AGFT_OK;
    if (cudaMemcpyAsync(hp, d_params, sizeof(agft_tuner_params) * c->n_tuners, cudaMemcpyDeviceToHost, s) !=
            cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        cudaGetLastError();
        st = AGFT_E_CUDA;
    }
    if (st == AGFT_OK) st = validate_params(c, hp);
    std::free(hp);
    return st;
}

agft_status cuda_status(agft_handle h, cudaError_t e)
{
    if (e == cudaSuccess) return AGFT_OK;
    if (h) h->sticky = AGFT_E_CUDA;
    return AGFT_E_CUDA;
}

ReplayArgs replay_args(agft_handle h, const void *records, uint32_t t0, uint32_t n_steps)
{
    const agft_config &c = h->cfg;
    ReplayArgs a{};
    std::memset(&a, 0, sizeof(a));
    a.w = h->ws;
    a.records = static_cast<const StepRec *>(records);
    a.n_tuners = c.n_tuners;
    a.K = c.grid.n_arms;
    a.n_traces = c.n_traces;
    a.t0 = t0;
    a.n_steps = n_steps;
    a.rec_stride = n_steps;
    a.rec_off = 0;
    a.median_window = c.policy.median_window;
    a.record_slots = c.record_slots;
    a.prune_enable = c.prune.enable;
    a.ext_L = c.prune.extreme_round_limit;
    a.ext_n = c.prune.extreme_min_samples;
    a.hist_t = c.prune.historical_min_round;
    a.hist_n = c.prune.historical_min_samples;
    a.f_min_mhz = c.grid.f_min_mhz;
    a.f_step_mhz = c.grid.f_step_mhz;
    a.tau = c.policy.tau;
    a.clip_lo = c.policy.clip_lo;
    a.clip_hi = c.policy.clip_hi;
    a.tie_rel = c.policy.tie_rel;
    a.ph_enable = c.phase.enable;
    a.ph_window = c.phase.window;
    a.ph_delta = c.phase.delta;
    a.ph_lambda = c.phase.lambda;
    a.rf_enable = c.refine.enable;
    a.rf_period = c.refine.period;
    a.rf_mature = c.refine.mature;
    a.rf_min_samples = c.refine.min_samples;
    a.rf_half_mhz = c.refine.half_mhz;
    a.rf_step_mhz = c.refine.step_mhz;
    // ENV.md §4.8: (double)F_k < cascade_fraction * (double)f_max_hw — one IEEE product
    volatile double cf = c.prune.cascade_fraction;
    a.cascade_limit = cf * (double)c.grid.f_max_hw_mhz;
    a.W = c.env.window_s;
    a.p_idle = c.env.p_idle;
    a.u_floor = c.env.u_floor;
    a.u_max = c.env.u_max;
    a.kv_total = c.trace.kv_total;
    a.cl_enable = c.closed.enable;
    a.cl_q_max = c.closed.q_max;
    a.cap = c.trace.cap;
    a.tc = c.trace;                                   // ENV-S arrivals (ENV.md §7)
    a.seed = c.env_seed;
    a.trace_base = c.trace_base;
    std::memcpy(a.norm_lo, c.norm_lo, sizeof(a.norm_lo));
    std::memcpy(a.norm_hi, c.norm_hi, sizeof(a.norm_hi));
    return a;
}

}  // namespace

extern "C" {

agft_status agft_validate(const agft_config *cfg) { return validate(cfg); }

uint32_t agft_struct_size(int which)
{
    switch (which) {
    case 0: return (uint32_t)sizeof(agft_config);
    case 1: return (uint32_t)sizeof(agft_tuner_params);
    case 2: return (uint32_t)sizeof(agft_tuner_stats);
    default: return 0;
    }
}

size_t agft_workspace_bytes(const agft_config *cfg)
{
    if (validate(cfg) != AGFT_OK) return 0;
    return make_layout(cfg->n_tuners, cfg->d, cfg->closed.enable == 2u).total;
}

agft_status agft_create(const agft_config *cfg, const agft_tuner_params *d_params, void *d_workspace,
                        size_t ws_bytes, void *stream, agft_handle *out)
{
    if (!out) return AGFT_E_INVALID_ARG;
    *out = nullptr;
    agft_status st = validate(cfg);
    if (st != AGFT_OK) return st;
    if (!d_params || !d_workspace) return AGFT_E_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(d_workspace) % 256 != 0) return AGFT_E_WORKSPACE;
    const Layout L = make_layout(cfg->n_tuners, cfg->d, cfg->closed.enable == 2u);
    if (ws_bytes < L.total) return AGFT_E_WORKSPACE;

    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return AGFT_E_DEVICE;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return AGFT_E_DEVICE;
    if (major != 10) return AGFT_E_DEVICE;
    if ((st = check_device_ptr(d_workspace, dev)) != AGFT_OK) return st;
    if ((st = check_device_ptr(d_params, dev)) != AGFT_OK) return st;
    if ((st = validate_device_params(cfg, d_params, static_cast<cudaStream_t>(stream))) != AGFT_OK) return st;

    agft_handle h = new (std::nothrow) agft_handle_s;
    if (!h) return AGFT_E_INVALID_ARG;
    h->cfg = *cfg;
    h->layout = L;
    h->ws = make_ws(d_workspace, L);
    h->stream = static_cast<cudaStream_t>(stream);
    h->t = 0;
    h->sweep_t = 0;
    h->live_pending = 0;
    h->sticky = AGFT_OK;
    h->prof_on = false;
    h->prof_serial = false;
    h->prof_used = 0;
    h->tl = nullptr;
    h->tl_cap = 0;
    h->tl_seq = 0;
    h->fork = nullptr;
    for (int c = 0; c < kNumCls; ++c) {
        h->side[c] = nullptr;
        h->join[c] = nullptr;
    }

    cudaError_t e = create_streams(h);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(h->ws.params, d_params, sizeof(agft_tuner_params) * cfg->n_tuners,
                            cudaMemcpyDeviceToDevice, h->stream);
    if (e == cudaSuccess) e = launch_init(h->ws, *cfg, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
        destroy_streams(h);
        delete h;
        return AGFT_E_CUDA;
    }
    *out = h;
    return AGFT_OK;
}

agft_status agft_attach(const agft_config *cfg, void *d_workspace, size_t ws_bytes, void *stream, uint32_t t,
                        uint32_t sweep_t, agft_handle *out)
{
    if (!out) return AGFT_E_INVALID_ARG;
    *out = nullptr;
    agft_status st = validate(cfg);
    if (st != AGFT_OK) return st;
    if (!d_workspace) return AGFT_E_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(d_workspace) % 256 != 0) return AGFT_E_WORKSPACE;
    const Layout L = make_layout(cfg->n_tuners, cfg->d, cfg->closed.enable == 2u);
    if (ws_bytes < L.total) return AGFT_E_WORKSPACE;
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return AGFT_E_DEVICE;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return AGFT_E_DEVICE;
    if (major != 10) return AGFT_E_DEVICE;
    if ((st = check_device_ptr(d_workspace, dev)) != AGFT_OK) return st;
    // the tuner parameters come from the restored workspace: validated like agft_create's
    if ((st = validate_device_params(cfg, make_ws(d_workspace, L).params, static_cast<cudaStream_t>(stream))) !=
        AGFT_OK)
        return st;
    agft_handle h = new (std::nothrow) agft_handle_s;
    if (!h) return AGFT_E_INVALID_ARG;
    h->cfg = *cfg;
    h->layout = L;
    h->ws = make_ws(d_workspace, L);
    h->stream = static_cast<cudaStream_t>(stream);
    h->t = t;
    h->sweep_t = sweep_t;
    h->live_pending = 0;
    h->sticky = AGFT_OK;
    h->prof_on = false;
    h->prof_serial = false;
    h->prof_used = 0;
    h->tl = nullptr;
    h->tl_cap = 0;
    h->tl_seq = 0;
    h->fork = nullptr;
    for (int c = 0; c < kNumCls; ++c) {
        h->side[c] = nullptr;
        h->join[c] = nullptr;
    }
    if (create_streams(h) != cudaSuccess) {
        destroy_streams(h);
        delete h;
        return AGFT_E_CUDA;
    }
    *out = h;
    return AGFT_OK;
}

agft_status agft_reset(agft_handle h)
{
    if (!h) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    agft_status st = cuda_status(h, launch_init(h->ws, h->cfg, h->stream));
    if (st == AGFT_OK) {
        h->t = 0;
        h->sweep_t = 0;
        h->live_pending = 0;
    }
    return st;
}

agft_status agft_trace_generate(agft_handle h, uint32_t t0, uint32_t n_steps, void *d_records, uint32_t *d_raw)
{
    if (!h || !d_records) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    const agft_config &c = h->cfg;
    TraceArgs a;
    std::memset(&a, 0, sizeof(a));
    a.tc = c.trace;
    a.env = c.env;
    std::memcpy(a.norm_lo, c.norm_lo, sizeof(a.norm_lo));
    std::memcpy(a.norm_hi, c.norm_hi, sizeof(a.norm_hi));
    a.seed = c.env_seed;
    a.trace_base = c.trace_base;
    a.n_traces = c.n_traces;
    a.t0 = t0;
    a.n_steps = n_steps;
    a.cap = c.trace.cap;
    a.f_max_hw_mhz = c.grid.f_max_hw_mhz;
    a.envc = h->ws.env;
    a.records = static_cast<StepRec *>(d_records);
    a.raw = d_raw;
    return cuda_status(h, launch_trace(a, h->stream));
}

constexpr int kProfClassify = 6, kProfRefine = 7;   // agft_profile slots after the kernel classes

// agft_profile_*: a timed event pair around one launch of class cls on stream st (no-op when off)
static cudaError_t prof_begin(agft_handle h, int cls, cudaStream_t st, ReplayArgs *a)
{
    if (!h->prof_on) return cudaSuccess;
    if (a) {
        a->prof = h->ws.prof;
        a->prof_cls = (uint32_t)cls;
    }
    if (h->prof_used == h->prof_ev.size()) {
        agft_handle_s::ProfEv ev{cls, nullptr, nullptr};
        cudaError_t e = cudaEventCreate(&ev.a);
        if (e == cudaSuccess) e = cudaEventCreate(&ev.b);
        if (e != cudaSuccess) return e;
        h->prof_ev.push_back(ev);
    }
    h->prof_ev[h->prof_used].cls = cls;
    return cudaEventRecord(h->prof_ev[h->prof_used].a, st);
}
static cudaError_t prof_end(agft_handle h, cudaStream_t st)
{
    if (!h->prof_on) return cudaSuccess;
    return cudaEventRecord(h->prof_ev[h->prof_used++].b, st);
}

// The replay scheduler: steps [t0, t0+n) in sub-chunks; before each sub-chunk every tuner
// is classified by its active-arm count and each class runs its kernel on its own stream.
static agft_status run_steps(agft_handle h, const void *d_records, uint32_t t0, uint32_t n, uint8_t *traj,
                             double *gap, uint32_t *chosen, const uint32_t *raw = nullptr)
{
    const agft_config &c = h->cfg;
    // frozen tuners are not scheduled (or return early): their d_chosen entry reads AGFT_NEVER
    if (chosen) {
        const cudaError_t e = cudaMemsetAsync(chosen, 0xFF, sizeof(uint32_t) * c.n_tuners, h->stream);
        if (e != cudaSuccess) return cuda_status(h, e);
    }
    for (uint32_t s = 0; s < n;) {
        const uint32_t t = t0 + s;
        uint32_t len = sub_chunk(t);
        if (len > n - s) len = n - s;
        else if (n - s - len < len / 2) len = n - s;   // absorb a short tail: one launch wave-tail less (A/B −2%)
        // refinement on the class schedule (ENV.md §4.11): sub-chunks end at the refinement points
        // ((t + 1) % period == 0), where a separate pass re-windows every tuner's action space;
        // the phase-triggered refinements and the closed loop keep the WIDE schedule
        const bool defer = c.refine.enable && !c.phase.enable && !c.closed.enable &&
                           c.kernel_policy != AGFT_POLICY_WIDE;
        if (defer) {
            const uint32_t to_point = c.refine.period - (t % c.refine.period);
            if (len > to_point) len = to_point;
        }
        ReplayArgs a = replay_args(h, d_records, t, len);
        a.tl = h->tl;
        a.tl_cap = (uint32_t)(h->tl_cap < 0xffffffffu ? h->tl_cap : 0xffffffffu);
        a.tl_seq = h->tl_seq;
        a.rec_stride = n;
        a.rec_off = s;
        a.rf_defer = defer ? 1u : 0u;
        a.traj = c.record_slots ? traj : nullptr;
        a.gap = c.record_slots ? gap : nullptr;
        a.chosen = chosen;
        a.raw = raw;
        cudaError_t e = cudaSuccess;
        // refinement re-admits arms, so a tuner's class can grow: without the deferred pass, one
        // warp per tuner throughout
        // (ENV-S servers, closed.enable = 2, run on the WIDE mapping: a warp per tuner drives its server)
        if (c.kernel_policy == AGFT_POLICY_WIDE || (c.refine.enable && !defer) || c.closed.enable == 2u) {
            ++h->tl_seq;
            e = prof_begin(h, kClsWide, h->stream, &a);
            if (e == cudaSuccess) e = launch_replay(a, c.d, h->stream);
            if (e == cudaSuccess) e = prof_end(h, h->stream);
        } else {
            e = prof_begin(h, kProfClassify, h->stream, nullptr);
            if (e == cudaSuccess) e = launch_classify(h->ws, c.n_tuners, h->stream);
            if (e == cudaSuccess) e = prof_end(h, h->stream);
            if (e == cudaSuccess) e = cudaEventRecord(h->fork, h->stream);
            for (int k = 0; k < kNumCls && e == cudaSuccess; ++k) {
                ReplayArgs ak = a;
                ak.list = h->ws.lists + (size_t)k * c.n_tuners;
                ak.count = h->ws.counts + k;
                ak.tl_cls = (uint32_t)k;
                ak.tl_seq = h->tl_seq++;
                // agft_profile_start(h, 1): every class alone on the handle's stream (per-kernel times)
                const cudaStream_t sk = h->prof_on && h->prof_serial ? h->stream : h->side[k];
                if (sk != h->stream) e = cudaStreamWaitEvent(sk, h->fork, 0);
                if (e == cudaSuccess) e = prof_begin(h, k, sk, &ak);
                if (e != cudaSuccess) break;
                switch (k) {
                case kClsWide: e = launch_replay(ak, c.d, sk); break;
                case kClsSeg32: e = launch_seg(ak, c.d, 16, sk); break;
                case kClsSeg16: e = launch_seg(ak, c.d, 8, sk); break;
                case kClsSeg8: e = launch_seg(ak, c.d, 4, sk); break;
                case kClsSeg64: e = launch_seg(ak, c.d, 32, sk); break;
                default: e = launch_solo(ak, c.d, sk); break;
                }
                if (e == cudaSuccess) e = prof_end(h, sk);
                if (sk == h->stream) continue;
                if (e == cudaSuccess) e = cudaEventRecord(h->join[k], sk);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, h->join[k], 0);
            }
        }
        if (e == cudaSuccess && defer && (t + len) % c.refine.period == 0u) {
            ReplayArgs r = replay_args(h, d_records, t + len - 1, 1);   // as of the sub-chunk's last step
            r.rec_stride = n;
            r.rec_off = s + len - 1;
            e = prof_begin(h, kProfRefine, h->stream, nullptr);
            if (e == cudaSuccess) e = launch_refine(r, c.d, h->stream);
            if (e == cudaSuccess) e = prof_end(h, h->stream);
        }
        if (e != cudaSuccess) return cuda_status(h, e);
        s += len;
    }
    return AGFT_OK;
}

agft_status agft_replay(agft_handle h, const void *d_records, uint32_t t0, uint32_t n_steps, uint8_t *d_traj,
                        double *d_gap)
{
    if (!h || !d_records) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    if (h->cfg.closed.enable) return AGFT_E_INVALID_ARG;     // needs the raw rows: agft_replay_raw
    if (t0 != h->t || h->live_pending) return AGFT_E_STATE;
    if (n_steps == 0) return AGFT_OK;
    agft_status st = run_steps(h, d_records, t0, n_steps, d_traj, d_gap, nullptr);
    if (st == AGFT_OK) h->t += n_steps;
    return st;
}

agft_status agft_replay_raw(agft_handle h, const void *d_records, const uint32_t *d_raw, uint32_t t0,
                            uint32_t n_steps, uint8_t *d_traj, double *d_gap)
{
    if (!h || !d_records || !d_raw) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    if (t0 != h->t || h->live_pending) return AGFT_E_STATE;
    if (n_steps == 0) return AGFT_OK;
    agft_status st = run_steps(h, d_records, t0, n_steps, d_traj, d_gap, nullptr, d_raw);
    if (st == AGFT_OK) h->t += n_steps;
    return st;
}

agft_status agft_step(agft_handle h, const void *d_records, uint32_t *d_chosen)
{
    if (!h || !d_records) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    if (h->cfg.closed.enable) return AGFT_E_INVALID_ARG;
    if (h->live_pending) return AGFT_E_STATE;
    agft_status st = run_steps(h, d_records, h->t, 1, nullptr, nullptr, d_chosen);
    if (st == AGFT_OK) h->t += 1;
    return st;
}

// Live two-phase step: one launch each, WIDE mapping (a warp per tuner), whatever the class.
agft_status agft_select(agft_handle h, const uint32_t *d_rows, uint32_t *d_chosen)
{
    if (!h || !d_rows || !d_chosen) return AGFT_E_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(d_rows) % 16 != 0) return AGFT_E_INVALID_ARG;
    if (h->cfg.closed.enable) return AGFT_E_INVALID_ARG;     // a live server is closed-loop by itself
    if (h->sticky != AGFT_OK) return h->sticky;
    if (h->live_pending) return AGFT_E_STATE;
    ReplayArgs a = replay_args(h, nullptr, h->t, 1);
    a.live_rows = d_rows;
    a.chosen = d_chosen;
    agft_status st = cuda_status(h, launch_live(a, h->cfg.d, 1, h->stream));
    if (st == AGFT_OK) h->live_pending = 1;
    return st;
}

agft_status agft_scores(agft_handle h, const uint32_t *d_rows, double *d_scores, uint32_t *d_chosen)
{
    if (!h || !d_rows || !d_scores) return AGFT_E_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(d_rows) % 16 != 0) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    if (h->live_pending) return AGFT_E_STATE;        // the pending record belongs to the select
    ReplayArgs a = replay_args(h, nullptr, h->t, 1);
    a.live_rows = d_rows;
    a.chosen = d_chosen;
    a.scores = d_scores;
    return cuda_status(h, launch_live(a, h->cfg.d, 1, h->stream));
}

agft_status agft_observe(agft_handle h, const double *d_resp)
{
    if (!h || !d_resp) return AGFT_E_INVALID_ARG;
    if (h->cfg.closed.enable) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    if (!h->live_pending) return AGFT_E_STATE;
    ReplayArgs a = replay_args(h, nullptr, h->t, 1);
    a.live_resp = d_resp;
    agft_status st = cuda_status(h, launch_live(a, h->cfg.d, 2, h->stream));
    if (st == AGFT_OK) {
        h->live_pending = 0;
        h->t += 1;
    }
    return st;
}

agft_status agft_stats(agft_handle h, agft_tuner_stats *d_out)
{
    if (!h || !d_out) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    return cuda_status(h, cudaMemcpyAsync(d_out, h->ws.acc, sizeof(agft_tuner_stats) * h->cfg.n_tuners,
                                          cudaMemcpyDeviceToDevice, h->stream));
}

agft_status agft_export_arms(agft_handle h, uint32_t tuner, double *d_ainv_packed, double *d_b, double *d_theta,
                             uint32_t *d_n, double *d_rbar, double *d_ebar, uint32_t *d_active_mask)
{
    if (!h) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    if (tuner >= h->cfg.n_tuners) return AGFT_E_INVALID_ARG;
    return cuda_status(h, launch_export(h->ws, tuner, h->cfg.grid.n_arms, h->cfg.d, d_ainv_packed, d_b, d_theta,
                                        d_n, d_rbar, d_ebar, d_active_mask, h->stream));
}

agft_status agft_sweep(agft_handle h, const void *d_records, uint32_t t0, uint32_t n_steps, double *d_S,
                       double *d_SP, uint32_t *d_NP, double *d_O, uint8_t *d_best)
{
    if (!h || !d_records || !d_S || !d_SP || !d_NP || !d_O) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    if (t0 != h->sweep_t) return AGFT_E_STATE;
    agft_status st = cuda_status(h, launch_sweep(h->ws, h->cfg, d_records, t0, n_steps, d_S, d_SP, d_NP, d_O,
                                                 d_best, h->stream));
    if (st == AGFT_OK) h->sweep_t += n_steps;
    return st;
}

agft_status agft_regret(agft_handle h, const double *d_S, const double *d_SP, const uint32_t *d_NP,
                        const double *d_O, uint8_t *d_koff, double *d_regret)
{
    if (!h || !d_S || !d_SP || !d_NP || !d_O || !d_koff) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    // the sweep is open-loop (ENV.md §5): regret against it is defined for open-loop tuners only
    if (h->cfg.closed.enable && d_regret) return AGFT_E_INVALID_ARG;
    return cuda_status(h, launch_regret(h->ws, h->cfg, d_S, d_SP, d_NP, d_O, d_koff, d_regret, h->stream));
}

agft_status agft_get_step(agft_handle h, uint32_t *t)
{
    if (!h || !t) return AGFT_E_INVALID_ARG;
    *t = h->t;
    return AGFT_OK;
}

agft_status agft_get_counters(agft_handle h, uint32_t *t, uint32_t *sweep_t, uint32_t *live_pending)
{
    if (!h) return AGFT_E_INVALID_ARG;
    if (t) *t = h->t;
    if (sweep_t) *sweep_t = h->sweep_t;
    if (live_pending) *live_pending = h->live_pending;
    return AGFT_OK;
}

agft_status agft_run(const agft_config *cfg, const agft_tuner_params *h_params, agft_tuner_params *d_params_buf,
                     uint32_t n_steps, uint32_t chunk_steps, void *d_workspace, size_t ws_bytes, void *d_scratch,
                     size_t scratch_bytes, agft_tuner_stats *d_stats_buf, agft_tuner_stats *h_stats, void *stream)
{
    agft_status st = validate(cfg);
    if (st != AGFT_OK) return st;
    if (!h_params || !d_params_buf || !d_scratch || !d_stats_buf || !h_stats || chunk_steps == 0)
        return AGFT_E_INVALID_ARG;
    if ((st = validate_params(cfg, h_params)) != AGFT_OK) return st;
    const size_t rec_bytes = (size_t)cfg->n_traces * chunk_steps * AGFT_RECORD_BYTES;
    const size_t raw_bytes = cfg->closed.enable ? (size_t)cfg->n_traces * chunk_steps * AGFT_ROW_WORDS * 4 : 0;
    if (scratch_bytes < rec_bytes + raw_bytes) return AGFT_E_WORKSPACE;
    uint32_t *d_raw = cfg->closed.enable ? reinterpret_cast<uint32_t *>(static_cast<char *>(d_scratch) + rec_bytes)
                                         : nullptr;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(d_params_buf, h_params, sizeof(agft_tuner_params) * cfg->n_tuners, cudaMemcpyHostToDevice,
                        s) != cudaSuccess)
        return AGFT_E_CUDA;
    agft_handle h = nullptr;
    st = agft_create(cfg, d_params_buf, d_workspace, ws_bytes, stream, &h);
    if (st != AGFT_OK) return st;
    for (uint32_t t0 = 0; t0 < n_steps && st == AGFT_OK; t0 += chunk_steps) {
        const uint32_t n = (n_steps - t0) < chunk_steps ? (n_steps - t0) : chunk_steps;
        st = agft_trace_generate(h, t0, n, d_scratch, d_raw);
        if (st == AGFT_OK)
            st = d_raw ? agft_replay_raw(h, d_scratch, d_raw, t0, n, nullptr, nullptr)
                       : agft_replay(h, d_scratch, t0, n, nullptr, nullptr);
    }
    if (st == AGFT_OK) st = agft_stats(h, d_stats_buf);
    if (st == AGFT_OK &&
        cudaMemcpyAsync(h_stats, d_stats_buf, sizeof(agft_tuner_stats) * cfg->n_tuners, cudaMemcpyDeviceToHost,
                        s) != cudaSuccess)
        st = AGFT_E_CUDA;
    if (st == AGFT_OK && cudaStreamSynchronize(s) != cudaSuccess) st = AGFT_E_CUDA;
    agft_destroy(h);
    return st;
}

agft_status agft_destroy(agft_handle h)
{
    if (!h) return AGFT_E_INVALID_ARG;
    cudaStreamSynchronize(h->stream);
    destroy_streams(h);
    for (auto &ev : h->prof_ev) {
        cudaEventDestroy(ev.a);
        cudaEventDestroy(ev.b);
    }
    delete h;
    return AGFT_OK;
}

agft_status agft_occupancy(const agft_config *cfg, int slot, uint32_t *tuners_per_sm)
{
    if (!tuners_per_sm || slot < 0 || slot > 5) return AGFT_E_INVALID_ARG;
    agft_status st = validate(cfg);
    if (st != AGFT_OK) return st;
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess || major != 10)
        return AGFT_E_DEVICE;
    int v = -1;
    switch (slot) {
    case kClsWide: v = occupancy_wide(cfg->d, cfg->grid.n_arms); break;
    case kClsSeg32: v = occupancy_seg2(cfg->d, 16); break;
    case kClsSeg16: v = occupancy_seg2(cfg->d, 8); break;
    case kClsSeg8: v = occupancy_seg2(cfg->d, 4); break;
    case kClsSeg64: v = occupancy_seg2(cfg->d, 32); break;
    default: v = occupancy_solo(cfg->d); break;
    }
    if (v < 0) {
        cudaGetLastError();
        return AGFT_E_CUDA;
    }
    *tuners_per_sm = (uint32_t)v;
    return AGFT_OK;
}

agft_status agft_profile_start(agft_handle h, int serialize)
{
    if (!h || serialize < 0 || serialize > 1) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    h->prof_on = true;
    h->prof_serial = serialize != 0;
    h->prof_used = 0;
    return cuda_status(h, cudaMemsetAsync(h->ws.prof, 0, 16 * sizeof(unsigned long long), h->stream));
}

agft_status agft_timeline(agft_handle h, void *d_buf, uint64_t cap_records)
{
    if (!h || (d_buf && cap_records == 0) || (d_buf && !AGFT_TIMELINE)) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    h->tl = static_cast<unsigned long long *>(d_buf);
    h->tl_cap = d_buf ? cap_records : 0;
    h->tl_seq = 0;
    if (!d_buf) return AGFT_OK;
    return cuda_status(h, cudaMemsetAsync(d_buf, 0, sizeof(unsigned long long), h->stream));
}

agft_status agft_profile_read(agft_handle h, agft_profile *out)
{
    if (!h || !out) return AGFT_E_INVALID_ARG;
    if (h->sticky != AGFT_OK) return h->sticky;
    std::memset(out, 0, sizeof(*out));
    unsigned long long cnt[16];
    cudaError_t e = cudaMemcpyAsync(cnt, h->ws.prof, sizeof(cnt), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);   // every class stream joins it
    for (size_t i = 0; i < h->prof_used && e == cudaSuccess; ++i) {
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, h->prof_ev[i].a, h->prof_ev[i].b);
        out->kernel_ms[h->prof_ev[i].cls] += ms;
        out->launches[h->prof_ev[i].cls] += 1u;
    }
    if (e != cudaSuccess) return cuda_status(h, e);
    for (int c = 0; c < 8; ++c) {
        out->tuner_steps[c] = cnt[c];
        out->active_arm_steps[c] = cnt[8 + c];
    }
    h->prof_on = false;
    h->prof_used = 0;
    return AGFT_OK;
}

uint64_t agft_kernel_launches(void) { return agft::g_launches.load(std::memory_order_relaxed); }

const char *agft_status_string(agft_status s)
{
    switch (s) {
    case AGFT_OK: return "ok";
    case AGFT_E_INVALID_ARG: return "invalid argument";
    case AGFT_E_INVALID_GRID: return "invalid frequency grid";
    case AGFT_E_EMPTY_ARMS: return "empty arm set";
    case AGFT_E_DIM: return "context dimension out of range";
    case AGFT_E_NONFINITE: return "non-finite or out-of-range coefficient";
    case AGFT_E_WORKSPACE: return "workspace too small or misaligned";
    case AGFT_E_STATE: return "step counter mismatch";
    case AGFT_E_CUDA: return "CUDA error";
    case AGFT_E_DEVICE: return "no sm_100 device";
    default: return "unknown status";
    }
}

}  // extern "C"
