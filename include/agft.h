/*
 * agft.h — C ABI of the B200-native AGFT hot path (ABI version AGFT_ABI_VERSION, below).
 *
 * What it computes: a batched replay of N independent AGFT frequency tuners
 * (arXiv 2508.01744 §4), each a contextual LinUCB bandit over a frequency grid,
 * against a synthetic serving trace and a closed-form latency/power response
 * (ENV.md).  One call advances every tuner by one or many decision windows.
 *
 * Conventions (all entry points):
 *  - Pointers prefixed d_ are DEVICE pointers, h_ are HOST pointers.  Every device
 *    buffer is allocated and owned by the caller (PyTorch); the library never
 *    allocates device memory.  The opaque handle is host memory owned by the library.
 *  - Calls are asynchronous and ordered on the stream given to agft_create (a
 *    cudaStream_t passed as void*).  Only agft_create and agft_run synchronise.
 *  - Errors are returned as negative agft_status codes; nothing is thrown.  A CUDA
 *    error is sticky on the handle (every later call returns AGFT_E_CUDA).
 *  - A handle is not thread-safe (single writer).
 *  - Device-side anomalies never abort: a non-finite EDP or reward sets bit 0 of
 *    the tuner's stats.flags and freezes that tuner; an update that leaves A⁻¹ not positive
 *    definite (xᵀA⁻¹x < 0, or a diagonal entry ≤ 0: a corrupted or numerically broken arm; SPEC
 *    S:207) sets bits 0 and 1 and freezes it (the step that detects it may still be counted).
 *  - Layout and arithmetic of every step follow ENV.md (the contract shared with
 *    the CPU oracle, which is a separate implementation).
 */
#ifndef AGFT_H
#define AGFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AGFT_ABI_VERSION 9u         /* 2: + agft_phase; 3: + agft_refine (and their stats); 4: + agft_select/agft_observe;
                                       5: + agft_closed / agft_replay_raw; 6: MSEG/LANE policies retired;
                                       7: + agft_profile_start / agft_profile_read (workspace +128 B);
                                       8: agft_closed.enable = 2 selects the ENV-S discrete-event server;
                                       9: + agft_timeline */
#define AGFT_MAX_ARMS 128u          /* K ≤ 128 */
#define AGFT_MAX_D 7u               /* the paper's 7-dim context */
#define AGFT_MAX_WINDOW 64u         /* reward-median window, AMB-3 */
#define AGFT_RECORD_BYTES 128u      /* ENV.md §3.2 per-window step record */
#define AGFT_ROW_WORDS 12u          /* ENV.md §2.2 raw trace row (uint32) */
#define AGFT_NO_RECORD 0xFFFFFFFFu  /* agft_tuner_params.record_slot: not recorded */
#define AGFT_POLICY_AUTO 0u         /* re-classify by active-arm count: SOLO (1), SEG<4/8/16/32> (2..64), WIDE (>64) */
#define AGFT_POLICY_WIDE 1u         /* one warp per tuner for every step (reference schedule) */

typedef struct agft_handle_s *agft_handle;

typedef enum {
    AGFT_OK = 0,
    AGFT_E_INVALID_ARG = -1,  /* NULL pointer, zero size, bad enum */
    AGFT_E_INVALID_GRID = -2, /* step = 0, K ∉ [1,128], f_min+(K-1)·step > f_max_hw */
    AGFT_E_EMPTY_ARMS = -3,   /* an empty arm set */
    AGFT_E_DIM = -4,          /* d ∉ [1,7] */
    AGFT_E_NONFINITE = -5,    /* a non-finite or out-of-range coefficient */
    AGFT_E_WORKSPACE = -6,    /* workspace too small or misaligned */
    AGFT_E_STATE = -7,        /* t0 disagrees with the handle's step counter */
    AGFT_E_CUDA = -8,         /* a CUDA launch/runtime error (sticky) */
    AGFT_E_DEVICE = -9        /* no sm_100 device / wrong architecture */
} agft_status;

/* Frequency grid: arm k ↔ f_min + k·step MHz; f_max_hw bounds the grid and
 * sets the cascade threshold. */
typedef struct { uint32_t f_min_mhz, f_step_mhz, n_arms, f_max_hw_mhz; } agft_grid;

/* Pruning, P:387-391 / S:255-258. The per-tuner thresholds (extreme reward
 * threshold, historical k) live in agft_tuner_params (sweep axes). */
typedef struct {
    uint32_t enable, extreme_round_limit, extreme_min_samples, historical_min_round,
             historical_min_samples, pad;
    double cascade_fraction;
} agft_prune;

/* Policy: α_t = α0/√(1+t/τ) (AMB-1), reward = clip(1 − EDP/median, lo, hi) over the
 * last median_window EDPs (AMB-3), near-tie tolerance (ENV.md §4.5). */
typedef struct { double tau, clip_lo, clip_hi, tie_rel; uint32_t median_window, pad; } agft_policy;

/* ENV-R constants (ENV.md §3). */
typedef struct {
    double window_s, p_idle, k_lin, k_cube, u_floor, u_max, c_prefill, c_decode, beta,
           sigma_e, sigma_t;
} agft_env;

/* ENV-T constants (ENV.md §2.1). */
typedef struct {
    double lambda0, burst_mult, t_iter0, t_iter1, e2e0, tau_ref;
    uint32_t seg_steps, steps_per_hour, burst_steps, burst_p32, cap, kv_total, pattern_mode, pad;
    uint32_t ctx_lo[5], ctx_hi[5], gen_lo[5], gen_hi[5], weight[5], pad2;
    double conc_mult[5], hit_rate[5], knot[24];
} agft_trace_cfg;

/* Exploitation phase (Eq. 2; ENV.md §4.10): a classical Page-Hinkley detector on
 * the reward stream.  enable = 0 is the §8(a) hot path.  When the
 * tuner has seen `window` observations since the last alarm it selects greedily (α_t = 0,
 * Eq. 2); an alarm (cum − min > lambda) resets the detector and re-enters Exploration. */
typedef struct { uint32_t enable, window; double delta, lambda; } agft_phase;

/* Mixed maturity-based refinement (ENV.md §4.11): every `period` rounds
 * (and on a phase transition) the action space becomes the ±half_mhz window on the step_mhz
 * lattice around an anchor — the lowest-mean-EDP arm with ≥ min_samples observations while
 * t < mature, the UCB argmax after — minus Extreme-pruned arms.  Without the phase switch it runs on
 * the class schedule with a refinement pass at every period end; with it, on the WIDE schedule. */
typedef struct { uint32_t enable, period, mature, min_samples, half_mhz, step_mhz; } agft_refine;

/* ENV-C closed loop (ENV.md §6): requests a window cannot
 * serve at the chosen clock (u > 1) wait into the next window, where the snapshot sees them
 * (x1, the concurrency penalty, TTFT); the f_max baseline carries its own backlog.  q_max caps
 * the backlog (requests).  Needs the raw rows: replay with agft_replay_raw.
 * enable = 2 selects ENV-S instead (ENV.md §7; SPEC inference_sim S:454-563; P:129-131 continuous
 * batching): every tuner drives its own discrete-event server iteration by iteration — FIFO
 * admission while the KV footprint fits, prefill of the uncached suffix, one token per iteration,
 * retirement — at the clock it chose; each decision reads the server's last-window MetricsSnapshot
 * and the reward comes from the simulated energy and TPOT.  The workspace then also holds
 * each tuner's server (128 + 512·24 + 128·24 B); no f_max baseline is accumulated (base sums 0);
 * the replay runs on the WIDE mapping.  q_max is unused. */
typedef struct { uint32_t enable, q_max; } agft_closed;

typedef struct {
    uint32_t abi_version;     /* must be AGFT_ABI_VERSION */
    uint32_t n_tuners;        /* N ≥ 1 */
    uint32_t d;               /* context dims, first d of x1..x7 (AMB-17) */
    uint32_t n_traces;        /* R: traces held by this handle (local ids 0..R-1) */
    uint32_t trace_base;      /* global id of local trace 0 (Philox key, ENV.md §1) */
    uint32_t record_slots;    /* rows of d_traj / d_gap in agft_replay (0 = none) */
    uint32_t kernel_policy;   /* AGFT_POLICY_AUTO or AGFT_POLICY_WIDE (anything else: AGFT_E_INVALID_ARG) */
    uint32_t pad0;
    agft_grid grid;
    agft_prune prune;
    agft_policy policy;
    agft_env env;
    agft_trace_cfg trace;
    double norm_lo[7], norm_hi[7];   /* context normalisation bounds (AMB-14) */
    uint64_t env_seed;               /* S in ENV.md §1 */
    agft_phase phase;                /* Page-Hinkley exploitation switch (ENV.md §4.10) */
    agft_refine refine;              /* mixed maturity-based refinement (ENV.md §4.11) */
    uint32_t pad1;
    agft_closed closed;              /* ENV-C closed loop (ENV.md §6) */
} agft_config;

/* Per-tuner parameters (the hyper-parameter sweep axes of C4/C5). */
typedef struct {
    uint32_t trace_id;        /* LOCAL trace index in [0, n_traces) */
    uint32_t record_slot;     /* row of d_traj/d_gap (< record_slots), or AGFT_NO_RECORD */
    double alpha0;            /* finite, ≥ 0 (0 = greedy, Eq. 2) */
    double extreme_reward_threshold; /* τ_E, P:387 (−1.2) */
    double historical_k;      /* k_h, P:388 (1.0); finite, ≥ 0 */
} agft_tuner_params;          /* 32 B.  agft_create / agft_attach / agft_run reject (AGFT_E_INVALID_ARG)
                                 a trace_id ≥ n_traces, a record_slot that is neither < record_slots
                                 nor AGFT_NO_RECORD, or a non-finite / negative alpha0, τ_E or k_h
                                 (τ_E finite, any sign). */

/* Per-tuner statistics (ENV.md §4.9–§4.11), 128 B. */
typedef struct {
    uint64_t traj_hash;       /* FNV-1a over the chosen arm of every step */
    uint64_t sum_active;      /* Σ_t |F_available(t)| before pruning (work counter) */
    uint32_t steps, last_arm, n_active, n_pruned_extreme, n_pruned_hist, n_pruned_cascade,
             near_tie_steps, flags;
    double sum_energy, sum_tpot, sum_ttft, sum_edp, sum_reward, base_energy, base_edp;
    uint32_t exploit_steps;   /* steps selected greedily (Eq. 2), §4.10 */
    uint32_t ph_alarms;       /* Page-Hinkley drift alarms */
    uint32_t first_exploit_t; /* first step after which the phase was Exploitation, AGFT_NEVER if none */
    uint32_t phase;           /* current phase: 0 Exploration, 1 Exploitation */
    uint32_t n_refine;        /* refinements applied (ENV.md §4.11) */
    uint32_t last_anchor;     /* arm index of the last refinement anchor, AGFT_NEVER if none */
} agft_tuner_stats;

#define AGFT_NEVER 0xFFFFFFFFu

/* Host-only validation of a config (the checks agft_create makes before touching
 * the device): grid, dimensions, finiteness/ranges. */
agft_status agft_validate(const agft_config *cfg);

/* sizeof of the ABI structs as compiled: which = 0 agft_config, 1 agft_tuner_params,
 * 2 agft_tuner_stats (lets bindings check their mirrors). */
uint32_t agft_struct_size(int which);

/* Bytes of device workspace a config needs (0 if the config is invalid). The
 * workspace must be 256-byte aligned.  It holds every tuner's bandit state — per arm A⁻¹ (packed
 * upper triangle), θ, b, n, r̄, ē (Eqs. 3–5), the active set F_available
 * (§4.3), the EDP window of the reward (AMB-3) and the stats —
 * so that the whole session state is one caller-owned buffer (checkpointable). */
size_t agft_workspace_bytes(const agft_config *cfg);

/* Validate cfg, lay out d_workspace, copy d_params [n_tuners] into it and initialise
 * every tuner: A⁻¹ = I, θ = b = 0, all arms active, empty EDP window (AMB-2).
 * stream is a cudaStream_t (NULL = legacy default stream).  Synchronises once. */
agft_status agft_create(const agft_config *cfg, const agft_tuner_params *d_params,
                        void *d_workspace, size_t ws_bytes, void *stream, agft_handle *out);

/* Checkpoint / resume ("state can be exported for checkpoint and analysis").  Every tuner's
 * state lives in the caller's workspace, so a checkpoint is the caller's copy of the workspace bytes
 * plus the step counter (agft_get_step) and the sweep counter; agft_attach builds a handle on a
 * workspace that already holds such a state (validating cfg exactly as agft_create does, touching
 * no tuner state) and sets the counters to t and sweep_t.  A workspace copied from a handle with the
 * same cfg resumes bit-identically. */
agft_status agft_attach(const agft_config *cfg, void *d_workspace, size_t ws_bytes, void *stream, uint32_t t,
                        uint32_t sweep_t, agft_handle *out);

/* Re-initialise every tuner of the handle (as agft_create does, keeping its params)
 * and set the step counter to 0.  Asynchronous. */
agft_status agft_reset(agft_handle h);

/* ENV-T + the per-window record for steps [t0, t0+n_steps) of every local trace:
 * d_records = [n_traces][n_steps][128 B] (ENV.md §3.2), d_raw = [n_traces][n_steps][12]
 * uint32 raw rows (ENV.md §2.2) or NULL.  Independent of tuner state. */
agft_status agft_trace_generate(agft_handle h, uint32_t t0, uint32_t n_steps, void *d_records,
                                uint32_t *d_raw);

/* One decision window for every tuner (Eq. 1 → response → reward → Eqs. 3–5 → §4.3)
 * at the handle's current step t; d_records = [n_traces][1][128 B] for step t;
 * d_chosen = [n_tuners] chosen arm index, or NULL.  Advances t by 1. */
agft_status agft_step(agft_handle h, const void *d_records, uint32_t *d_chosen);
/* (d_chosen of a frozen tuner — stats.flags bit 0 — reads AGFT_NEVER.) */

/* ---- Live two-phase step.  The paper's controller runs one decision
 * per sampling window on a live server (§4): read the window's metrics, pick
 * a frequency, run the window at it, measure energy and latency, update.  agft_step splits here
 * into the two halves a real controller (NVML + the serving engine's metrics) calls:
 *
 * agft_select: d_rows [n_tuners][12] uint32, 16-byte aligned — each tuner's MetricsSnapshot
 *   counters of the last window in ENV.md §2.2 word order (waiting, running, prefill, decode,
 *   iterations, kv_used, hits, misses; words 8..11 ignored).  Builds x_t (§4.1, with
 *   the config's normalisation bounds), scores every active arm (Eq. 1), takes the argmax (lowest
 *   frequency on ties) and writes d_chosen [n_tuners] = arm index k* (f = f_min + k*·step MHz), or
 *   AGFT_NEVER for a frozen tuner.  Tuner state is not modified.
 * agft_observe: d_resp [n_tuners][3] fp64 = (energy J, TPOT s, TTFT s) measured over the window
 *   run at the selected frequency.  EDP = E × TPOT (AMB-4), then the reward, the
 *   update of the chosen arm (Eqs. 3–5), pruning (§4.3), the exploitation phase / refinement if
 *   configured, and the stats — exactly the replay's a8–a11.  Advances the step counter by 1.
 *   A non-finite E, TPOT or TTFT sets flags bit 0 and freezes that tuner.  The f_max baseline
 *   (base_energy, base_edp) is not measurable live and is not accumulated.
 * Alternation is strict: a second agft_select, or agft_step / agft_replay, between a
 * select and its observe returns AGFT_E_STATE, as does an agft_observe without a select.
 * Both are asynchronous on the handle's stream (one kernel launch each). */
agft_status agft_select(agft_handle h, const uint32_t *d_rows, uint32_t *d_chosen);
agft_status agft_observe(agft_handle h, const double *d_resp);

/* Read-only prediction ("read-only operations (predict, select_*)"): Eq. 1
 * at the handle's step t for the contexts of d_rows (as agft_select) — d_scores [n_tuners][K] fp64
 * = θ_fᵀx_t + α_t·√(x_tᵀA_f⁻¹x_t) for every arm f ∈ F_available (α_t = 0 in Exploitation, Eq. 2),
 * quiet NaN for pruned arms and for every arm of a frozen tuner; d_chosen [n_tuners] (may be NULL)
 * = the arg max agft_select would return.  Changes no state and does not open a select; returns
 * AGFT_E_STATE between a select and its observe. */
agft_status agft_scores(agft_handle h, const uint32_t *d_rows, double *d_scores, uint32_t *d_chosen);

/* The paper's decision loop (§4.2: the context x_t → Eq. 1 arg max over
 * F_available → execute f_t → reward from the measured EDP → Eqs. 3–5 update of the executed
 * arm; then §4.3 pruning) run for n_steps consecutive windows of every tuner, fused
 * into one call: steps [t0, t0+n_steps); t0 must equal the handle's step counter (AGFT_E_STATE
 * otherwise; AGFT_E_INVALID_ARG on a closed-loop handle or a NULL d_records).
 * d_records = [n_traces][n_steps][128 B] as agft_trace_generate writes them.
 * d_traj = [record_slots][n_steps] chosen arms and d_gap = [record_slots][n_steps]
 * relative top-2 score gaps (ENV.md §4.5) for tuners with a record_slot; either may be NULL. */
agft_status agft_replay(agft_handle h, const void *d_records, uint32_t t0, uint32_t n_steps,
                        uint8_t *d_traj, double *d_gap);

/* agft_replay with the raw ENV-T rows of the same windows alongside: d_raw = [n_traces][n_steps][12]
 * uint32 as agft_trace_generate writes them.  Required when closed.enable (ENV-C reads arrivals,
 * running and waiting from the rows); otherwise identical to agft_replay.  agft_replay, agft_step,
 * agft_select and agft_observe return AGFT_E_INVALID_ARG on a closed-loop handle. */
agft_status agft_replay_raw(agft_handle h, const void *d_records, const uint32_t *d_raw, uint32_t t0,
                            uint32_t n_steps, uint8_t *d_traj, double *d_gap);

/* Copy the per-tuner statistics into d_out [n_tuners] (caller-owned device buffer;
 * asynchronous).  These are the analysis export of SPEC.md:224 and the per-tuner analogues of the
 * paper's cumulative energy / EDP and mean TTFT / TPOT figures against the f_max default
 * (Tables 2–3). */
agft_status agft_stats(agft_handle h, agft_tuner_stats *d_out);

/* One tuner's arm state (for checkpoints and parity; "bandit state (all arms …)
 * serializes … for session checkpointing and post-hoc analysis"): d_ainv_packed [K][d(d+1)/2]
 * (row-major upper triangle of A⁻¹), d_b [K][d], d_theta [K][d], d_n [K], d_rbar [K],
 * d_ebar [K], d_active_mask [4] (bit k of word k/32).  Any pointer may be NULL. */
agft_status agft_export_arms(agft_handle h, uint32_t tuner, double *d_ainv_packed, double *d_b,
                             double *d_theta, uint32_t *d_n, double *d_rbar, double *d_ebar,
                             uint32_t *d_active_mask);

/* The handle's current step counter. */
agft_status agft_get_step(agft_handle h, uint32_t *t);

/* The counters a checkpoint needs besides the workspace bytes (agft_attach): the step counter t,
 * the offline-sweep counter sweep_t, and live_pending = 1 between an agft_select and its
 * agft_observe (a checkpoint taken then would lose the pending selection; callers refuse it).
 * Any pointer may be NULL. */
agft_status agft_get_counters(agft_handle h, uint32_t *t, uint32_t *sweep_t, uint32_t *live_pending);

/* End to end from HOST buffers: copies h_params [n_tuners] host→device, creates the
 * tuners in d_workspace, replays steps [0, n_steps) generating the trace in chunks of
 * chunk_steps into d_scratch (≥ n_traces·chunk_steps·128 B; ·176 B with closed.enable, the raw
 * rows following the records), and copies the statistics
 * device→host into h_stats [n_tuners].  d_params_buf is a device buffer of n_tuners
 * agft_tuner_params and d_stats_buf of n_tuners agft_tuner_stats.  Synchronises. */
agft_status agft_run(const agft_config *cfg, const agft_tuner_params *h_params,
                     agft_tuner_params *d_params_buf, uint32_t n_steps, uint32_t chunk_steps,
                     void *d_workspace, size_t ws_bytes, void *d_scratch, size_t scratch_bytes,
                     agft_tuner_stats *d_stats_buf, agft_tuner_stats *h_stats, void *stream);

/* ---- Offline frequency sweep (ENV.md §5): every arm of the grid
 * held fixed over the same windows, as the paper's offline sweep does ("we iterated
 * through all core frequencies … calculated the corresponding EDP"), giving Table 6's
 * "Offline" optimum and each tuner's regret.
 *
 * agft_sweep: windows [t0, t0+n_steps) of every local trace, from the same d_records as
 * agft_replay ([n_traces][n_steps][128 B]).  ACCUMULATES (+=) into caller-zeroed buffers:
 *   d_S  [n_traces][K][3]  Σ_t E, Σ_t TPOT, Σ_t EDP per arm (left-to-right in t)
 *   d_SP [n_traces][5][K]  Σ_t EDP per Table-1 prototype and arm
 *   d_NP [n_traces][5]     windows per prototype
 *   d_O  [n_traces][2]     Σ_t EDP and Σ_t E at the per-window EDP-minimising arm k°
 * and writes d_best [n_traces][n_steps] = k° (smallest index on ties), or NULL.
 * t0 must equal the handle's sweep counter (0 after create/reset; AGFT_E_STATE otherwise),
 * so that chunked sweeps accumulate in window order.  Independent of tuner state. */
agft_status agft_sweep(agft_handle h, const void *d_records, uint32_t t0, uint32_t n_steps, double *d_S,
                       double *d_SP, uint32_t *d_NP, double *d_O, uint8_t *d_best);

/* From the sweep sums: d_koff [n_traces][6] = k_off(r, p) for prototypes p < 5 (0xFF if
 * prototype p never occurred) and k_off(r) at index 5 (smallest index on ties); and, if
 * d_regret is not NULL, d_regret [n_tuners][2] = (sum_edp − Σ EDP at k°, sum_edp −
 * Σ EDP at k_off(r)) for each tuner's current statistics (compare after the same windows).
 * The sweep is open-loop (ENV.md §5): d_regret on a closed-loop handle returns AGFT_E_INVALID_ARG. */
agft_status agft_regret(agft_handle h, const double *d_S, const double *d_SP, const uint32_t *d_NP,
                        const double *d_O, uint8_t *d_koff, double *d_regret);

/* ---- Per-class accounting (measurement; SURVEY §8(d) asks for the roofline of the dominant kernel,
 * and the replay runs one kernel per active-arm class).  Slots 0..5 are the replay classes
 * (0 WIDE K_act > 64 or the WIDE schedule, 1 SEG G=16 (17–32 arms), 2 SEG G=8 (9–16), 3 SEG G=4
 * (2–8), 4 SOLO (1 arm), 5 SEG G=32 (33–64)), 6 the classification kernels, 7 the refinement pass.
 * agft_profile_start zeroes the counters and records a timed CUDA event pair on the launching
 * stream around every later launch.  serialize = 0 keeps the product schedule (the classes of a
 * sub-chunk run concurrently on their own streams, so a class's event time spans its wait for SMs
 * held by the others); serialize = 1 runs every class alone on the handle's stream, so each event
 * pair times one kernel (results are identical either way).  agft_profile_read synchronises the
 * handle's stream and returns:
 *   tuner_steps[c]      tuner-steps the class's kernels processed (Σ over its tuners of the steps)
 *   active_arm_steps[c] Σ over those tuner-steps of |F_available| before pruning (the Eq. 1 work)
 *   kernel_ms[c]        Σ over the class's launches of the event time on its launching stream
 *   launches[c]         launches recorded
 * and stops recording.  Profiling adds two events per launch and two atomics per tuner and launch. */
typedef struct {
    uint64_t tuner_steps[8];
    uint64_t active_arm_steps[8];
    double kernel_ms[8];
    uint32_t launches[8];
} agft_profile;
agft_status agft_profile_start(agft_handle h, int serialize);
/* Resident tuners per SM of replay class `slot` (0..5 as above) for cfg's d and grid, from the CUDA
 * occupancy calculator (registers, shared memory, block size): the residency term of the latency
 * roofline (resident tuners ÷ chain latency per window).  Needs the device; no kernel launched. */
agft_status agft_occupancy(const agft_config *cfg, int slot, uint32_t *tuners_per_sm);
agft_status agft_profile_read(agft_handle h, agft_profile *out);
/* Block-scheduling timeline (measurement): while d_buf is set, every warp of every
 * replay-class launch appends one record when it exits — word 0 = launch sequence << 32 | class slot
 * (0..5 as above) << 16 | SM id, words 1–2 = the %globaltimer values (ns) at the warp's start and end.
 * d_buf is a caller-owned DEVICE buffer of 8 × (1 + 3 × cap_records) bytes; word 0 counts the records
 * appended (records past cap_records are counted, not written).  The call zeroes the counter on the
 * handle's stream and restarts the launch sequence; d_buf = null turns recording off.  Results are
 * identical with or without it.  Recording exists only in a library built with -DAGFT_TIMELINE=1
 * (tools/timeline.py builds that variant; the kernels of the product build carry no timeline code):
 * the product build returns AGFT_E_INVALID_ARG for a non-null d_buf.  AGFT_E_INVALID_ARG also for a
 * null handle or cap_records = 0 with a buffer. */
agft_status agft_timeline(agft_handle h, void *d_buf, uint64_t cap_records);

/* Frees the host handle only; the caller frees its device buffers. */
agft_status agft_destroy(agft_handle h);

/* Process-wide number of CUDA kernels this library has launched so far (host counter,
 * incremented at every <<<>>> the library issues; never synchronises). */
uint64_t agft_kernel_launches(void);

const char *agft_status_string(agft_status s);

#ifdef __cplusplus
}
#endif
#endif /* AGFT_H */
