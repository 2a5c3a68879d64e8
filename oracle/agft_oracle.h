/*
 * agft_oracle.h — the CPU ORACLE of the AGFT hot path (TEST INFRASTRUCTURE ONLY).
 *
 * A plain, slow, fp64 implementation of the method of arXiv 2508.01744 (AGFT,
 * §4.1–§4.3) plus the synthetic environment of ENV.md, written from the paper
 * and ENV.md.  It shares no code with the CUDA path (paper_2508_01744_b200/csrc):
 * no headers, no helpers, no tables.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions whose result is not pinned
 * by anything but ENV.md itself (ENV-T, ENV-R against the paper) are marked
 * "parity unpinned (vs paper)" — they are pinned only to ENV.md's own closed
 * forms and SPEC's worked examples.
 */
#ifndef AGFT_ORACLE_H
#define AGFT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_ARMS 128
#define ORC_MAX_D 7
#define ORC_MAX_WINDOW 64
#define ORC_ROW_WORDS 12

typedef struct {
    /* frequency grid, P:257 (210..1800 MHz step 15) */
    uint32_t f_min_mhz, f_step_mhz, n_arms, f_max_hw_mhz;
    uint32_t d;                        /* context dims used (first d of x1..x7), AMB-17 */
    uint32_t median_window;            /* reward reference window, AMB-3 */
    uint32_t prune_enable;             /* §4.3 on/off (Table 5 ablation flag) */
    uint32_t ext_round_limit, ext_min_samples, hist_min_round, hist_min_samples;
    uint32_t pattern_mode;             /* ENV.md §2.1 */
    uint32_t seg_steps, steps_per_hour, burst_steps, burst_p32, cap, kv_total;
    uint32_t ctx_lo[5], ctx_hi[5], gen_lo[5], gen_hi[5], weight[5];
    uint32_t pad0;
    uint64_t seed;
    double norm_lo[7], norm_hi[7];
    double tau, clip_lo, clip_hi, cascade_fraction, tie_rel;
    double W, p_idle, k_lin, k_cube, u_floor, u_max, c_p, c_d, beta, sigma_e, sigma_t;
    double lambda0, burst_mult, t_iter0, t_iter1, e2e0, tau_ref;
    double conc_mult[5], hit_rate[5], knot[24];
    /* Page-Hinkley exploitation switch (ENV.md §4.10; Eq. 2) */
    uint32_t ph_enable, ph_window;     /* on/off; quiet window W (50) */
    double ph_delta, ph_lambda;        /* δ (0.005), λ (50·δ) */
    /* Mixed maturity-based refinement (ENV.md §4.11) */
    uint32_t rf_enable, rf_period;     /* on/off; evaluated every rf_period rounds (25) */
    uint32_t rf_mature, rf_min_samples;/* t_mature (100); statistical anchor needs n ≥ 4 */
    uint32_t rf_half_mhz, rf_step_mhz; /* window ±150 MHz, step 15 MHz */
    /* ENV-C closed loop (ENV.md §6) */
    uint32_t cl_enable, cl_q_max;      /* on/off; backlog cap (requests) */
} orc_config;

typedef struct {                       /* per-tuner hyper-parameters (the sweep axes) */
    uint32_t trace_id, pad;
    double alpha0, ext_reward_threshold, hist_k;
} orc_tuner;

typedef struct {                       /* ENV.md §4.9 */
    uint64_t traj_hash, sum_active;
    uint32_t steps, last_arm, n_active, n_pruned_extreme, n_pruned_hist, n_pruned_cascade,
             near_tie_steps, follow_violations;
    double sum_energy, sum_tpot, sum_ttft, sum_edp, sum_reward, base_energy, base_edp;
    double max_viol_rel;               /* follow mode: worst (s_max - s_gpu)/scale seen */
    /* ENV.md §4.10 */
    uint32_t exploit_steps;            /* steps selected greedily (Eq. 2) */
    uint32_t ph_alarms;                /* Page-Hinkley drift alarms */
    uint32_t first_exploit_t;          /* first step t after which the phase became Exploitation (ORC_NEVER) */
    uint32_t phase;                    /* final phase: 0 Exploration, 1 Exploitation */
    uint32_t n_refine;                 /* refinements applied (ENV.md §4.11) */
    uint32_t last_anchor;              /* arm index of the last anchor (ORC_NEVER if none) */
} orc_stats;

#define ORC_NEVER 0xFFFFFFFFu

typedef struct {                       /* final per-arm state, row-major */
    double A[ORC_MAX_ARMS][ORC_MAX_D][ORC_MAX_D];
    double Ainv[ORC_MAX_ARMS][ORC_MAX_D][ORC_MAX_D];
    double b[ORC_MAX_ARMS][ORC_MAX_D];
    double theta[ORC_MAX_ARMS][ORC_MAX_D];
    double rbar[ORC_MAX_ARMS], ebar[ORC_MAX_ARMS];
    uint32_t n[ORC_MAX_ARMS];
    uint8_t active[ORC_MAX_ARMS];
} orc_arms;

typedef struct {                       /* ENV.md §3.2 per-window step record */
    double x[7], g, invIm, invAm, wIm, nT, nE, baseE, baseEDP;
    uint32_t I, P;
} orc_steprec;

typedef struct {                       /* optional per-step record (any pointer may be NULL) */
    uint8_t *arm;                      /* [T] chosen arm */
    uint8_t *near_tie;                 /* [T] 1 if the near-tie set had >1 member (§4.5) */
    double *reward, *edp, *energy, *tpot, *ttft; /* [T] */
    double *scores;                    /* [T][n_arms], NaN for inactive arms */
    double *x;                         /* [T][d] */
    uint32_t *n_active;                /* [T] after pruning */
    uint32_t *active_mask;             /* [T][4] after pruning (caller zeroes it) */
    uint32_t *backlog;                 /* [T] ENV-C q carried out of window t (§6) */
    double *gap;                       /* [T] relative top-2 gap of the executed arm (ENV.md §4.5) */
} orc_record;

typedef struct {                       /* unit-test / live environment: replaces ENV-T/ENV-R */
    const double *x;                   /* [T][d] contexts */
    const double *edp;                 /* [T][n_arms] EDP of choosing arm k at t (NULL: 1.0) */
    const double *reward;              /* [T][n_arms] reward override (NULL: median rule) */
    /* Live controller: the context is built
     * from each window's MetricsSnapshot counters and the response is MEASURED, not modelled. */
    const uint32_t *rows;              /* [T][12] snapshot rows; x_t = orc_context(row_t) (overrides x) */
    const double *resp;                /* [T][n_arms][3] measured (E, TPOT, TTFT) of choosing arm k at t;
                                          EDP = E × TPOT (AMB-4); overrides edp */
} orc_inject;

#define ORC_FREE 255                   /* follow[t] == ORC_FREE: no forced choice at step t */

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t orc_prototype(const orc_config *c, uint32_t trace_id, uint32_t t);
void orc_trace_row(const orc_config *c, uint32_t trace_id, uint32_t t, uint32_t row[ORC_ROW_WORDS]);
void orc_trace_rows(const orc_config *c, uint32_t trace_id, uint32_t t0, uint32_t n,
                    uint32_t *rows /* [n][12] */);
void orc_context(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], double x[7]);
void orc_step_record(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], orc_steprec *rec);
void orc_response(const orc_config *c, const orc_steprec *rec, uint32_t f_mhz,
                  double out[4] /* E, TPOT, TTFT, EDP */);
void orc_env_response(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], uint32_t f_mhz,
                      double out[4] /* E, TPOT, TTFT, EDP */);
double orc_median(const double *v, uint32_t n);
double orc_reward(double edp, const double *window, uint32_t n, double clip_lo, double clip_hi);
double orc_tree128(const double v[128]);
int orc_invert(uint32_t d, const double *A /*[d][d]*/, double *Ainv /*[d][d]*/);
int orc_solve(uint32_t d, const double *A, const double *b, double *xout);

/* Run one tuner for steps [0, T).  follow == NULL: free-running.  follow != NULL:
 * follow-GPU mode — at each step check follow[t] is in the oracle's near-tie set
 * (§4.5, counted in stats->follow_violations) and adopt it. Returns 0 or <0 on bad args. */
int orc_run_tuner(const orc_config *c, const orc_tuner *tu, uint32_t T, const uint8_t *follow,
                  orc_stats *stats, orc_arms *arms /* may be NULL */, const orc_record *rec);

int orc_run_tuner_ex(const orc_config *c, const orc_tuner *tu, uint32_t T, const uint8_t *follow,
                     const orc_inject *inj, orc_stats *stats, orc_arms *arms, const orc_record *rec);

/* struct sizes, for the Python mirror's layout check */
/* ENV.md §5 offline sweep (accumulating) and argmin helper */
void orc_sweep(const orc_config *c, uint32_t trace_id, uint32_t t0, uint32_t n, double *S /*[K][3]*/,
               double *SP /*[5][K]*/, uint32_t *NP /*[5]*/, double *O /*[2]*/, uint8_t *best /*[n] or NULL*/);
uint32_t orc_argmin(const double *v, uint32_t K, uint32_t stride);

/* ENV.md §4.11 helpers (also used by the run loop): the statistical anchor (smallest ē among
 * non-extreme arms with n ≥ min_samples, ties to the lowest arm; ORC_NEVER if none) and the
 * refined action space around an anchor (window minus extreme-pruned arms). */
uint32_t orc_stat_anchor(const orc_config *c, const uint32_t *n, const double *ebar, const uint8_t *extreme);
uint32_t orc_refine_window(const orc_config *c, uint32_t anchor, const uint8_t *extreme, uint8_t *active_out);

/* ENV.md §6: the backlog carried out of a window with snapshot `row` (waiting NOT yet including
 * the carried-in backlog q) run at F MHz: q' = min(q_max, D - served), D = arrivals + q. */
uint32_t orc_closed_next(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], uint32_t q, uint32_t F_mhz);

/* ENV.md §7 ENV-S: the discrete-event continuous-batching server (SPEC inference_sim, S:454-563;
 * P:129-131), selected by cl_enable = 2.  State of one tuner's server and one window's outcome. */
#define ORC_DES_RMAX 128
#define ORC_DES_QMAX 512
#define ORC_DES_OVER 0.004
typedef struct { double arr; uint32_t ctx, gen, tmpl, pad; } orc_des_req;
typedef struct { double arr; uint32_t ctx, gen, done, pre, used, pad; } orc_des_slot;
typedef struct {
    double clock;
    orc_des_req q[ORC_DES_QMAX];
    uint32_t qhead, qlen, nrun, kv, dropped, pad;
    orc_des_slot run[ORC_DES_RMAX];
    uint32_t store[16];                /* template prefix cached (512 bits) */
    uint32_t snap[8];                  /* the last window's MetricsSnapshot (§2.2 word order) */
} orc_des;
typedef struct { double E, tpot, ttft, edp; } orc_des_out;
void orc_des_init(orc_des *s);
/* queue one request (ENV.md §7 arrival rule); returns 0, or 1 if it was dropped */
int orc_des_push(orc_des *s, const orc_config *c, double arr, uint32_t ctx, uint32_t gen, uint32_t tmpl);
/* run the engine until t_end at F MHz and measure the window (updates snap) */
void orc_des_run(orc_des *s, const orc_config *c, uint32_t F, double t_end, orc_des_out *o);
/* window t of trace r: its arrivals (§7), then orc_des_run to (t+1)·W */
void orc_des_window(orc_des *s, const orc_config *c, uint32_t r, uint32_t t, uint32_t F, orc_des_out *o);

uint32_t orc_sizeof(int which /* 0 config 1 tuner 2 stats 3 arms 4 steprec 5 record 6 inject 7 des */);

/* Free-running batch over a pthread pool; stats[i] for tuners[i]. threads<=0: all cores. */
int orc_run_batch(const orc_config *c, const orc_tuner *tuners, uint32_t n_tuners, uint32_t T,
                  int threads, orc_stats *stats);

#ifdef __cplusplus
}
#endif
#endif
