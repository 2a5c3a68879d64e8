/*
 * agft_oracle.c — CPU ORACLE for the AGFT hot path.  TEST INFRASTRUCTURE ONLY:
 * only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl
 * reference) may load it; the product path never does.
 *
 * Plain fp64, written step by step from the paper (arXiv 2508.01744) and ENV.md,
 * in the paper's order and notation.  Build: gcc -O2 -ffp-contract=off (no
 * -ffast-math, no -march=native) so every "a*b+c" rounds twice, as ENV.md §0 says.
 *
 *   LinUCB (§4.2): A_f = I + Σ x xᵀ, b_f = Σ r x, A_f⁻¹ by Gauss–Jordan, θ_f by
 *   solving A_f θ = b_f (Eq. 5) — the plain definition, no
 *   Sherman–Morrison.  Only the arm updated at step t is re-inverted/re-solved;
 *   every other arm's A, b are unchanged so its cached A⁻¹, θ are exactly what
 *   recomputation would give.
 *
 * Pins (tests/test_oracle_*.py): Philox known-answer vectors; SPEC worked
 * examples (S:67-68, S:77-78, S:163-164, S:183-184, S:283-285, S:293-295,
 * S:303-305); exact-rational brute force of
 * A⁻¹/θ (Fractions); ridge equivalence; closed forms (Sherman–Morrison of I,
 * d=1 ridge-mean UCB); invariants (SPD, symmetric, pruned never chosen,
 * cascade monotone, never empty).  ENV-T / ENV-R against the paper: parity
 * unpinned (the paper's environment is a physical A6000, AMB-22/23); they are
 * pinned to ENV.md's closed forms and SPEC's power example only.
 */
#include "agft_oracle.h"
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---------------------------------------------------------------- Philox (ENV.md §1) */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void draw(const orc_config *c, uint32_t trace_id, uint32_t c0, uint32_t c1, uint32_t c2,
                 uint32_t c3, uint32_t out[4])
{
    uint32_t ctr[4] = {c0, c1, c2, c3};
    uint32_t key[2] = {(uint32_t)c->seed ^ trace_id, (uint32_t)(c->seed >> 32)};
    orc_philox4x32_10(ctr, key, out);
}

static double u32tounit(uint32_t v) { return (double)v * (1.0 / 4294967296.0); }

static double u53(uint32_t a, uint32_t b)
{
    uint64_t m = ((uint64_t)a << 21) ^ ((uint64_t)b >> 11);
    return (double)m * (1.0 / 9007199254740992.0);
}

static uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }

/* ENV.md §2.2: the Table-1 prototype of the 10-minute segment holding window t */
uint32_t orc_prototype(const orc_config *c, uint32_t r, uint32_t t)
{
    uint32_t u4[4];
    draw(c, r, t / c->seg_steps, 1, 0, 0, u4);
    uint32_t v = u4[0] >> 24;
    uint32_t p = 0, cum = 0;
    for (p = 0; p < 5; ++p) {
        cum += c->weight[p];
        if (v < cum) break;
    }
    if (p >= 5) p = 4;
    return p;
}

/* ---------------------------------------------------------------- ENV-T (ENV.md §2.2)
 * Shapes: Table 1 prototypes, §2.4 non-stationarity.
 * parity unpinned (vs paper): the Azure trace is proprietary (AMB-23). */
void orc_trace_row(const orc_config *c, uint32_t r, uint32_t t, uint32_t row[ORC_ROW_WORDS])
{
    uint32_t pattern;
    if (c->pattern_mode < 3) pattern = c->pattern_mode;
    else if (c->pattern_mode == 3) pattern = r % 3;
    else pattern = 1 + r % 2;

    uint32_t u4[4];
    uint32_t p = orc_prototype(c, r, t);

    double m = 1.0;
    if (pattern >= 1) {
        uint32_t s = t % (24u * c->steps_per_hour);
        uint32_t h = s / c->steps_per_hour;
        double fr = (double)(s - h * c->steps_per_hour) / (double)c->steps_per_hour;
        m = c->knot[h] + (c->knot[(h + 1) % 24] - c->knot[h]) * fr;
        if (pattern == 2) {
            draw(c, r, t / c->burst_steps, 2, 0, 0, u4);
            if (u4[0] < c->burst_p32) m = m * c->burst_mult;
        }
    }
    double lam = (c->lambda0 * c->conc_mult[p]) * m;

    uint32_t U[16];
    for (uint32_t j = 0; j < 4; ++j) draw(c, r, t, 3, j, 0, &U[4 * j]);
    double z = u32tounit(U[0]);
    for (int i = 1; i < 12; ++i) z = z + u32tounit(U[i]);
    z = z - 6.0;                                   /* Irwin–Hall ≈ N(0,1) */
    double mu = lam * c->W;
    double va = (mu + sqrt(mu) * z) + 0.5;
    uint32_t a = va < 0.0 ? 0u : (uint32_t)floor(va);

    uint32_t ctx = c->ctx_lo[p] + (uint32_t)(((uint64_t)U[12] * (uint64_t)(c->ctx_hi[p] - c->ctx_lo[p] + 1)) >> 32);
    uint32_t gen = c->gen_lo[p] + (uint32_t)(((uint64_t)U[13] * (uint64_t)(c->gen_hi[p] - c->gen_lo[p] + 1)) >> 32);
    uint32_t hits = umin(a, (uint32_t)floor((double)a * c->hit_rate[p] + 0.5));
    uint32_t misses = a - hits;
    uint32_t ctot = (uint32_t)floor(lam * (c->e2e0 + (double)gen * c->tau_ref) + 0.5);
    uint32_t running = umin(ctot, c->cap);
    uint32_t waiting = ctot - running;
    uint32_t iters = running > 0 ? (uint32_t)floor(c->W / (c->t_iter0 + c->t_iter1 * (double)running)) : 0u;
    uint32_t decode = running * iters;
    uint32_t prefill = a * ctx - hits * (ctx / 2);
    uint32_t kv_used = umin(c->kv_total, running * (ctx + gen / 2));
    draw(c, r, t, 4, 0, 0, u4);

    row[0] = waiting; row[1] = running; row[2] = prefill; row[3] = decode;
    row[4] = iters;   row[5] = kv_used; row[6] = hits;    row[7] = misses;
    row[8] = u4[0];   row[9] = u4[1];   row[10] = u4[2];  row[11] = u4[3];
}

void orc_trace_rows(const orc_config *c, uint32_t r, uint32_t t0, uint32_t n, uint32_t *rows)
{
    for (uint32_t i = 0; i < n; ++i) orc_trace_row(c, r, t0 + i, rows + (size_t)ORC_ROW_WORDS * i);
}

/* ---------------------------------------------------------------- context (§4.1) */
void orc_context(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], double x[7])
{
    uint32_t waiting = row[0], running = row[1], prefill = row[2], decode = row[3];
    uint32_t iters = row[4], kv_used = row[5], hits = row[6], misses = row[7];
    double raw[7];
    raw[0] = waiting > 0 ? 1.0 : 0.0;                                   /* x1 queue presence */
    raw[1] = (double)prefill / c->W;                                    /* x2 prefill throughput */
    raw[2] = (double)decode / c->W;                                     /* x3 decode throughput */
    raw[3] = (double)((uint64_t)prefill + (uint64_t)decode) / (double)(iters > 0 ? iters : 1u); /* x4 */
    raw[4] = (double)running;                                           /* x5 concurrency */
    raw[5] = (double)kv_used / (double)c->kv_total;                     /* x6 KV usage */
    raw[6] = (hits + misses) > 0 ? (double)hits / (double)(hits + misses) : 0.0; /* x7 hit rate */
    for (int i = 0; i < 7; ++i) {                                       /* S:56 normalisation */
        double lo = c->norm_lo[i], hi = c->norm_hi[i];
        if (hi > lo) {
            double v = (raw[i] - lo) / (hi - lo);
            if (v < 0.0) v = 0.0;
            if (v > 1.0) v = 1.0;
            x[i] = v;
        } else {
            x[i] = 0.0;
        }
    }
}

/* ---------------------------------------------------------------- ENV-R (ENV.md §3)
 * EDP = Energy × Delay with Delay = window TPOT (AMB-4).
 * parity unpinned (vs paper): the paper's response is a physical A6000 (AMB-22). */

/* §3.1: per-frequency constants */
static void freq_consts(const orc_config *c, uint32_t F, double *dec, double *pre, double *pw)
{
    double fmax = (double)c->f_max_hw_mhz / 1000.0;
    double f = (double)F / 1000.0;
    *dec = c->c_d / (c->beta + ((1.0 - c->beta) * (f / fmax)));
    *pre = c->c_p / f;
    *pw = (c->k_lin * f) + (c->k_cube * ((f * f) * f));
}

/* §3.3: the response of one window at frequency F */
void orc_response(const orc_config *c, const orc_steprec *rec, uint32_t F, double out[4])
{
    double dec, pre, pw;
    freq_consts(c, F, &dec, &pre, &pw);
    double invW = 1.0 / c->W;
    double q_over = 1.0 / (c->u_max * (1.0 - c->u_max));
    double t_dec = (double)rec->I * dec;
    double t_pre = (double)rec->P * pre;
    double busy = (t_dec + t_pre) * rec->g;
    double u = busy * invW;
    double q = u <= c->u_max ? 1.0 / (1.0 - u) : u * q_over;
    double tpot = (((dec + (t_pre * rec->invIm)) * rec->g) * q) * rec->nT;
    double ue = u > 1.0 ? 1.0 : u;
    if (ue < c->u_floor) ue = c->u_floor;
    double E = ((c->p_idle + (pw * ue)) * c->W) * rec->nE;
    double ttft = ((t_pre * rec->invAm) + (t_dec * rec->wIm)) * q;
    out[0] = E;
    out[1] = tpot;
    out[2] = ttft;
    out[3] = E * tpot;
}

/* §3.2: the per-window step record (row-only, tuner-independent) */
void orc_step_record(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], orc_steprec *rec)
{
    uint32_t waiting = row[0], running = row[1], prefill = row[2], iters = row[4];
    uint32_t a = row[6] + row[7];
    orc_context(c, row, rec->x);
    rec->I = iters;
    rec->P = prefill;
    double rho = (double)(running + waiting) / (double)c->cap;
    rec->g = rho > 1.0 ? rho * sqrt(rho) : 1.0;
    rec->invIm = 1.0 / (double)(iters > 0 ? iters : 1u);
    rec->invAm = 1.0 / (double)(a > 0 ? a : 1u);
    rec->wIm = (double)waiting * rec->invIm;
    rec->nT = 1.0 + c->sigma_t * ((2.0 * u53(row[8], row[9])) - 1.0);
    rec->nE = 1.0 + c->sigma_e * ((2.0 * u53(row[10], row[11])) - 1.0);
    double base[4];
    rec->baseE = 0.0;
    rec->baseEDP = 0.0;
    orc_response(c, rec, c->f_max_hw_mhz, base);
    rec->baseE = base[0];
    rec->baseEDP = base[0] * base[1];
}

void orc_env_response(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], uint32_t F, double out[4])
{
    orc_steprec rec;
    orc_step_record(c, row, &rec);
    orc_response(c, &rec, F, out);
}

/* ---------------------------------------------------------------- offline sweep (ENV.md §5)
 * every frequency of the grid held fixed over the same windows; Table 6
 * "Offline" = the EDP-minimising fixed frequency.  Plain loops in the order
 * §5 writes; sums accumulate (+=) across calls in ascending t. */
void orc_sweep(const orc_config *c, uint32_t r, uint32_t t0, uint32_t n, double *S /*[K][3]*/,
               double *SP /*[5][K]*/, uint32_t *NP /*[5]*/, double *O /*[2]*/, uint8_t *best /*[n] or NULL*/)
{
    uint32_t K = c->n_arms;
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t t = t0 + i;
        uint32_t row[ORC_ROW_WORDS];
        orc_trace_row(c, r, t, row);
        orc_steprec rec;
        orc_step_record(c, row, &rec);
        uint32_t p = orc_prototype(c, r, t);
        NP[p] += 1u;
        uint32_t kb = 0;
        double eb = 0.0, Eb = 0.0;
        for (uint32_t k = 0; k < K; ++k) {
            double out[4];
            orc_response(c, &rec, c->f_min_mhz + k * c->f_step_mhz, out);
            S[3 * k + 0] = S[3 * k + 0] + out[0];
            S[3 * k + 1] = S[3 * k + 1] + out[1];
            S[3 * k + 2] = S[3 * k + 2] + out[3];
            SP[p * K + k] = SP[p * K + k] + out[3];
            if (k == 0 || out[3] < eb) {          /* strict: ties keep the smaller k */
                kb = k;
                eb = out[3];
                Eb = out[0];
            }
        }
        O[0] = O[0] + eb;
        O[1] = O[1] + Eb;
        if (best) best[i] = (uint8_t)kb;
    }
}

/* smallest k minimising v[k * stride] over k < K */
uint32_t orc_argmin(const double *v, uint32_t K, uint32_t stride)
{
    uint32_t kb = 0;
    for (uint32_t k = 1; k < K; ++k)
        if (v[k * stride] < v[kb * stride]) kb = k;
    return kb;
}

/* ---------------------------------------------------------------- small helpers */
static int cmp_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* median of n values (AMB-3): sort, middle value or mean of the two middle values */
double orc_median(const double *v, uint32_t n)
{
    double s[ORC_MAX_WINDOW];
    memcpy(s, v, sizeof(double) * n);
    qsort(s, n, sizeof(double), cmp_double);
    if (n % 2 == 1) return s[n / 2];
    return (s[n / 2 - 1] + s[n / 2]) * 0.5;
}

/* canonical pairwise reduction over 128 slots (ENV.md §4.8) */
double orc_tree128(const double v[128])
{
    double s[128];
    memcpy(s, v, sizeof(s));
    for (int len = 128; len > 1; len /= 2)
        for (int i = 0; i < len / 2; ++i) s[i] = s[2 * i] + s[2 * i + 1];
    return s[0];
}

/* Gauss–Jordan inversion with partial pivoting of [A | I]. */
int orc_invert(uint32_t d, const double *A, double *Ainv)
{
    double M[ORC_MAX_D][2 * ORC_MAX_D];
    for (uint32_t i = 0; i < d; ++i)
        for (uint32_t j = 0; j < d; ++j) {
            M[i][j] = A[i * d + j];
            M[i][d + j] = (i == j) ? 1.0 : 0.0;
        }
    for (uint32_t col = 0; col < d; ++col) {
        uint32_t piv = col;
        for (uint32_t r = col + 1; r < d; ++r)
            if (fabs(M[r][col]) > fabs(M[piv][col])) piv = r;
        if (M[piv][col] == 0.0) return -1;
        if (piv != col)
            for (uint32_t j = 0; j < 2 * d; ++j) {
                double tmp = M[col][j]; M[col][j] = M[piv][j]; M[piv][j] = tmp;
            }
        double pv = M[col][col];
        for (uint32_t j = 0; j < 2 * d; ++j) M[col][j] = M[col][j] / pv;
        for (uint32_t r = 0; r < d; ++r) {
            if (r == col) continue;
            double fct = M[r][col];
            for (uint32_t j = 0; j < 2 * d; ++j) M[r][j] = M[r][j] - fct * M[col][j];
        }
    }
    for (uint32_t i = 0; i < d; ++i)
        for (uint32_t j = 0; j < d; ++j) Ainv[i * d + j] = M[i][d + j];
    return 0;
}

/* Solve A x = b by Gaussian elimination with partial pivoting + back substitution. */
int orc_solve(uint32_t d, const double *A, const double *b, double *xout)
{
    double M[ORC_MAX_D][ORC_MAX_D + 1];
    for (uint32_t i = 0; i < d; ++i) {
        for (uint32_t j = 0; j < d; ++j) M[i][j] = A[i * d + j];
        M[i][d] = b[i];
    }
    for (uint32_t col = 0; col < d; ++col) {
        uint32_t piv = col;
        for (uint32_t r = col + 1; r < d; ++r)
            if (fabs(M[r][col]) > fabs(M[piv][col])) piv = r;
        if (M[piv][col] == 0.0) return -1;
        if (piv != col)
            for (uint32_t j = 0; j <= d; ++j) {
                double tmp = M[col][j]; M[col][j] = M[piv][j]; M[piv][j] = tmp;
            }
        for (uint32_t r = col + 1; r < d; ++r) {
            double fct = M[r][col] / M[col][col];
            for (uint32_t j = col; j <= d; ++j) M[r][j] = M[r][j] - fct * M[col][j];
        }
    }
    for (int i = (int)d - 1; i >= 0; --i) {
        double s = M[i][d];
        for (uint32_t j = (uint32_t)i + 1; j < d; ++j) s = s - M[i][j] * xout[j];
        xout[i] = s / M[i][i];
    }
    return 0;
}

/* ---------------------------------------------------------------- one tuner */
typedef struct {
    double A[ORC_MAX_ARMS][ORC_MAX_D * ORC_MAX_D];
    double Ainv[ORC_MAX_ARMS][ORC_MAX_D * ORC_MAX_D];
    double b[ORC_MAX_ARMS][ORC_MAX_D];
    double theta[ORC_MAX_ARMS][ORC_MAX_D];
    double rbar[ORC_MAX_ARMS], ebar[ORC_MAX_ARMS];
    uint32_t n[ORC_MAX_ARMS];
    int active[ORC_MAX_ARMS];
    double window[ORC_MAX_WINDOW];     /* chronological ring of EDPs */
    uint32_t wcount, whead;
    /* Page-Hinkley detector (ENV.md §4.10) */
    uint32_t phase, ph_quiet, ph_n;
    double ph_mean, ph_cum, ph_min;
    uint8_t extreme[ORC_MAX_ARMS];     /* removed by Extreme pruning: never re-admitted */
} tuner_state;

/* ENV.md §4.11 statistical anchor: the arm with the lowest historical
 * mean EDP among arms with at least min_samples observations; ties to the lowest frequency. */
uint32_t orc_stat_anchor(const orc_config *c, const uint32_t *n, const double *ebar, const uint8_t *extreme)
{
    uint32_t best = ORC_NEVER;
    for (uint32_t k = 0; k < c->n_arms; ++k) {
        if (extreme[k] || n[k] < c->rf_min_samples) continue;
        if (best == ORC_NEVER || ebar[k] < ebar[best]) best = k;
    }
    return best;
}

/* ENV.md §4.11 refine: every grid frequency within ±half of the anchor on
 * the refine step, minus the Extreme-pruned ones.  Returns the number of active arms. */
uint32_t orc_refine_window(const orc_config *c, uint32_t anchor, const uint8_t *extreme, uint8_t *active_out)
{
    uint32_t na = 0;
    const int64_t fa = (int64_t)c->f_min_mhz + (int64_t)anchor * c->f_step_mhz;
    for (uint32_t k = 0; k < c->n_arms; ++k) {
        const int64_t fk = (int64_t)c->f_min_mhz + (int64_t)k * c->f_step_mhz;
        const int64_t dist = fk > fa ? fk - fa : fa - fk;
        const int in = dist <= (int64_t)c->rf_half_mhz && dist % (int64_t)c->rf_step_mhz == 0 && !extreme[k];
        active_out[k] = (uint8_t)in;
        na += (uint32_t)in;
    }
    return na;
}

/* ENV.md §4.10, observe_reward: classical Page-Hinkley on the reward
 * stream; an alarm (cum - min > λ) resets the detector and re-enters Exploration; W quiet
 * observations since the last reset enter Exploitation. */
static void ph_observe(const orc_config *c, tuner_state *S, double r, uint32_t t, orc_stats *st)
{
    S->ph_n += 1;
    double inv = 1.0 / (double)S->ph_n;
    S->ph_mean = S->ph_mean + (r - S->ph_mean) * inv;
    S->ph_cum = S->ph_cum + ((r - S->ph_mean) - c->ph_delta);
    if (S->ph_cum < S->ph_min) S->ph_min = S->ph_cum;
    S->ph_quiet += 1;
    if (S->ph_cum - S->ph_min > c->ph_lambda) {          /* drift alarm */
        st->ph_alarms += 1;
        S->ph_quiet = 0;
        S->ph_n = 0;
        S->ph_mean = 0.0;
        S->ph_cum = 0.0;
        S->ph_min = 0.0;
        S->phase = 0;
    } else if (S->phase == 0 && S->ph_quiet >= c->ph_window) {   /* stable: Exploitation */
        S->phase = 1;
        if (st->first_exploit_t == ORC_NEVER) st->first_exploit_t = t;
    }
}

/* a8 reward (AMB-3): r = clip(1 - EDP/median(window), lo, hi); 0 on an empty window */
double orc_reward(double edp, const double *window, uint32_t n, double clip_lo, double clip_hi)
{
    if (n == 0) return 0.0;
    double ref = orc_median(window, n);
    double r = 1.0 - edp / ref;
    if (r < clip_lo) r = clip_lo;
    if (r > clip_hi) r = clip_hi;
    return r;
}

/* ENV.md §6 (ENV-C): requests the server running window `row` at F leaves queued for the next
 * window.  The window's utilisation u is §3.3's (busy / W) on the record of the row with the
 * carried-in backlog added to `waiting`; a window that needs u > 1 windows of work serves only
 * floor(D / u) of its D = arrivals + backlog requests (the rest keep waiting). */
static uint32_t closed_next(const orc_config *c, const orc_steprec *rec, uint32_t a, uint32_t q, uint32_t F)
{
    double dec, pre, pw;
    freq_consts(c, F, &dec, &pre, &pw);
    double invW = 1.0 / c->W;
    double u = ((((double)rec->I * dec) + ((double)rec->P * pre)) * rec->g) * invW;
    uint32_t D = a + q;
    uint32_t served = u > 1.0 ? (uint32_t)floor((double)D / u) : D;
    uint32_t left = D - served;
    return left < c->cl_q_max ? left : c->cl_q_max;
}

uint32_t orc_closed_next(const orc_config *c, const uint32_t row[ORC_ROW_WORDS], uint32_t q, uint32_t F)
{
    uint32_t rq[ORC_ROW_WORDS];
    memcpy(rq, row, sizeof(rq));
    rq[0] = row[0] + q;
    orc_steprec rec;
    orc_step_record(c, rq, &rec);
    return closed_next(c, &rec, row[6] + row[7], q, F);
}

int orc_run_tuner(const orc_config *c, const orc_tuner *tu, uint32_t T, const uint8_t *follow,
                  orc_stats *st, orc_arms *arms_out, const orc_record *rec)
{
    return orc_run_tuner_ex(c, tu, T, follow, NULL, st, arms_out, rec);
}

int orc_run_tuner_ex(const orc_config *c, const orc_tuner *tu, uint32_t T, const uint8_t *follow,
                     const orc_inject *inj, orc_stats *st, orc_arms *arms_out, const orc_record *rec)
{
    const uint32_t K = c->n_arms, d = c->d;
    if (K < 1 || K > ORC_MAX_ARMS || d < 1 || d > ORC_MAX_D) return -1;
    if (c->median_window < 1 || c->median_window > ORC_MAX_WINDOW) return -1;
    tuner_state *S = (tuner_state *)calloc(1, sizeof(tuner_state));
    if (!S) return -2;
    orc_des *des = NULL;                                             /* §7 ENV-S server of this tuner */
    if (!inj && c->cl_enable == 2) {
        des = (orc_des *)calloc(1, sizeof(orc_des));
        if (!des) { free(S); return -2; }
    }

    /* init (AMB-2): A = I, b = 0, θ = 0, all arms active */
    for (uint32_t k = 0; k < K; ++k) {
        for (uint32_t i = 0; i < d; ++i) {
            S->A[k][i * d + i] = 1.0;
            S->Ainv[k][i * d + i] = 1.0;
        }
        S->active[k] = 1;
    }
    memset(st, 0, sizeof(*st));
    st->traj_hash = 0xcbf29ce484222325ull;
    st->first_exploit_t = ORC_NEVER;
    st->last_anchor = ORC_NEVER;

    /* f_max baseline response constants are folded into orc_env_response */
    uint32_t row[ORC_ROW_WORDS];
    orc_steprec srec, srecb;
    uint32_t cl_q = 0, cl_qb = 0;                                    /* ENV-C backlogs (§6) */
    double x[7];
    double s[ORC_MAX_ARMS], mag[ORC_MAX_ARMS];

    for (uint32_t t = 0; t < T; ++t) {
        if (inj) {                                                   /* unit-test environment */
            memset(&srec, 0, sizeof(srec));                          /* no f_max baseline */
            if (inj->rows) {                                          /* live: §4.1 from the snapshot */
                double xr[7];
                orc_context(c, inj->rows + (size_t)t * ORC_ROW_WORDS, xr);
                for (uint32_t i = 0; i < 7; ++i) x[i] = i < d ? xr[i] : 0.0;
            } else {
                for (uint32_t i = 0; i < 7; ++i) x[i] = i < d ? inj->x[(size_t)t * d + i] : 0.0;
            }
        } else if (c->cl_enable == 2) {                              /* §7 ENV-S: last window's snapshot */
            uint32_t snap12[ORC_ROW_WORDS] = {0};
            memcpy(snap12, des->snap, sizeof(des->snap));
            double xr[7];
            orc_context(c, snap12, xr);
            memset(&srec, 0, sizeof(srec));                          /* no f_max baseline */
            for (uint32_t i = 0; i < 7; ++i) x[i] = i < d ? xr[i] : 0.0;
        } else {
            orc_trace_row(c, tu->trace_id, t, row);                  /* a0 */
            if (c->cl_enable == 1) {                                 /* §6: the servers see their backlog */
                uint32_t rq[ORC_ROW_WORDS], rb[ORC_ROW_WORDS];
                memcpy(rq, row, sizeof(rq));
                memcpy(rb, row, sizeof(rb));
                rq[0] = row[0] + cl_q;
                rb[0] = row[0] + cl_qb;
                orc_step_record(c, rq, &srec);
                orc_step_record(c, rb, &srecb);
                srec.baseE = srecb.baseE;                            /* baseline = the f_max server */
                srec.baseEDP = srecb.baseEDP;
            } else {
                orc_step_record(c, row, &srec);                      /* a2 + the row-only part of a7 */
            }
            for (uint32_t i = 0; i < 7; ++i) x[i] = srec.x[i];
        }
        double alpha = tu->alpha0 / sqrt(1.0 + (double)t / c->tau);   /* a3, AMB-1 */
        if (c->ph_enable && S->phase == 1) {                          /* Exploitation: Eq. 2 greedy */
            alpha = 0.0;
            st->exploit_steps += 1;
        }

        uint32_t n_act = 0;
        for (uint32_t k = 0; k < K; ++k) n_act += S->active[k] ? 1u : 0u;
        st->sum_active += n_act;

        /* a4: Eq. 1 score for every active arm */
        for (uint32_t k = 0; k < K; ++k) {
            if (!S->active[k]) { s[k] = NAN; mag[k] = NAN; continue; }
            double p = 0.0;
            for (uint32_t i = 0; i < d; ++i) p = p + S->theta[k][i] * x[i];
            double qf = 0.0;
            for (uint32_t i = 0; i < d; ++i) {
                double row_i = 0.0;
                for (uint32_t j = 0; j < d; ++j) row_i = row_i + S->Ainv[k][i * d + j] * x[j];
                qf = qf + x[i] * row_i;
            }
            double bonus = alpha * sqrt(qf > 0.0 ? qf : 0.0);          /* AMB-19 */
            s[k] = p + bonus;
            mag[k] = fabs(p) + bonus;
        }
        /* a5/a6: argmax over F_available, ties to the lowest frequency (AMB-5) */
        uint32_t kstar = K;
        for (uint32_t k = 0; k < K; ++k)
            if (S->active[k] && (kstar == K || s[k] > s[kstar])) kstar = k;
        /* near-tie set (§4.5, AMB-6) */
        uint32_t tie_count = 0;
        for (uint32_t k = 0; k < K; ++k) {
            if (!S->active[k] || k == kstar) continue;
            double scale = mag[kstar] > mag[k] ? mag[kstar] : mag[k];
            if (s[kstar] - s[k] < c->tie_rel * scale && !(S->n[kstar] == 0 && S->n[k] == 0)) ++tie_count;
        }
        if (tie_count > 0) st->near_tie_steps++;
        if (rec && rec->near_tie) rec->near_tie[t] = tie_count > 0;
        if (rec && rec->scores)
            for (uint32_t k = 0; k < K; ++k) rec->scores[(size_t)t * K + k] = s[k];
        if (rec && rec->x)
            for (uint32_t i = 0; i < d; ++i) rec->x[(size_t)t * d + i] = x[i];
        if (follow && follow[t] != ORC_FREE) {
            uint32_t kg = follow[t];
            int ok = kg < K && S->active[kg];
            if (ok && kg != kstar) {
                double scale = mag[kstar] > mag[kg] ? mag[kstar] : mag[kg];
                double rel = (s[kstar] - s[kg]) / (scale > 0.0 ? scale : 1.0);
                if (rel > st->max_viol_rel) st->max_viol_rel = rel;
                ok = s[kstar] - s[kg] < c->tie_rel * scale && !(S->n[kstar] == 0 && S->n[kg] == 0);
            }
            if (!ok) st->follow_violations++;
            if (kg < K && S->active[kg]) kstar = kg;                  /* adopt the GPU's choice */
        }
        if (rec && rec->gap) {        /* §4.5: (s_k* − s_k2) / max(m_k*, m_k2), k2 = best other active arm */
            int k2 = -1;
            for (uint32_t k = 0; k < K; ++k)
                if (S->active[k] && k != kstar && (k2 < 0 || s[k] > s[k2])) k2 = (int)k;
            if (k2 < 0) {
                rec->gap[t] = INFINITY;
            } else {
                double den = mag[kstar] > mag[k2] ? mag[kstar] : mag[k2];
                rec->gap[t] = den > 0.0 ? (s[kstar] - s[k2]) / den : 0.0;
            }
        }

        /* a7: response at the chosen frequency; a8: EDP and reward */
        uint32_t F = c->f_min_mhz + kstar * c->f_step_mhz;
        double resp[4];
        if (inj) {
            if (inj->resp) {                                          /* measured response */
                const double *m = inj->resp + ((size_t)t * K + kstar) * 3;
                resp[0] = m[0]; resp[1] = m[1]; resp[2] = m[2];
                resp[3] = m[0] * m[1];                                /* EDP = E × TPOT */
            } else {
                resp[0] = 0.0; resp[1] = 0.0; resp[2] = 0.0;
                resp[3] = inj->edp ? inj->edp[(size_t)t * K + kstar] : 1.0;
            }
        } else if (c->cl_enable == 2) {                              /* §7: the window on the tuner's server */
            orc_des_out o;
            orc_des_window(des, c, tu->trace_id, t, F, &o);
            resp[0] = o.E; resp[1] = o.tpot; resp[2] = o.ttft; resp[3] = o.edp;
        } else {
            orc_response(c, &srec, F, resp);
        }
        double E = resp[0], tpot = resp[1], ttft = resp[2], edp = resp[3];
        if (!inj && c->cl_enable == 1) {                                   /* §6: backlog into window t+1 */
            const uint32_t a = row[6] + row[7];
            cl_q = closed_next(c, &srec, a, cl_q, F);
            cl_qb = closed_next(c, &srecb, a, cl_qb, c->f_max_hw_mhz);
        }
        if (rec && rec->backlog) rec->backlog[t] = cl_q;
        double r = orc_reward(edp, S->window, S->wcount, c->clip_lo, c->clip_hi);
        if (inj && inj->reward) r = inj->reward[(size_t)t * K + kstar];
        const uint32_t phase_sel = S->phase;
        if (c->ph_enable) ph_observe(c, S, r, t, st);                /* §4.10, after a8 */
        if (S->wcount < c->median_window) {
            S->window[S->wcount++] = edp;
        } else {                                   /* overwrite the oldest */
            S->window[S->whead] = edp;
            S->whead = (S->whead + 1) % c->median_window;
        }

        /* a9: Eqs. 3–5 on the chosen arm; Welford means */
        {
            uint32_t k = kstar;
            for (uint32_t i = 0; i < d; ++i)
                for (uint32_t j = 0; j < d; ++j) S->A[k][i * d + j] = S->A[k][i * d + j] + x[i] * x[j];
            for (uint32_t i = 0; i < d; ++i) S->b[k][i] = S->b[k][i] + r * x[i];
            orc_invert(d, S->A[k], S->Ainv[k]);
            orc_solve(d, S->A[k], S->b[k], S->theta[k]);
            S->n[k] += 1;
            double inv = 1.0 / (double)S->n[k];
            S->rbar[k] = S->rbar[k] + (r - S->rbar[k]) * inv;
            S->ebar[k] = S->ebar[k] + (edp - S->ebar[k]) * inv;
        }

        /* a10: §4.3 pruning on the post-update state */
        if (c->prune_enable) {
            int ext[ORC_MAX_ARMS] = {0}, hist[ORC_MAX_ARMS] = {0}, cas[ORC_MAX_ARMS] = {0};
            for (uint32_t k = 0; k < K; ++k)
                ext[k] = S->active[k] && t < c->ext_round_limit && S->n[k] >= c->ext_min_samples &&
                         S->rbar[k] < tu->ext_reward_threshold;
            uint32_t nq = 0;
            double best = INFINITY;
            double v[128];
            for (uint32_t k = 0; k < 128; ++k) v[k] = 0.0;
            for (uint32_t k = 0; k < K; ++k)
                if (S->active[k] && S->n[k] >= c->hist_min_samples) {
                    ++nq;
                    if (S->ebar[k] < best) best = S->ebar[k];
                    v[k] = S->ebar[k];
                }
            if (t >= c->hist_min_round && nq >= 2) {
                double mu = orc_tree128(v) / (double)nq;
                double w2[128];
                for (uint32_t k = 0; k < 128; ++k) w2[k] = 0.0;
                for (uint32_t k = 0; k < K; ++k)
                    if (S->active[k] && S->n[k] >= c->hist_min_samples)
                        w2[k] = (S->ebar[k] - mu) * (S->ebar[k] - mu);
                double sd = sqrt(orc_tree128(w2) / (double)nq);
                double thr = best + tu->hist_k * sd;
                for (uint32_t k = 0; k < K; ++k)
                    hist[k] = S->active[k] && S->n[k] >= c->hist_min_samples && S->ebar[k] > thr;
            }
            int kc = -1;
            for (uint32_t k = 0; k < K; ++k)
                if ((ext[k] || hist[k]) &&
                    (double)(c->f_min_mhz + k * c->f_step_mhz) < c->cascade_fraction * (double)c->f_max_hw_mhz)
                    kc = (int)k;
            for (int j = 0; j < kc; ++j) cas[j] = S->active[j] && !ext[j] && !hist[j];
            uint32_t remaining = 0;
            for (uint32_t k = 0; k < K; ++k)
                if (S->active[k] && !ext[k] && !hist[k] && !cas[k]) ++remaining;
            int restore = -1;
            if (remaining == 0) {               /* AMB-11: never empty the action space */
                for (uint32_t k = 0; k < K; ++k)
                    if ((ext[k] || hist[k] || cas[k]) && (restore < 0 || S->rbar[k] > S->rbar[restore]))
                        restore = (int)k;
            }
            for (uint32_t k = 0; k < K; ++k) {
                if (!(ext[k] || hist[k] || cas[k]) || (int)k == restore) continue;
                S->active[k] = 0;
                if (ext[k]) {
                    st->n_pruned_extreme++;
                    S->extreme[k] = 1;
                }
                else if (hist[k]) st->n_pruned_hist++;
                else st->n_pruned_cascade++;
            }
        }

        /* §4.11 mixed maturity-based refinement, after pruning: every rf_period rounds and on a
         * phase transition */
        if (c->rf_enable && ((t + 1) % c->rf_period == 0 || (c->ph_enable && S->phase != phase_sel))) {
            uint32_t anchor = ORC_NEVER;
            if (t < c->rf_mature) {                                   /* Statistical */
                uint8_t ex[ORC_MAX_ARMS];
                for (uint32_t k = 0; k < K; ++k) ex[k] = S->extreme[k];
                anchor = orc_stat_anchor(c, S->n, S->ebar, ex);
            } else {                                                  /* Predictive */
                double a_ucb = tu->alpha0 / sqrt(1.0 + (double)t / c->tau);   /* Eq. 1's α_t */
                double best = 0.0;
                for (uint32_t k = 0; k < K; ++k) {
                    if (!S->active[k]) continue;
                    double p = 0.0;
                    for (uint32_t i = 0; i < d; ++i) p = p + S->theta[k][i] * x[i];
                    double qf = 0.0;
                    for (uint32_t i = 0; i < d; ++i) {
                        double row_i = 0.0;
                        for (uint32_t j = 0; j < d; ++j) row_i = row_i + S->Ainv[k][i * d + j] * x[j];
                        qf = qf + x[i] * row_i;
                    }
                    double ucb = p + a_ucb * sqrt(qf > 0.0 ? qf : 0.0);
                    if (anchor == ORC_NEVER || ucb > best) { anchor = k; best = ucb; }
                }
            }
            if (anchor != ORC_NEVER) {
                uint8_t ex[ORC_MAX_ARMS], act[ORC_MAX_ARMS];
                for (uint32_t k = 0; k < K; ++k) ex[k] = S->extreme[k];
                orc_refine_window(c, anchor, ex, act);
                for (uint32_t k = 0; k < K; ++k) S->active[k] = act[k];
                st->n_refine += 1;
                st->last_anchor = anchor;
            }
        }

        /* a11: stats, in ENV.md §4.9 order */
        st->sum_energy += E;
        st->sum_tpot += tpot;
        st->sum_ttft += ttft;
        st->sum_edp += edp;
        st->sum_reward += r;
        st->base_energy += srec.baseE;
        st->base_edp += srec.baseEDP;
        st->traj_hash = (st->traj_hash ^ (uint64_t)kstar) * 0x100000001b3ull;
        st->steps += 1;
        st->last_arm = kstar;

        if (rec) {
            if (rec->arm) rec->arm[t] = (uint8_t)kstar;
            if (rec->reward) rec->reward[t] = r;
            if (rec->edp) rec->edp[t] = edp;
            if (rec->energy) rec->energy[t] = E;
            if (rec->tpot) rec->tpot[t] = tpot;
            if (rec->ttft) rec->ttft[t] = ttft;
            if (rec->n_active) {
                uint32_t na = 0;
                for (uint32_t k = 0; k < K; ++k) na += S->active[k] ? 1u : 0u;
                rec->n_active[t] = na;
            }
            if (rec->active_mask)
                for (uint32_t k = 0; k < K; ++k)
                    if (S->active[k]) rec->active_mask[(size_t)t * 4 + k / 32] |= 1u << (k % 32);
        }
    }
    uint32_t na = 0;
    for (uint32_t k = 0; k < K; ++k) na += S->active[k] ? 1u : 0u;
    st->n_active = na;
    st->phase = S->phase;

    if (arms_out) {
        memset(arms_out, 0, sizeof(*arms_out));
        for (uint32_t k = 0; k < K; ++k) {
            for (uint32_t i = 0; i < d; ++i) {
                for (uint32_t j = 0; j < d; ++j) {
                    arms_out->A[k][i][j] = S->A[k][i * d + j];
                    arms_out->Ainv[k][i][j] = S->Ainv[k][i * d + j];
                }
                arms_out->b[k][i] = S->b[k][i];
                arms_out->theta[k][i] = S->theta[k][i];
            }
            arms_out->rbar[k] = S->rbar[k];
            arms_out->ebar[k] = S->ebar[k];
            arms_out->n[k] = S->n[k];
            arms_out->active[k] = (uint8_t)S->active[k];
        }
    }
    free(S);
    free(des);
    return 0;
}

/* ---------------------------------------------------------------- thread pool over tuners */
typedef struct {
    const orc_config *c;
    const orc_tuner *tuners;
    orc_stats *stats;
    uint32_t n, T, stride, first;
    int rc;
} batch_job;

static void *batch_worker(void *arg)
{
    batch_job *j = (batch_job *)arg;
    for (uint32_t i = j->first; i < j->n; i += j->stride) {
        int rc = orc_run_tuner(j->c, &j->tuners[i], j->T, NULL, &j->stats[i], NULL, NULL);
        if (rc) j->rc = rc;
    }
    return NULL;
}

int orc_run_batch(const orc_config *c, const orc_tuner *tuners, uint32_t n, uint32_t T, int threads,
                  orc_stats *stats)
{
    if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    if ((uint32_t)threads > n) threads = (int)(n > 0 ? n : 1);
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    batch_job *jobs = (batch_job *)calloc((size_t)threads, sizeof(batch_job));
    if (!th || !jobs) { free(th); free(jobs); return -2; }
    for (int i = 0; i < threads; ++i) {
        jobs[i] = (batch_job){c, tuners, stats, n, T, (uint32_t)threads, (uint32_t)i, 0};
        pthread_create(&th[i], NULL, batch_worker, &jobs[i]);
    }
    int rc = 0;
    for (int i = 0; i < threads; ++i) {
        pthread_join(th[i], NULL);
        if (jobs[i].rc) rc = jobs[i].rc;
    }
    free(th);
    free(jobs);
    return rc;
}

/* ---------------------------------------------------------------- ENV.md §7: ENV-S
 * The discrete-event continuous-batching server of SPEC's inference_sim, written
 * out as ENV.md §7 states it: FIFO admission while the KV footprint fits, one prefill
 * iteration per admitted request (the uncached suffix; a template seen before skips half the
 * prompt), then one output token per iteration, retirement at the target length; iteration time
 * overhead + max(prefill, decode) × the concurrency penalty; energy p_idle·W + pw·max(u, u_floor)·W
 * while busy. Plain loops over the queue and the slots, in slot order. */
static const uint32_t des_pool[5] = {500, 500, 500, 500, 5};

void orc_des_init(orc_des *s) { memset(s, 0, sizeof(*s)); }

int orc_des_push(orc_des *s, const orc_config *c, double arr, uint32_t ctx, uint32_t gen, uint32_t tmpl)
{
    if ((uint64_t)ctx + gen > c->kv_total || s->qlen == ORC_DES_QMAX) {
        s->dropped += 1;
        return 1;
    }
    orc_des_req *q = &s->q[(s->qhead + s->qlen) % ORC_DES_QMAX];
    q->arr = arr;
    q->ctx = ctx;
    q->gen = gen;
    q->tmpl = tmpl;
    s->qlen += 1;
    return 0;
}

void orc_des_run(orc_des *s, const orc_config *c, uint32_t F, double t_end, orc_des_out *o)
{
    const double fmax = (double)c->f_max_hw_mhz / 1000.0;
    const double f = (double)F / 1000.0;
    const double dec = c->c_d / (c->beta + ((1.0 - c->beta) * (f / fmax)));   /* §3.1 */
    const double pre = c->c_p / f;
    const double pw = (c->k_lin * f) + (c->k_cube * ((f * f) * f));
    uint32_t P = 0, Dc = 0, I = 0, hits = 0, misses = 0, n_tok = 0, n_first = 0;
    double busy = 0.0, sdec = 0.0, sfirst = 0.0;
    uint8_t fresh[ORC_DES_RMAX];
    while (s->clock < t_end) {
        uint32_t npre = 0;
        memset(fresh, 0, sizeof(fresh));
        while (s->qlen > 0) {                                       /* admission, head of line */
            orc_des_req *h = &s->q[s->qhead];
            if (!(h->arr <= s->clock) || s->nrun >= ORC_DES_RMAX || (uint64_t)s->kv + h->ctx + h->gen > c->kv_total)
                break;
            uint32_t hit = (s->store[h->tmpl >> 5] >> (h->tmpl & 31)) & 1u;
            s->store[h->tmpl >> 5] |= 1u << (h->tmpl & 31);
            hits += hit;
            misses += 1u - hit;
            npre += h->ctx - (hit ? h->ctx / 2 : 0u);
            s->kv += h->ctx + h->gen;
            uint32_t k = 0;
            while (s->run[k].used) ++k;                              /* the lowest free slot */
            s->run[k].arr = h->arr;
            s->run[k].ctx = h->ctx;
            s->run[k].gen = h->gen;
            s->run[k].done = 0;
            s->run[k].pre = 0;
            s->run[k].used = 1;
            fresh[k] = 1;
            s->nrun += 1;
            s->qhead = (s->qhead + 1) % ORC_DES_QMAX;
            s->qlen -= 1;
        }
        uint32_t ndec = 0;
        for (uint32_t k = 0; k < ORC_DES_RMAX; ++k) ndec += (s->run[k].used && s->run[k].pre) ? 1u : 0u;
        if (npre == 0 && ndec == 0) {                                /* idle until the next arrival */
            const double nxt = s->qlen > 0 ? s->q[s->qhead].arr : t_end;
            s->clock = nxt < t_end ? nxt : t_end;
            continue;
        }
        const double rho = (double)s->nrun / (double)c->cap;
        const double g = rho > 1.0 ? rho * sqrt(rho) : 1.0;
        const double tp = (double)npre * pre, td = ndec > 0 ? dec : 0.0;
        const double dt = ORC_DES_OVER + ((tp > td ? tp : td) * g);
        s->clock = s->clock + dt;
        for (uint32_t k = 0; k < ORC_DES_RMAX; ++k) {                /* one output token each */
            orc_des_slot *q = &s->run[k];
            if (!q->used || !q->pre) continue;
            q->done += 1;
            if (q->done == 1) {
                sfirst = sfirst + (s->clock - q->arr);
                n_first += 1;
            }
            if (q->done == q->gen) {
                s->kv -= q->ctx + q->gen;
                q->used = 0;
                s->nrun -= 1;
            }
        }
        for (uint32_t k = 0; k < ORC_DES_RMAX; ++k)
            if (fresh[k]) s->run[k].pre = 1;
        P += npre;
        Dc += ndec;
        I += 1;
        n_tok += ndec;
        busy = busy + dt;
        sdec = sdec + (dt * (double)ndec);
    }
    const double u = busy / c->W;
    double ue = busy > 0.0 ? (u > 1.0 ? 1.0 : u) : 0.0;
    if (busy > 0.0 && ue < c->u_floor) ue = c->u_floor;
    o->E = (c->p_idle + (pw * ue)) * c->W;
    o->tpot = n_tok > 0 ? sdec / (double)n_tok : dec;
    o->ttft = n_first > 0 ? sfirst / (double)n_first : 0.0;
    o->edp = o->E * o->tpot;
    const uint32_t snap[8] = {s->qlen, s->nrun, P, Dc, I, s->kv, hits, misses};
    memcpy(s->snap, snap, sizeof(snap));
}

void orc_des_window(orc_des *s, const orc_config *c, uint32_t r, uint32_t t, uint32_t F, orc_des_out *o)
{
    uint32_t row[ORC_ROW_WORDS];
    orc_trace_row(c, r, t, row);
    const uint32_t p = orc_prototype(c, r, t);
    const uint32_t a = row[6] + row[7];                              /* §2.2 arrivals */
    for (uint32_t i = 0; i < a; ++i) {
        const double arr = ((double)t * c->W) + ((((double)i + 0.5) / (double)a) * c->W);
        uint32_t u4[4];
        draw(c, r, t, 5, i, 0, u4);
        const uint32_t ctx = c->ctx_lo[p] + (uint32_t)(((uint64_t)u4[0] * (c->ctx_hi[p] - c->ctx_lo[p] + 1u)) >> 32);
        const uint32_t gen = c->gen_lo[p] + (uint32_t)(((uint64_t)u4[1] * (c->gen_hi[p] - c->gen_lo[p] + 1u)) >> 32);
        const uint32_t tmpl = (uint32_t)(((uint64_t)u4[2] * des_pool[p]) >> 32);
        orc_des_push(s, c, arr, ctx, gen, tmpl);
    }
    orc_des_run(s, c, F, (double)(t + 1) * c->W, o);
}

uint32_t orc_sizeof(int which)
{
    switch (which) {
    case 0: return (uint32_t)sizeof(orc_config);
    case 1: return (uint32_t)sizeof(orc_tuner);
    case 2: return (uint32_t)sizeof(orc_stats);
    case 3: return (uint32_t)sizeof(orc_arms);
    case 4: return (uint32_t)sizeof(orc_steprec);
    case 5: return (uint32_t)sizeof(orc_record);
    case 6: return (uint32_t)sizeof(orc_inject);
    case 7: return (uint32_t)sizeof(orc_des);
    default: return 0;
    }
}
