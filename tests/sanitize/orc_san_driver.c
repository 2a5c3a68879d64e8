/* orc_san_driver.c — runs the CPU oracle (test infrastructure) built with AddressSanitizer and
 * UndefinedBehaviorSanitizer (race / memory checking of both implementations).
 *
 *   orc_san_driver CFG_BIN TUNERS_BIN T OUT_BIN
 * CFG_BIN is one orc_config, TUNERS_BIN n × orc_tuner (as oracle/__init__.py marshals them).
 * Every tuner runs free-running with every per-step record and the final arm state requested
 * (so each oracle array is written through), then once in follow mode along its own trajectory,
 * and trace 0 is swept over [0, T) (ENV.md §5).  OUT_BIN receives n × orc_stats of the free runs,
 * then the sweep sums S [K][3], SP [5][K], NP [5], O [2].  Exit status 0 = clean. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../oracle/agft_oracle.h"

static void *slurp(const char *path, size_t *len)
{
    FILE *f = fopen(path, "rb");
    if (!f) return NULL;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    void *p = malloc((size_t)n);
    if (p && fread(p, 1, (size_t)n, f) != (size_t)n) { free(p); p = NULL; }
    fclose(f);
    *len = (size_t)n;
    return p;
}

int main(int argc, char **argv)
{
    if (argc != 5) return 2;
    size_t lc = 0, lt = 0;
    orc_config *c = slurp(argv[1], &lc);
    orc_tuner *tu = slurp(argv[2], &lt);
    const uint32_t T = (uint32_t)strtoul(argv[3], NULL, 10);
    if (!c || !tu || lc != sizeof(orc_config) || lt % sizeof(orc_tuner)) return 2;
    const uint32_t n = (uint32_t)(lt / sizeof(orc_tuner)), K = c->n_arms, d = c->d;
    orc_stats *st = calloc(n, sizeof(orc_stats));
    orc_arms *arms = malloc(sizeof(orc_arms));
    uint8_t *arm = malloc(T), *near = malloc(T);
    double *rw = malloc(T * 8), *edp = malloc(T * 8), *en = malloc(T * 8), *tp = malloc(T * 8),
           *tt = malloc(T * 8), *gap = malloc(T * 8);
    double *sc = malloc((size_t)T * K * 8), *x = malloc((size_t)T * d * 8);
    uint32_t *na = malloc(T * 4), *mask = calloc((size_t)T * 4, 4), *bl = malloc(T * 4);
    orc_record rec = {arm, near, rw, edp, en, tp, tt, sc, x, na, mask, bl, gap};
    for (uint32_t i = 0; i < n; ++i) {
        memset(mask, 0, (size_t)T * 16);
        if (orc_run_tuner(c, &tu[i], T, NULL, &st[i], arms, &rec) != 0) return 3;
        orc_stats fs;
        if (orc_run_tuner(c, &tu[i], T, arm, &fs, NULL, NULL) != 0) return 3;
        if (fs.traj_hash != st[i].traj_hash || fs.follow_violations) return 4;
    }
    double *S = calloc((size_t)K * 3, 8), *SP = calloc((size_t)5 * K, 8), O[2] = {0, 0};
    uint32_t NP[5] = {0, 0, 0, 0, 0};
    uint8_t *best = malloc(T);
    orc_sweep(c, 0, 0, T, S, SP, NP, O, best);
    FILE *f = fopen(argv[4], "wb");
    if (!f) return 2;
    fwrite(st, sizeof(orc_stats), n, f);
    fwrite(S, 8, (size_t)K * 3, f);
    fwrite(SP, 8, (size_t)5 * K, f);
    fwrite(NP, 4, 5, f);
    fwrite(O, 8, 2, f);
    fclose(f);
    free(st); free(arms); free(arm); free(near); free(rw); free(edp); free(en); free(tp); free(tt); free(gap);
    free(sc); free(x); free(na); free(mask); free(bl); free(S); free(SP); free(best); free(c); free(tu);
    return 0;
}
