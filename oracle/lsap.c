/*
 * CPU oracle (TEST INFRASTRUCTURE ONLY): exact dense linear sum assignment.
 *
 * The reference projects the final gradient with
 * scipy.optimize.linear_sum_assignment (/root/reference/pkg/src/otmatch/lap.py:55,
 * called from matcher.py:211).  That solver is third-party and not vendored
 * (scipy 1.18.1 in this image, binary only).  Its published algorithm is the
 * shortest-augmenting-path LSAP of D. F. Crouse, "On implementing 2D
 * rectangular assignment algorithms", IEEE TAES 52(4), 2016: one Dijkstra
 * search per row over reduced costs with dual updates, columns scanned from a
 * "remaining" list initialised in reverse order and compacted by swap-removal,
 * ties on the minimum broken in favour of a free column.  This file restates
 * that algorithm for square cost matrices so the device solver
 * (paper_2111_05366_b200/csrc/lap.cu) can be checked against an independent CPU
 * statement of the same visiting order; tests/test_oracle.py pins this file to
 * scipy's binary on random, integer tie-heavy and constant matrices.
 *
 * Built by oracle/Makefile into oracle/_build/liblsap_oracle.so.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Returns 0 on success, -1 if infeasible, -2 on allocation failure.
 * cost: n*n row-major (minimisation); assign[i] = column of row i. */
int oracle_lsap_min(int64_t n, const double *cost, int64_t *assign)
{
    double *u = calloc((size_t)n, sizeof(double));
    double *v = calloc((size_t)n, sizeof(double));
    double *spc = malloc((size_t)n * sizeof(double));
    int64_t *path = malloc((size_t)n * sizeof(int64_t));
    int64_t *col4row = malloc((size_t)n * sizeof(int64_t));
    int64_t *row4col = malloc((size_t)n * sizeof(int64_t));
    int64_t *remaining = malloc((size_t)n * sizeof(int64_t));
    unsigned char *SR = malloc((size_t)n);
    unsigned char *SC = malloc((size_t)n);
    int rc = 0;
    if (!u || !v || !spc || !path || !col4row || !row4col || !remaining || !SR || !SC) {
        rc = -2;
        goto out;
    }
    for (int64_t k = 0; k < n; ++k) { col4row[k] = -1; row4col[k] = -1; path[k] = -1; }

    for (int64_t cur = 0; cur < n; ++cur) {
        /* Dijkstra from row `cur` over reduced costs. */
        double minv = 0.0;
        int64_t nrem = n;
        for (int64_t it = 0; it < n; ++it) remaining[it] = n - 1 - it;
        memset(SR, 0, (size_t)n);
        memset(SC, 0, (size_t)n);
        for (int64_t k = 0; k < n; ++k) spc[k] = INFINITY;
        int64_t i = cur, sink = -1;
        while (sink < 0) {
            int64_t pick = -1;
            double low = INFINITY;
            SR[i] = 1;
            const double *crow = cost + i * n;
            for (int64_t it = 0; it < nrem; ++it) {
                int64_t j = remaining[it];
                double r = minv + crow[j] - u[i] - v[j];
                if (r < spc[j]) { path[j] = i; spc[j] = r; }
                if (spc[j] < low || (spc[j] == low && row4col[j] == -1)) {
                    low = spc[j];
                    pick = it;
                }
            }
            minv = low;
            if (minv == INFINITY) { rc = -1; goto out; }
            int64_t j = remaining[pick];
            if (row4col[j] == -1) sink = j; else i = row4col[j];
            SC[j] = 1;
            remaining[pick] = remaining[--nrem];
        }
        /* dual update */
        u[cur] += minv;
        for (int64_t r = 0; r < n; ++r)
            if (SR[r] && r != cur) u[r] += minv - spc[col4row[r]];
        for (int64_t c = 0; c < n; ++c)
            if (SC[c]) v[c] -= minv - spc[c];
        /* augment along the alternating path */
        int64_t j = sink;
        for (;;) {
            int64_t r = path[j];
            row4col[j] = r;
            int64_t t = col4row[r]; col4row[r] = j; j = t;
            if (r == cur) break;
        }
    }
    for (int64_t k = 0; k < n; ++k) assign[k] = col4row[k];
out:
    free(u); free(v); free(spc); free(path); free(col4row); free(row4col);
    free(remaining); free(SR); free(SC);
    return rc;
}
