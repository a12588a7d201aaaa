/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the exact top-k
 * maximum-inner-product search that SearchAgent-X's retriever performs
 * (§2.1 "exact nearest neighbor (ENN) search"; the
 * vLLM_ENN baseline "exhaustive search", App. B.3; top-k documents
 * concatenated into the context).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  It shares no code, header, table or
 * constant with paper_2505_12065_b200/ (the CUDA path), and never calls it.
 *
 * Definitions (readings R1-R6):
 *   - inputs are the bf16 values the library stores (RNE from fp32, R3),
 *     widened exactly to double;
 *   - s_i = sum_{j<d} q_j * x_{i,j}, summed sequentially in j, in double (R1);
 *   - rank by (s descending, global id ascending) (R5), -0.0 == +0.0;
 *   - return the first min(k, n) entries, pad with (id -1, score -INF) (R6).
 *
 * Pins: tests/test_oracle_pins.py (P1-P6, P9 of SURVEY.md §8(c)).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* bf16 bits -> double, exact (a bf16 is the top half of an IEEE binary32). */
static double bf16_to_double(uint16_t b)
{
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* IEEE binary32 -> bf16, round to nearest, ties to even (reading R3).
 * Textbook definition: add 0x7FFF plus the lsb of the kept half, truncate.
 * NaN stays NaN (quietened).  Pinned against torch's cast in the tests. */
void oracle_bf16_round(const float *x, uint16_t *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) {
        uint32_t u;
        memcpy(&u, &x[i], sizeof u);
        if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) {
            out[i] = (uint16_t)((u >> 16) | 0x0040u);
            continue;
        }
        uint32_t lsb = (u >> 16) & 1u;
        u += 0x7FFFu + lsb;
        out[i] = (uint16_t)(u >> 16);
    }
}

/* One inner product in double, summed in index order. */
double oracle_dot(const uint16_t *q, const uint16_t *x, int32_t d)
{
    double s = 0.0;
    for (int32_t j = 0; j < d; ++j)
        s += bf16_to_double(q[j]) * bf16_to_double(x[j]);
    return s;
}

/* Does (s, id) rank strictly before (t, jd)?  Empty slots (jd < 0) rank last. */
static int ranks_before(double s, int64_t id, double t, int64_t jd)
{
    if (jd < 0) return 1;
    if (s > t) return 1;
    if (s < t) return 0;
    return id < jd;
}

/* Initialise nq running lists of length kk to (-1, -INF). */
void oracle_topk_init(int64_t nq, int32_t kk, int64_t *ids, double *scores)
{
    for (int64_t i = 0; i < nq * (int64_t)kk; ++i) {
        ids[i] = -1;
        scores[i] = -INFINITY;
    }
}

/*
 * Fold rows [0, n) of a corpus chunk, whose first row has global id `id0`,
 * into the running top-kk lists of nq queries.
 *   X      bf16 bits [n, d] row-major          Q   bf16 bits [nq, d] row-major
 *   ids    int64 [nq, kk] running list (in/out), sorted by rank
 *   scores double [nq, kk] running list (in/out)
 * Each query's list is updated by plain insertion, one row at a time, so
 * calling this over consecutive chunks equals one call over their union.
 */
void oracle_topk_update(const uint16_t *X, int64_t n, int32_t d, int64_t id0,
                        const uint16_t *Q, int64_t nq, int32_t kk,
                        int64_t *ids, double *scores)
{
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < nq; ++qi) {
        const uint16_t *q = Q + qi * (int64_t)d;
        int64_t *li = ids + qi * (int64_t)kk;
        double *ls = scores + qi * (int64_t)kk;
        for (int64_t i = 0; i < n; ++i) {
            double s = oracle_dot(q, X + i * (int64_t)d, d);
            int64_t id = id0 + i;
            if (!ranks_before(s, id, ls[kk - 1], li[kk - 1]))
                continue;
            int32_t p = kk - 1;
            while (p > 0 && ranks_before(s, id, ls[p - 1], li[p - 1])) {
                ls[p] = ls[p - 1];
                li[p] = li[p - 1];
                --p;
            }
            ls[p] = s;
            li[p] = id;
        }
    }
}

/* Convenience: the whole definition in one call (init + one update). */
void oracle_flat_topk(const uint16_t *X, int64_t n, int32_t d,
                      const uint16_t *Q, int64_t nq, int32_t k,
                      int64_t *ids, double *scores)
{
    oracle_topk_init(nq, k, ids, scores);
    oracle_topk_update(X, n, d, 0, Q, nq, k, ids, scores);
}

/* Scores of explicitly listed (query, row) pairs, for sampled checks at full
 * size:  out[p] = s(Q[qidx[p]], X[ridx[p]]). */
void oracle_pair_scores(const uint16_t *X, int32_t d, const uint16_t *Q,
                        const int64_t *qidx, const int64_t *ridx, int64_t npairs,
                        double *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npairs; ++p)
        out[p] = oracle_dot(Q + qidx[p] * (int64_t)d, X + ridx[p] * (int64_t)d, d);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
