/* C restatement of the paircount hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * Used by tests/ (parity at sizes the numpy port cannot reach in seconds)
 * and nowhere in the product.  Pinned against the reference outputs in
 * tests/golden/ by tests/test_oracle.py.  Build: oracle/build.py
 * (gcc -O2 -fopenmp -ffp-contract=off: the predicate must not be fused).
 *
 * Reference algorithms restated (paths under /root/reference/pkg/src/paircount):
 *   row ownership, standard / balanced   spi_engine.py:102-106, pair_schedule.py:49-59
 *   collision_indicator (float64, strict <, numpy order (dx^2+dy^2)+dz^2)
 *                                        spi_engine.py:62-73
 *   softened inverse square 1/(1+d^2)    tests/test_spi_engine.py:108-111
 *   _run_outer row-range partial          spi_engine.py:109-120
 *   oracle_collisions / oracle_contacts   lattice_counter.py:227-255
 */
#include <stdint.h>
#include <stdlib.h>

static int64_t steps_for(int64_t n, int64_t i) {
    if (n & 1) return (n - 1) / 2;
    return i < n / 2 ? n / 2 : n / 2 - 1;
}

/* Row-range partial of the sphere collision count and inverse-square sum.
 * xyz: n x 3 float64, row-major.  schedule: 0 standard, 1 balanced.
 * Per-row results are combined in row order (deterministic). */
int orc_rows_f64(const double* xyz, int64_t n, int schedule, int64_t lo, int64_t hi,
                 int64_t* count_out, double* inv_sum_out, int64_t* pairs_out) {
    if (lo < 0 || hi > n || lo > hi) return 1;
    int64_t rows = hi - lo;
    int64_t* rc = (int64_t*)calloc(rows > 0 ? rows : 1, sizeof(int64_t));
    double* rs = (double*)calloc(rows > 0 ? rows : 1, sizeof(double));
    int64_t pairs = 0;
    #pragma omp parallel for schedule(dynamic, 16) reduction(+:pairs)
    for (int64_t r = 0; r < rows; ++r) {
        int64_t i = lo + r;
        int64_t m = schedule ? steps_for(n, i) : n - 1 - i;
        const double ax = xyz[3 * i], ay = xyz[3 * i + 1], az = xyz[3 * i + 2];
        int64_t c = 0;
        double s = 0.0;
        for (int64_t k = 1; k <= m; ++k) {
            int64_t j = schedule ? (i + k) % n : i + k;
            double dx = ax - xyz[3 * j], dy = ay - xyz[3 * j + 1], dz = az - xyz[3 * j + 2];
            double d2 = (dx * dx + dy * dy) + dz * dz;
            c += d2 < 1.0;
            s += 1.0 / (1.0 + d2);
        }
        rc[r] = c;
        rs[r] = s;
        pairs += m;
    }
    int64_t count = 0;
    double sum = 0.0;
    for (int64_t r = 0; r < rows; ++r) { count += rc[r]; sum += rs[r]; }
    free(rc);
    free(rs);
    *count_out = count;
    *inv_sum_out = sum;
    *pairs_out = pairs;
    return 0;
}

/* Exact-coincidence and unit-Manhattan pair counts over all i < j.
 * xyz: n x 3 int64 row-major.  numpy int64 arithmetic wraps (lattice_counter.py:
 * 238-255), so the differences and |d| are taken in uint64: no signed overflow,
 * and |INT64_MIN| wraps to 2^63 exactly as np.abs does. */
static uint64_t wrap_abs(uint64_t d) { return (d >> 63) ? (uint64_t)0 - d : d; }

int orc_int_pairs(const int64_t* xyz, int64_t n, int64_t* collisions_out, int64_t* contacts_out) {
    int64_t col = 0, con = 0;
    const uint64_t* u = (const uint64_t*)xyz;
    #pragma omp parallel for schedule(dynamic, 64) reduction(+:col, con)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = i + 1; j < n; ++j) {
            uint64_t dx = u[3 * i] - u[3 * j];
            uint64_t dy = u[3 * i + 1] - u[3 * j + 1];
            uint64_t dz = u[3 * i + 2] - u[3 * j + 2];
            if (dx == 0 && dy == 0 && dz == 0) ++col;
            uint64_t man = wrap_abs(dx) + wrap_abs(dy) + wrap_abs(dz);
            if (man == 1) ++con;
        }
    }
    *collisions_out = col;
    *contacts_out = con;
    return 0;
}

/* Row-range partial of the integer predicates under a schedule (the row
 * ownership of orc_rows_f64; lattice_counter.py:238-255 predicates). */
int orc_int_rows(const int64_t* xyz, int64_t n, int schedule, int64_t lo, int64_t hi, int64_t* collisions_out,
                 int64_t* contacts_out) {
    if (lo < 0 || hi > n || lo > hi) return 1;
    int64_t col = 0, con = 0;
    const uint64_t* u = (const uint64_t*)xyz;
    #pragma omp parallel for schedule(dynamic, 16) reduction(+:col, con)
    for (int64_t i = lo; i < hi; ++i) {
        const int64_t m = schedule ? steps_for(n, i) : n - 1 - i;
        for (int64_t k = 1; k <= m; ++k) {
            const int64_t j = schedule ? (i + k) % n : i + k;
            const uint64_t dx = u[3 * i] - u[3 * j], dy = u[3 * i + 1] - u[3 * j + 1], dz = u[3 * i + 2] - u[3 * j + 2];
            if (dx == 0 && dy == 0 && dz == 0) ++col;
            if (wrap_abs(dx) + wrap_abs(dy) + wrap_abs(dz) == 1) ++con;
        }
    }
    *collisions_out = col;
    *contacts_out = con;
    return 0;
}

/* Whole-triangle totals for the headline sizes (2^20 / 2^22 points, 5.5e11 /
 * 8.8e12 pairs): the contact count and the inverse-square sum over every pair
 * i < j with i in [lo, hi) -- the standard schedule's rows, so [0, n) is the
 * full total that every schedule and partition sums to (spi_engine.py:147-230).
 * Same predicate and term as orc_rows_f64, per pair: d2 = (dx*dx + dy*dy) +
 * dz*dz in float64 without contraction, d2 < 1.0, 1.0 / (1.0 + d2).  Only the
 * float64 summation order differs (per-row partials, then rows in order).
 * Rows are blocked 16 at a time against 2048-column chunks so a chunk stays in
 * L1/L2; with AVX-512 (tests/golden/make_full_totals.py compiles this file with
 * -O3 -march=native) the inner loop runs 8 pairs per vector. */
#ifdef __AVX512F__
#include <immintrin.h>
#endif

int orc_total_f64(const double* xyz, int64_t n, int64_t lo, int64_t hi, int64_t* count_out,
                  double* sum_out) {
    if (lo < 0 || hi > n || lo > hi) return 1;
    double* X = (double*)malloc((size_t)(n > 0 ? n : 1) * 3 * sizeof(double));
    double *Y = X + n, *Z = X + 2 * n;
    for (int64_t k = 0; k < n; ++k) { X[k] = xyz[3 * k]; Y[k] = xyz[3 * k + 1]; Z[k] = xyz[3 * k + 2]; }
    const int64_t rows = hi - lo, RB = 16, CB = 2048;
    int64_t* rc = (int64_t*)calloc(rows > 0 ? rows : 1, sizeof(int64_t));
    double* rs = (double*)calloc(rows > 0 ? rows : 1, sizeof(double));
    const int64_t nblk = (rows + RB - 1) / RB;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nblk; ++b) {
        const int64_t i0 = lo + b * RB, i1 = i0 + RB < hi ? i0 + RB : hi;
        for (int64_t c0 = i0 + 1; c0 < n; c0 += CB) {
            const int64_t c1 = c0 + CB < n ? c0 + CB : n;
            for (int64_t i = i0; i < i1; ++i) {
                int64_t j = c0 > i + 1 ? c0 : i + 1;
                if (j >= c1) continue;
                const double ax = X[i], ay = Y[i], az = Z[i];
                int64_t c = 0;
                double s = 0.0;
#ifdef __AVX512F__
                const __m512d vax = _mm512_set1_pd(ax), vay = _mm512_set1_pd(ay), vaz = _mm512_set1_pd(az);
                const __m512d one = _mm512_set1_pd(1.0);
                __m512d vs = _mm512_setzero_pd();
                __m512i vc = _mm512_setzero_si512();
                for (; j < c1; j += 8) {
                    const int64_t left = c1 - j;
                    const __mmask8 m = left >= 8 ? (__mmask8)0xff : (__mmask8)((1u << left) - 1u);
                    const __m512d dx = _mm512_sub_pd(vax, _mm512_maskz_loadu_pd(m, X + j));
                    const __m512d dy = _mm512_sub_pd(vay, _mm512_maskz_loadu_pd(m, Y + j));
                    const __m512d dz = _mm512_sub_pd(vaz, _mm512_maskz_loadu_pd(m, Z + j));
                    const __m512d d2 = _mm512_add_pd(_mm512_add_pd(_mm512_mul_pd(dx, dx), _mm512_mul_pd(dy, dy)),
                                                     _mm512_mul_pd(dz, dz));
                    const __mmask8 hit = _mm512_mask_cmp_pd_mask(m, d2, one, _CMP_LT_OQ);
                    vc = _mm512_mask_add_epi64(vc, hit, vc, _mm512_set1_epi64(1));
                    vs = _mm512_mask_add_pd(vs, m, vs, _mm512_div_pd(one, _mm512_add_pd(one, d2)));
                }
                c = _mm512_reduce_add_epi64(vc);
                s = _mm512_reduce_add_pd(vs);
#else
                for (; j < c1; ++j) {
                    const double dx = ax - X[j], dy = ay - Y[j], dz = az - Z[j];
                    const double d2 = (dx * dx + dy * dy) + dz * dz;
                    c += d2 < 1.0;
                    s += 1.0 / (1.0 + d2);
                }
#endif
                rc[i - lo] += c;
                rs[i - lo] += s;
            }
        }
    }
    int64_t count = 0;
    double sum = 0.0;
    for (int64_t r = 0; r < rows; ++r) { count += rc[r]; sum += rs[r]; }
    free(rc);
    free(rs);
    free(X);
    *count_out = count;
    *sum_out = sum;
    return 0;
}
