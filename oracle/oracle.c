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
 * xyz: n x 3 int64 row-major. */
int orc_int_pairs(const int64_t* xyz, int64_t n, int64_t* collisions_out, int64_t* contacts_out) {
    int64_t col = 0, con = 0;
    #pragma omp parallel for schedule(dynamic, 64) reduction(+:col, con)
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = i + 1; j < n; ++j) {
            int64_t dx = xyz[3 * i] - xyz[3 * j];
            int64_t dy = xyz[3 * i + 1] - xyz[3 * j + 1];
            int64_t dz = xyz[3 * i + 2] - xyz[3 * j + 2];
            if (dx == 0 && dy == 0 && dz == 0) ++col;
            uint64_t man = (uint64_t)llabs(dx) + (uint64_t)llabs(dy) + (uint64_t)llabs(dz);
            if (man == 1) ++con;
        }
    }
    *collisions_out = col;
    *contacts_out = con;
    return 0;
}
