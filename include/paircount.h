/* paircount.h -- C ABI of libpaircount.so, the B200 (sm_100a) hot path of
 * arXiv 1901.11204 ("High Performance Algorithms for Counting Collisions and
 * Pairwise Interactions").
 *
 * The reference (`paircount`, pure Python + numpy) has no FFI: its operator
 * boundary is the Python function surface.  Each entry point below is what a
 * ctypes binding of that surface binds; the reference function it replaces
 * is cited (paths under /root/reference/pkg/src/paircount/).  The Python
 * mirror in paper_1901_11204_b200/ is exactly such a binding.
 *
 * Conventions
 *   - Plain pointers and sizes only; no CUDA or torch types.  `stream` is a
 *     cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - Coordinates are n x 3, row-major (the reference's (N,3) ndarray).
 *   - Functions act on the calling thread's current CUDA device.
 *   - Return value: PC_OK (0); < 0 a CUDA failure (text in pc_last_error());
 *     > 0 a domain error mapped by the Python layer onto the reference's
 *     exception type, with detail in the result struct.
 *   - Thread-safe: library-owned scratch (the *_host entry points) is
 *     per device and mutex-guarded; everything else is stateless.
 *   - The library never frees caller memory.
 */
#ifndef PAIRCOUNT_H
#define PAIRCOUNT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ codes ---- */
#define PC_OK 0
#define PC_ERR_CUDA (-1)
#define PC_ERR_ARG 1       /* bad argument (ValueError / TypeError)                       */
#define PC_ERR_DOMAIN 2    /* counts: a non-finite coordinate -> InteractionDomainError (spi_engine.py:32-33,
                              70-71); sums: a NaN term (inf - inf or a NaN coordinate in an owned pair)
                              -> AccumulationError (spi_engine.py:93-95).  A sum with non-finite
                              coordinates but no NaN term is evaluated in float64 exactly as the
                              reference does (1/(1+inf) = 0) and returns PC_OK.                   */
#define PC_ERR_RANGE 3     /* bead outside [-a,a]^3 -> CoordinateRangeError (lattice_counter.py:31-32,98-105);
                              detail = index of the first offending bead                   */
#define PC_ERR_OVERFLOW 4  /* occupancy >= 2^32-1 -> OccupancyOverflowError (lattice_counter.py:132-135) */
#define PC_ERR_ODD 5       /* odd doubled contact sum -> ArithmeticError (lattice_counter.py:188-189) */

/* element types of the coordinate array */
#define PC_F32 0
#define PC_F64 1
#define PC_I32 2
#define PC_I64 3

/* outer-row schedules (spi_engine.py:27-29, 102-106) */
#define PC_STANDARD 0      /* Alg. 3: row i owns (i, j) for j in (i, n)                 */
#define PC_BALANCED 1      /* Alg. 4: row i owns (i, (i+s) mod n), 1 <= s <= steps_for(n, i) */

/* interactions (what the Python layer maps the reference's `f` onto) */
#define PC_COLLISION 1     /* collision_indicator: float64 |a-b|^2 < 1 (spi_engine.py:62-73)       */
#define PC_COLLISION_INVSQ 2 /* the above + sum of 1/(1+|a-b|^2) (test_spi_engine.py:108-111)        */
#define PC_COINCIDE 3      /* integer points, exact coincidence (lattice_counter.py:227-241)        */
#define PC_MANHATTAN1 4    /* integer points, Manhattan distance 1 (lattice_counter.py:244-255)     */

/* GPU tilings of the pair triangle */
#define PC_TILE_AUTO 0     /* balanced -> FLAT, standard -> PER_ROW_TILE                           */
#define PC_TILE_PER_ROW_TILE 1 /* paper's GPU scheme: one CTA per 1024-row tile walking its own
                              partner columns -- the straightforward kernel when
                              the schedule is standard                                         */
#define PC_TILE_FLAT 2     /* balanced schedule lifted to uniform tiles: the (row tile, column)
                              space of equal-length windows split evenly over a persistent grid */
#define PC_TILE_TC 3       /* the FLAT count on the tensor cores (tcgen05 Gram filter + exact
                              re-check); counts only, balanced schedule, any row ranges.
                              PC_TILE_AUTO picks it when 2^14 <= n < 2^21 and the ranges
                              cover at least n/8 rows                                          */
#define PC_TILE_SORTED 4   /* fp32 spheres on spatially (Morton) sorted points -- what
                              PC_TILE_AUTO does for a whole-range call from 2^15 points: the
                              inverse-square sum with far chunks in tile-local Gram form, and
                              the contact count with box pruning (chunks beyond contact distance
                              of the tile are decided by their boxes, not evaluated; reported in
                              pc_pairs_profile.chunks_far).  Row ranges then index the SORTED
                              order, so each range's result is a partial of the same total
                              (multi-GPU slabs), not the reference's _run_outer over those rows */
#define PC_TILE_KEY 5      /* exact coincidence counts (PC_COINCIDE, balanced) by comparing 30-bit
                              packed keys on the INT32 pipe -- points whose bounding box spans
                              <= 1023 per axis; else the result's error is PC_ERR_ARG.  The A/B
                              alternative to the FP32 Gram filter            */
#define PC_TILE_THREAD_ROW 6 /* the paper's own GPU scheme, literally: one
                              thread per outer row in 1024-row blocks, columns through shared
                              memory; with the standard schedule the straightforward kernel
                              (block- and warp-level imbalance), with the balanced one Alg. 4.
                              fp32 spheres; a baseline for the naive-vs-balanced comparison   */

typedef struct {
    int64_t count;         /* integer pair count (collisions / coincidences / contacts)           */
    double sum;            /* sum of 1/(1+|a-b|^2) over the owned pairs (PC_COLLISION_INVSQ)       */
    int64_t pairs;         /* pairs owned by the row range (closed form, spi_engine.py:113-120)    */
    int64_t exact_checks;  /* pairs re-evaluated by the exact float64/int64 predicate             */
    int32_t error;         /* PC_OK or PC_ERR_DOMAIN                                               */
    int32_t reserved;
} pc_pairs_result;

/* What the kernels of one pc_pairs* call did (pc_pairs_last_profile /
 * pc_pairs_profile_read): chunks per inner loop (a chunk = pairs_per_chunk
 * pair cells, T rows x W columns, some masked on edge chunks), rows the slow
 * path re-tested, exact re-checks, work claims.  Evidence for bench.py's
 * executed-instruction roofline; integers, identical on every run. */
typedef struct {
    int64_t chunks_gram;     /* sum on sorted points, tile-local Gram form            */
    int64_t chunks_main;     /* unmasked main loop (direct sum / Gram count filter)    */
    int64_t chunks_near;     /* sorted sum, direct formula + per-row contact minimum   */
    int64_t chunks_far;      /* sorted sum: direct formula, no contact test needed;
                                sorted count: chunks decided by their boxes (not evaluated) */
    int64_t chunks_edge;     /* masked per-pair chunks                                 */
    int64_t rows_rescanned;  /* flagged (row, chunk) re-tests by the slow path         */
    int64_t exact_checks;    /* pairs re-evaluated by the exact predicate              */
    int64_t claims;          /* FLAT work claims (float64 partial slots)               */
    int64_t pairs;           /* pairs owned by the call's rows                         */
    int64_t pairs_per_chunk; /* T x W of the kernel (0: tensor-core or no kernel)      */
    int32_t kernel;          /* 1 Gram count, 2 direct sum, 3 sorted sum, 4 compensated sum, 5 tensor-core
                                count, 6 INT32 key count, 7 thread-per-row (paper), 8 pruned sorted count,
                                9 sorted sum of float64 points, 10 sorted sum with tensor-core Gram chunks,
                                11 sorted sum of float64 points with tensor-core Gram chunks */
    int32_t f64_taken;       /* 1: the float64 kernel evaluated the sum (non-finite / huge / wide input) */
    int64_t chunks_tc;       /* sorted sum: T x W chunks evaluated on the tensor cores (pairs_tcs_kernel) */
} pc_pairs_profile;

typedef struct {
    int64_t count;         /* CountReport.count (collisions) or contacts                          */
    int64_t beads_processed;
    int64_t cells_touched; /* CountReport.cells_touched                                           */
    int64_t doubled;       /* contact_accumulator() value (contacts only)                          */
    int32_t error;         /* PC_OK, PC_ERR_RANGE, PC_ERR_OVERFLOW, PC_ERR_ODD                      */
    int32_t reserved;
    int64_t detail;        /* first bad bead index for PC_ERR_RANGE                               */
} pc_lattice_result;

/* ------------------------------------------------------- housekeeping -- */
const char* pc_last_error(void);
const char* pc_version(void);
int pc_device_count(int32_t* count);
int pc_set_device(int32_t device);
int pc_device_alloc(size_t bytes, void** ptr);           /* zero-filled */
int pc_device_free(void* ptr);
int pc_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int pc_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int pc_stream_sync(void* stream);

/* ----------------------------------------------------- all-pairs path -- */
/* Replaces spi_standard / spi_balanced (spi_engine.py:147-176),
 * spi_parallel + _partition (spi_engine.py:179-230) and the row-range
 * partial _run_outer (spi_engine.py:109-120) for collision_indicator and
 * the softened inverse square; and oracle_collisions / oracle_contacts
 * (lattice_counter.py:227-255) for integer points.
 *
 * Row ranges: nranges consecutive ranges [bounds[k], bounds[k+1]) of outer
 * rows (bounds has nranges+1 entries, non-decreasing, within [0, n]); range k
 * accumulates exactly the pairs the reference's row ownership assigns to
 * those rows under `schedule`, so per-range results equal the reference's
 * per-worker partials.  results[] has nranges entries. */

/* workspace for pc_pairs / pc_pairs_async on caller-owned device input */
size_t pc_pairs_workspace_bytes(int64_t n, int32_t nranges);

/* device input, caller workspace, results copied to host, stream synchronised */
int pc_pairs(const void* xyz, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
             int32_t tiling, int32_t nranges, const int64_t* bounds, void* workspace,
             size_t workspace_bytes, pc_pairs_result* results, void* stream);

/* as pc_pairs but asynchronous: results is a DEVICE array, nothing synchronised */
int pc_pairs_async(const void* xyz, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                   int32_t tiling, int32_t nranges, const int64_t* bounds, void* workspace,
                   size_t workspace_bytes, pc_pairs_result* results_device, void* stream);

/* host input (pageable or pinned): library-owned device scratch and stream;
 * H2D copy, compute, D2H of the results.  What the drop-in binding calls. */
int pc_pairs_host(const void* xyz_host, int32_t dtype, int64_t n, int32_t interaction,
                  int32_t schedule, int32_t tiling, int32_t nranges, const int64_t* bounds,
                  pc_pairs_result* results);

/* One part of a row range for multi-GPU work: the kernel's row tiles of
 * [lo, hi) dealt round-robin over nparts calls in blocks of four tiles
 * (blocks part, part + nparts, ...; four tiles are one origin group of the
 * tensor-core sum), so every part holds the same mix of near and far work however the
 * points are ordered (with PC_TILE_SORTED, spatially sorted).  The nparts
 * results add up to the [lo, hi) result (counts exactly).  A part is not a
 * reference worker's partial: spi_parallel partials use contiguous ranges. */
int pc_pairs_part_async(const void* xyz, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                        int32_t tiling, int64_t lo, int64_t hi, int32_t part, int32_t nparts, void* workspace,
                        size_t workspace_bytes, pc_pairs_result* result_device, void* stream);
int pc_pairs_part_host(const void* xyz_host, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                       int32_t tiling, int64_t lo, int64_t hi, int32_t part, int32_t nparts,
                       pc_pairs_result* result);

/* the profile of the last pc_pairs_host / pc_pairs_part_host call on this thread */
int pc_pairs_last_profile(pc_pairs_profile* out);
/* the profile of the last pc_pairs / pc_pairs_async / pc_pairs_part_async call on
 * this workspace (n as passed to it); synchronises `stream` */
int pc_pairs_profile_read(const void* workspace, int64_t n, pc_pairs_profile* out, void* stream);

/* Single-process multi-GPU all-pairs (SURVEY.md §8(b) pc_multi_pairs): device
 * d computes the rows [bounds[d], bounds[d+1]) of the host input (bounds[0] = 0,
 * bounds[ndev] = n; equal-work slabs as distributed.row_slabs) with
 * pc_pairs_host on devices[d], one host thread per slab; per_device[d] is
 * that slab's result and *total their sum in ascending d (count, float64 sum,
 * pairs).  The exchange is host-side: the partials are 40 bytes each.  The
 * same ordinal may repeat (slabs then run one after another).  For one
 * process per GPU use distributed.spi_distributed (NCCL all-reduce). */
int pc_pairs_multi(const void* xyz_host, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                   int32_t tiling, int32_t ndev, const int32_t* devices, const int64_t* bounds,
                   pc_pairs_result* per_device, pc_pairs_result* total);

/* All pairs of each of nvec small HOST vectors (vectors[v] -> lengths[v]
 * points, dtype as pc_pairs) in one launch: the quadratic side of the
 * reference's linear-vs-quadratic harness (bench_cli.py:129-179, one
 * oracle_collisions call per vector there).  One CTA per vector with the
 * vector in shared memory; the reference predicate in the reference's own
 * arithmetic (float64 for collision_indicator and the inverse-square sum,
 * int64 with wrap-around for the integer ones), so counts are exact.
 * results[v]: count, sum (PC_COLLISION_INVSQ), pairs = n(n-1)/2; error
 * PC_ERR_DOMAIN for non-finite coordinates, PC_ERR_ARG for a vector of more
 * than 4096 points (run it through pc_pairs_host). */
int pc_pairs_batch(const void* const* vectors, const int64_t* lengths, int32_t dtype, int32_t nvec,
                   int32_t interaction, pc_pairs_result* results, void* stream);

/* number of kernel launches the last pc_pairs* call on this thread issued */
int32_t pc_last_launch_count(void);

/* CUDA-event timing of the main all-pairs kernel of subsequent pc_pairs*
 * calls on this thread (enable resets the record); _read waits for the
 * recorded events and returns the summed kernel time and launch count. */
int pc_kernel_timing(int32_t enable);
int pc_kernel_timing_read(double* total_ms, int32_t* launches);
/* The same events split by kernel: ms[0] / launches[0] the FFMA all-pairs kernels, ms[1] /
   launches[1] the tensor-core sum kernel (pairs_tcs_kernel); both arrays of 2.  Resets. */
int pc_kernel_timing_read_split(double* ms, int32_t* launches);

/* -------------------------------------------------- counting array ---- */
/* Dense occupancy grid of side 2a+3 per axis (one zero padding cell per
 * face), uint32 cells, flat index ((x+a+1)*side + (y+a+1))*side + (z+a+1)
 * (LatticeSpace, lattice_counter.py:62-111).  The grid is caller-owned
 * device memory of pc_lattice_grid_cells(a) uint32 cells. */
int64_t pc_lattice_grid_cells(int64_t half_extent);
/* bytes per touched key (4 when the grid has < 2^32 cells, else 8) */
int32_t pc_lattice_key_bytes(int64_t half_extent);

/* Alg. 1: place beads with one atomic increment each and
 * count collisions as the sum of the pre-increment occupancies; replaces
 * count_collisions + _place (lattice_counter.py:125-156).  xyz is host
 * (xyz_on_device = 0) or device memory, dtype PC_I32/PC_I64.  keys (device,
 * n * key_bytes) receives the flat cell index of every bead -- the space's
 * touched list (lattice_counter.py:136), used by pc_lattice_reset_keys.
 * assume_clean = 1 asserts the grid was all-zero on entry (fresh or reset);
 * 0 evaluates the reference's formulas on a populated grid exactly. */
int pc_lattice_collisions(const void* xyz, int32_t dtype, int32_t xyz_on_device, int64_t n,
                          int64_t half_extent, uint32_t* grid, void* keys, int32_t assume_clean,
                          pc_lattice_result* result, void* stream);

/* Alg. 2: contacts; replaces count_contacts /
 * contact_accumulator (lattice_counter.py:159-195). */
int pc_lattice_contacts(const void* xyz, int32_t dtype, int32_t xyz_on_device, int64_t n,
                        int64_t half_extent, uint32_t* grid, void* keys, int32_t assume_clean,
                        pc_lattice_result* result, void* stream);

/* reset_sparse via the touched list (lattice_counter.py:205-210) */
int pc_lattice_reset_keys(uint32_t* grid, int64_t half_extent, const void* keys, int64_t nkeys,
                          void* stream);
/* Batched small vectors -- the paper's experiments count 100-1000 bead
 * vectors per execution (bench_cli.py:129-141 `_linear_pass`).
 * Vector v is beads [offsets[v], offsets[v+1]) of xyz (offsets: host, nvec+1
 * entries); results[v] equals count_collisions(vector, space) on a clean
 * space followed by reset_sparse -- one launch for all vectors, one CTA per
 * vector, Alg. 1 on an on-chip hashed counting array.  results[v].error:
 * PC_ERR_RANGE (detail = first bad bead within the vector) or PC_ERR_ARG for
 * a vector longer than 4096 beads, which the caller counts through a grid. */
int pc_lattice_collisions_batch(const void* xyz, int32_t dtype, int32_t xyz_on_device, const int64_t* offsets,
                                int32_t nvec, int64_t half_extent, pc_lattice_result* results, void* stream);
/* Same as pc_lattice_collisions_batch for nvec separate HOST vectors
 * (vectors[v] -> lengths[v] beads of (x,y,z), int32 or int64), as the
 * reference's _linear_pass holds them (bench_cli.py:129-141): the library
 * gathers them with host threads into pinned staging, narrowing int64 to
 * int32 (a coordinate outside [-a,a] maps to INT32_MAX, still out of range,
 * so PC_ERR_RANGE names the same first bad bead), then one H2D copy and one
 * launch.  half_extent < INT32_MAX. */
int pc_lattice_collisions_vectors(const void* const* vectors, const int64_t* lengths, int32_t dtype, int32_t nvec,
                                  int64_t half_extent, pc_lattice_result* results, void* stream);

/* count_collisions over several GPUs of one process (the
 * counting array split by key range).  Device d owns the x-planes
 * [-a + P*d/ndev, -a + P*(d+1)/ndev), P = 2a+1, on a private slab grid of
 * (planes+2) x (2a+3)^2 cells; it copies all host beads in, validates every
 * bead (PC_ERR_RANGE, detail = first bad bead, identical on every device),
 * compacts its own beads and runs Alg. 1 on them.  Cells of different
 * devices are disjoint, so *total = the sums of count and cells_touched =
 * count_collisions(beads, new_space(a)) on one grid.  The slab grids are left
 * zero; no LatticeSpace is involved.  The same ordinal may repeat. */
int pc_lattice_collisions_multi(const void* xyz_host, int32_t dtype, int64_t n, int64_t half_extent, int32_t ndev,
                                const int32_t* devices, pc_lattice_result* per_device, pc_lattice_result* total);

/* Zero the whole grid with one streaming write (cudaMemsetAsync).  The
 * Python reset_sparse uses it in place of pc_lattice_reset_keys when the
 * touched keys number more than 1/32 of the cells AND every other cell is
 * known to be zero -- then both leave the identical all-zero grid, and the
 * streaming write beats 32-byte-sector scattered stores. */
int pc_lattice_clear(uint32_t* grid, int64_t half_extent, void* stream);
/* reset_sparse via beads: each bead's cell and its six neighbours
 * (lattice_counter.py:211-217); PC_ERR_RANGE if a bead is outside [-a,a]^3 */
int pc_lattice_reset_beads(const void* xyz, int32_t dtype, int32_t xyz_on_device, int64_t n,
                           int64_t half_extent, uint32_t* grid, pc_lattice_result* result,
                           void* stream);
/* LatticeSpace.is_zero (lattice_counter.py:95-96): *nonzero = number of nonzero cells */
int pc_grid_count_nonzero(const uint32_t* grid, int64_t cells, int64_t* nonzero, void* stream);

/* ---------------------------------------------------------- evidence -- */
/* FP32 pipe micro-benchmark: lane-instructions per second of a dependent-
 * free 3-register FFMA stream over all SMs (kind 0), or of the all-pairs
 * inner loop (kind 1: 3 FFMA + 1/2 FMNMX3 per pair, reported as pairs/s).
 * Used by bench.py as the measured roofline denominator. */
int pc_microbench(int32_t kind, double* per_second, double* seconds);

#ifdef __cplusplus
}
#endif
#endif /* PAIRCOUNT_H */
