// libpaircount.so -- sm_100a kernels and the C ABI of include/paircount.h.
//
// Hot path (BASELINE.json north_star):
//   * all-pairs count over the i<j triangle under the reference's two outer
//     schedules (standard = Alg. 3, balanced = Alg. 4; spi_engine.py:102-106,
//     pair_schedule.py:49-59), exact for collision_indicator
//     (spi_engine.py:62-73) and the integer oracles (lattice_counter.py:
//     227-255), plus the softened inverse-square sum;
//   * the O(N) counting array (Alg. 1/2; lattice_counter.py:125-217).
//
// Files (one translation unit):
//   paircount.cu      helpers, prep kernels (bounding box, pair-array staging),
//                     all-pairs host driver, per-device arena, the C ABI
//   pairs_kernel.cuh  the all-pairs kernel: warp-private row tiles, packed
//                     FP32 Gram filter (count) / direct formula (sum), exact
//                     re-check slow path, FLAT uniform tiles with dynamic claims;
//                     SORTED: the sum on Morton-sorted points (sort kernels in
//                     this file) with tile-local Gram chunks
//   pairs_tc.cuh      the count filter on the tensor cores: tcgen05.mma tf32
//                     (3xTF32) into TMEM, warp-specialised loader / MMA /
//                     drain warps, candidate queues + exact pass
//   pairs_tcsum.cuh   the sorted sum's Gram chunks on the tensor cores:
//                     chunk bitmap, tcgen05.mma kind::f16 on three-way bf16
//                     splits (operands built in shared memory per item), TMEM
//                     drained with eight terms per two reciprocals
//   pairs_key.cuh     exact coincidences by 30-bit keys on the INT32 pipe
//   pairs_row.cuh     the paper's thread-per-row schemes (a baseline)
//   lattice.cuh       counting-array kernels (sparse regime) and the driver
//   lattice_slab.cuh  dense regime: key partition + shared-memory slabs + TMA
//                     bulk stores
//   batch.cuh         many small vectors in one launch (counting array and
//                     all-pairs), host gather into pinned staging
//
// DESIGN.md §3 has the arithmetic (error bands, compensated staging), the
// instruction-dispatch model the loops are tuned against, and measurements.

#include "../../include/paircount.h"

#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;

// Optional CUDA-event timing of the main all-pairs kernel (bench.py's
// roofline needs that kernel's own duration, on the stream it runs on).
struct EvPair {
    cudaEvent_t a, b;
    int kind;  // 0: FFMA all-pairs kernels, 1: the tensor-core sum kernel (pairs_tcs_kernel)
};
thread_local bool g_timing = false;
thread_local EvPair g_ev[4096];
thread_local int g_ev_used = 0, g_ev_made = 0;

int cuda_fail(const char* what, cudaError_t e) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return PC_ERR_CUDA;
}
int arg_fail(const char* what) {
    g_err = what;
    return PC_ERR_ARG;
}

#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return cuda_fail(#call, e_);       \
    } while (0)
#define CK_LAUNCH(what)                                           \
    do {                                                          \
        ++g_launches;                                             \
        cudaError_t e_ = cudaGetLastError();                      \
        if (e_ != cudaSuccess) return cuda_fail(what, e_);        \
    } while (0)

constexpr int kPredSphere = 0, kPredCoincide = 1, kPredManhattan1 = 2;

// Checked build (python -m paper_1901_11204_b200.build --checked -> build/checked/): device-side
// bounds checks on every index the kernels compute for global memory and claim slots; a violation
// traps (the call fails with PC_ERR_CUDA) instead of corrupting memory.  compute-sanitizer is
// closed on the GPU pool, so scripts/sanitize_cases.py runs this build, with poisoned scratch
// (PAIRCOUNT_POISON) and canaries around caller buffers, as the memory-safety evidence.
#ifndef PC_CHECKED
#define PC_CHECKED 0
#endif
#define PC_CHECK(cond)                         \
    do {                                       \
        if (PC_CHECKED && !(cond)) __trap();   \
    } while (0)

// ------------------------------------------------------------------------
// small device helpers
// ------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long enc_f64(double d) {
    unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double dec_f64(unsigned long long e) {
    unsigned long long b = (e >> 63) ? (e & 0x7fffffffffffffffull) : ~e;
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}
// ordered code 0 (memset value) means "no point seen": decode as 0.0
__host__ __device__ __forceinline__ double dec_f64_or0(unsigned long long e) { return e ? dec_f64(e) : 0.0; }
__device__ __forceinline__ unsigned long long enc_i64(long long v) {
    return (unsigned long long)v ^ 0x8000000000000000ull;
}
__host__ __device__ __forceinline__ long long dec_i64(unsigned long long e) {
    return (long long)(e ^ 0x8000000000000000ull);
}

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// coordinate k of point i, as double / int64
__device__ __forceinline__ double coord_f64(const void* xyz, int dtype, long long i, int k) {
    switch (dtype) {
        case PC_F32: return (double)((const float*)xyz)[3 * i + k];
        case PC_F64: return ((const double*)xyz)[3 * i + k];
        case PC_I32: return (double)((const int*)xyz)[3 * i + k];
        default: return (double)((const long long*)xyz)[3 * i + k];
    }
}
__device__ __forceinline__ long long coord_i64(const void* xyz, int dtype, long long i, int k) {
    return dtype == PC_I32 ? (long long)((const int*)xyz)[3 * i + k]
                           : ((const long long*)xyz)[3 * i + k];
}

// The reference predicates, evaluated exactly as the reference evaluates them.
__device__ bool exact_pair(const void* xyz, int dtype, int pred, long long i, long long j) {
    if (pred == kPredSphere) {
        // collision_indicator (spi_engine.py:68-73): float64 upcast,
        // d2 = ((a-b)**2).sum(-1) in numpy order (dx^2 + dy^2) + dz^2, no FMA,
        // strict < 1.0.
        double dx = __dsub_rn(coord_f64(xyz, dtype, i, 0), coord_f64(xyz, dtype, j, 0));
        double dy = __dsub_rn(coord_f64(xyz, dtype, i, 1), coord_f64(xyz, dtype, j, 1));
        double dz = __dsub_rn(coord_f64(xyz, dtype, i, 2), coord_f64(xyz, dtype, j, 2));
        double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        return d2 < 1.0;
    }
    long long d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        d[k] = (long long)((unsigned long long)coord_i64(xyz, dtype, i, k) -
                           (unsigned long long)coord_i64(xyz, dtype, j, k));
    if (pred == kPredCoincide) return d[0] == 0 && d[1] == 0 && d[2] == 0;  // lattice_counter.py:238-241
    // Manhattan == 1 with numpy int64 wrap-around semantics (lattice_counter.py:252-255)
    unsigned long long man = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) man += (unsigned long long)(d[k] < 0 ? -d[k] : d[k]);
    return man == 1ull;
}
__device__ __noinline__ bool exact_pair_call(const void* xyz, int dtype, int pred, long long i, long long j) {
    return exact_pair(xyz, dtype, pred, i, j);
}

// ------------------------------------------------------------------------
// preparation: bounding box, centring, float4 staging, error bands
// ------------------------------------------------------------------------
struct PrepStats {
    unsigned long long mn[3], mx[3];  // ordered encodings (f64 for float input, i64 for int input)
    unsigned long long maxabs;        // ordered f64: max |coordinate| (raw)
    unsigned long long mnorm;         // ordered f64: max |q|^2 of the staged fp32 coordinates
    int nonfinite;
    int pad;
    unsigned long long work_ctr;
};

__device__ __forceinline__ bool is_int_dtype(int dtype) { return dtype >= PC_I32; }

__global__ void prep_bbox_kernel(const void* __restrict__ xyz, int dtype, long long n,
                                 PrepStats* __restrict__ st) {
    const bool isint = is_int_dtype(dtype);
    unsigned long long mn[3], mx[3];
    double maxabs = 0.0;
    int bad = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) { mn[k] = ~0ull; mx[k] = 0ull; }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            unsigned long long e;
            if (isint) {
                long long v = coord_i64(xyz, dtype, i, k);
                e = enc_i64(v);
                maxabs = fmax(maxabs, fabs((double)v));
            } else {
                double v = coord_f64(xyz, dtype, i, k);
                if (!isfinite(v)) { bad = 1; v = 0.0; }
                e = enc_f64(v);
                maxabs = fmax(maxabs, fabs(v));
            }
            mn[k] = mn[k] < e ? mn[k] : e;
            mx[k] = mx[k] > e ? mx[k] : e;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            unsigned long long a = __shfl_xor_sync(0xffffffffu, mn[k], o);
            unsigned long long b = __shfl_xor_sync(0xffffffffu, mx[k], o);
            mn[k] = mn[k] < a ? mn[k] : a;
            mx[k] = mx[k] > b ? mx[k] : b;
        }
        maxabs = fmax(maxabs, __shfl_xor_sync(0xffffffffu, maxabs, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            atomicMin(&st->mn[k], mn[k]);
            atomicMax(&st->mx[k], mx[k]);
        }
        atomicMax(&st->maxabs, enc_f64(maxabs));
        if (bad) atomicOr(&st->nonfinite, 1);
    }
}

// Centre of the bounding box; for integer input an exact int64 midpoint so
// p - centre is exact (SURVEY.md hard part 1 / DESIGN.md "error band").
__device__ __forceinline__ void bbox_centre(const PrepStats& st, int dtype, double c[3], long long ci[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (is_int_dtype(dtype)) {
            long long lo = dec_i64(st.mn[k]), hi = dec_i64(st.mx[k]);
            ci[k] = lo + (long long)(((unsigned long long)hi - (unsigned long long)lo) >> 1);
            c[k] = 0.0;
        } else {
            c[k] = 0.5 * dec_f64(st.mn[k]) + 0.5 * dec_f64(st.mx[k]);
            ci[k] = 0;
        }
    }
}

// Largest per-axis extent of the bounding box (float64).
__device__ __forceinline__ double bbox_span(const PrepStats& st, int dtype) {
    double e = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double d = is_int_dtype(dtype) ? (double)dec_i64(st.mx[k]) - (double)dec_i64(st.mn[k])
                                             : dec_f64(st.mx[k]) - dec_f64(st.mn[k]);
        e = fmax(e, d);
    }
    return e;
}
// The compensated (hi + lo) sum keeps each term within 4u + 2u^2*E relative; beyond
// this span that passes 1e-7 and the sum takes pairs_f64_kernel instead.
constexpr double kCompMaxSpan = 67108864.0;  // 2^26

// Inverse-square sums the float64 kernel (pairs_f64_kernel) evaluates instead of the fp32
// kernels, decided on the device from the prep statistics (no host synchronisation):
//   * a non-finite coordinate: every term is then the reference's own float64 value --
//     1/(1+inf) = 0 for a pair with an isolated inf, NaN where inf - inf or a NaN enters
//     (spi_engine.py:84-99: the host layer turns a NaN sum into AccumulationError);
//   * |coordinate| >= 1e18, where fp32 squares overflow;
//   * a compensated (non-f32) call whose span defeats the hi + lo staging.
__device__ __forceinline__ bool f64_takes(const PrepStats& st, int dtype, bool comp) {
    return st.nonfinite || !(dec_f64_or0(st.maxabs) < 1e18) || (comp && bbox_span(st, dtype) > kCompMaxSpan);
}

// Staged value of point i: centred fp32 q and w = -|q|^2/2 (Gram), or the
// raw fp32 coordinates (direct formula).
template <bool DIRECT>
__device__ __forceinline__ float4 staged_point(const void* xyz, int dtype, long long i, const double c[3],
                                               const long long ci[3], double* nq_out) {
    float q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (DIRECT) {
            q[k] = (float)coord_f64(xyz, dtype, i, k);  // raw coordinates: exact for fp32 input
        } else if (is_int_dtype(dtype)) {
            long long v = (long long)((unsigned long long)coord_i64(xyz, dtype, i, k) - (unsigned long long)ci[k]);
            q[k] = (float)(double)v;
        } else {
            q[k] = (float)(coord_f64(xyz, dtype, i, k) - c[k]);
        }
    }
    double nq = (double)q[0] * q[0] + (double)q[1] * q[1] + (double)q[2] * q[2];
    if (!(nq <= 1e300)) nq = INFINITY;
    *nq_out = nq;
    return make_float4(q[0], q[1], q[2], DIRECT ? 0.0f : (float)(-0.5 * nq));
}

// Compensated staging (direct formula, non-f32 input): the centred coordinate
// q = p - c (exact int64 difference for integer input) as the unevaluated
// fp32 sum hi + lo, so pair separations survive however far the points sit
// from the centre (fp32 rounding of q alone would cost u*|q| absolute).
__device__ __forceinline__ void staged_point_comp(const void* xyz, int dtype, long long i, const double c[3],
                                                  const long long ci[3], float h[3], float l[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double q;
        if (is_int_dtype(dtype))
            q = (double)(long long)((unsigned long long)coord_i64(xyz, dtype, i, k) - (unsigned long long)ci[k]);
        else
            q = coord_f64(xyz, dtype, i, k) - c[k];
        h[k] = (float)q;
        l[k] = (float)(q - (double)h[k]);
    }
}

// Pair arrays for packed FP32: entry j>>1 of `even` (j even) / `odd` (j odd)
// holds points j and (j+1) mod n interleaved as (x_j, x_j1, y_j, y_j1),
// (z_j, z_j1, w_j, w_j1) -- or, COMP, (xh, xh1, yh, yh1)(zh, zh1, xl, xl1)
// (yl, yl1, zl, zl1).  Thread per j; every point is staged twice.
template <bool DIRECT, bool COMP>
__global__ void prep_stage_kernel(const void* __restrict__ xyz, int dtype, long long n,
                                  PrepStats* __restrict__ st, float4* __restrict__ even, float4* __restrict__ odd) {
    double c[3];
    long long ci[3];
    bbox_centre(*st, dtype, c, ci);
    double mnorm = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (COMP) {
            float h0[3], l0[3], h1[3], l1[3];
            staged_point_comp(xyz, dtype, i, c, ci, h0, l0);
            staged_point_comp(xyz, dtype, i + 1 == n ? 0 : i + 1, c, ci, h1, l1);
            float4* dst = ((i & 1) ? odd : even) + 3 * (i >> 1);
            dst[0] = make_float4(h0[0], h1[0], h0[1], h1[1]);
            dst[1] = make_float4(h0[2], h1[2], l0[0], l1[0]);
            dst[2] = make_float4(l0[1], l1[1], l0[2], l1[2]);
            continue;
        }
        double nq, nq1;
        const float4 p = staged_point<DIRECT>(xyz, dtype, i, c, ci, &nq);
        const float4 p1 = staged_point<DIRECT>(xyz, dtype, i + 1 == n ? 0 : i + 1, c, ci, &nq1);
        mnorm = fmax(mnorm, nq);
        float4* dst = ((i & 1) ? odd : even) + 2 * (i >> 1);
        dst[0] = make_float4(p.x, p1.x, p.y, p1.y);
        dst[1] = make_float4(p.z, p1.z, p.w, p1.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mnorm = fmax(mnorm, __shfl_xor_sync(0xffffffffu, mnorm, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&st->mnorm, enc_f64(mnorm));
}

// ------------------------------------------------------------------------
// the all-pairs kernel
// ------------------------------------------------------------------------
// One record per CTA.  path[] counts the chunks each inner loop evaluated (kPath*), the
// evidence behind the bench's executed-instruction roofline; rescans counts the rows the
// slow path re-tested.  All integer: the order CTAs finish in cannot change them.
constexpr int kPathGram = 0;   // sum on sorted points: tile-local Gram form
constexpr int kPathMain = 1;   // unmasked main loop: direct formula (sum) / Gram filter (count)
constexpr int kPathNear = 2;   // sum on sorted points: direct formula + per-row minimum (contact test)
constexpr int kPathFar = 3;    // sum on sorted points: direct formula, boxes too far apart for a contact
constexpr int kPathEdge = 4;   // masked per-pair chunk (leading / trailing / ragged)
constexpr int kNumPaths = 5;
struct Slot {
    unsigned long long count;
    unsigned long long checks;
    double sum;
    unsigned path[kNumPaths];
    unsigned rescans;
    unsigned pad[4];  // pad[0]: chunks the tensor-core sum kernel evaluated
};
static_assert(sizeof(Slot) == 64, "Slot is one 64-byte record");
// kernel ids recorded in pc_pairs_profile.kernel
constexpr int kKernGram = 1, kKernDirect = 2, kKernSorted = 3, kKernComp = 4, kKernTc = 5, kKernKey = 6,
              kKernRow = 7, kKernSortedCount = 8, kKernCompSorted = 9, kKernSortedTc = 10, kKernCompSortedTc = 11;

// FLAT work claims (guided self-scheduling): claim c of stage k covers columns
// [b0[k] + (c - c0[k]) * s[k], + s[k]) of the flat (row tile, window column) space.  Stage k
// hands out P claims (P = the grid's warps) of half the remaining work split P ways, the last
// stage single chunks, so the tail is one chunk and a claim's index is a fixed function of
// its columns: the float64 sum of claim c goes to claim_sums[c] and the finalize adds those
// in index order -- bit-reproducible sums whichever warp ran which claim.
#ifndef PC_GUIDED
#define PC_GUIDED 1
#endif
#ifndef PC_CLAIM_MAX
#define PC_CLAIM_MAX 16
#endif
constexpr int kMaxStages = 48;
#ifndef PC_CLAIMS_CAP
#define PC_CLAIMS_CAP (1 << 20)
#endif
constexpr long long kClaimsCap = PC_CLAIMS_CAP;

struct PairsArgs {
    const float4* pts_even;  // pair arrays, see prep_stage_kernel
    const float4* pts_odd;
    const void* xyz;
    const PrepStats* st;
    Slot* slots;
    unsigned long long* work_ctr;  // FLAT: super-chunk claim counter (zeroed per launch)
    int dtype, pred, sched;
    float thr;
    int n, lo, hi;      // n < 2^31 enforced on the host
    int n_tiles;        // row tiles in [lo, hi)
    long long L;        // FLAT: window length shared by every row tile
    long long total;    // FLAT: n_tiles * L
    const float4* blk_box;   // SORTED: per-32-point bounding boxes (min, max) of the sorted points
    const float4* blk2_box;  // SORTED count: per-1024-point boxes
    int nblk;
    int tstride, toff;   // row tiles of this call: toff, toff + tstride, ... (pc_pairs_part_async)
    int tile_rows;       // T of the launched kernel (the float64 kernel follows the same tiles)
    double* claim_sums;  // FLAT direct: one float64 partial per claim
    int nstage;          // FLAT: claim stages (see kMaxStages)
    long long blk_cols;  // FLAT: columns per block of the transposed claim order (pairs_kernel.cuh)
    long long win_blks;  // FLAT: blocks per tile window
    long long st_c0[kMaxStages + 1], st_b0[kMaxStages], st_s[kMaxStages];
    int tc_split;        // SORTED sum: the dense chunks tcs_takes() accepts are left to pairs_tcs_kernel
    const unsigned* tc_bits;  // ... marked in this bitmap (bit t * tc_cpw_pad + chunk), or null: decided in-loop
    long long tc_cpw_pad;
};

__device__ __forceinline__ int steps_for_dev(int n, int i) {
    // pair_schedule.py:49-59
    if (n & 1) return (n - 1) >> 1;
    return i < (n >> 1) ? (n >> 1) : (n >> 1) - 1;
}

#include "pairs_kernel.cuh"
#include "pairs_tc.cuh"
#include "pairs_tcsum.cuh"
#include "pairs_tcs2.cuh"
#include "pairs_key.cuh"
#include "pairs_row.cuh"

// First stage of the claim-sum reduction for large claim counts: block b adds claims
// [b*per, (b+1)*per) in a fixed thread partition and tree -- a fixed association, so the
// finalize's total stays bit-reproducible; one block for 2^18 claims took 0.3 ms.
constexpr int kRedBlocks = 128;
__global__ void claims_reduce_kernel(const double* __restrict__ claims, int nclaims, double* __restrict__ red) {
    __shared__ double ss[256];
    const int per = (nclaims + kRedBlocks - 1) / kRedBlocks;
    const int b0 = blockIdx.x * per, b1 = min(nclaims, b0 + per);
    double s = 0.0;
    for (int q = b0 + threadIdx.x; q < b1; q += blockDim.x) s += claims[q];
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) ss[threadIdx.x] += ss[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) red[blockIdx.x] = ss[0];
}

// Fixed-order sum of the CTA slots and the claim partials into one result record (one
// block of 256 threads, a fixed partition and tree: the float64 sum is bit-reproducible),
// and the call's path counters added into the workspace's profile record.
__global__ void finalize_kernel(const Slot* __restrict__ slots, int nslots, const double* __restrict__ claims,
                                int nclaims, int claims_hold_sums, int claims_total, const PrepStats* __restrict__ st,
                                int dtype,
                                long long pairs, int direct,
                                pc_pairs_result* __restrict__ out, pc_pairs_profile* __restrict__ prof,
                                int kernel_id, long long pairs_per_chunk) {
    __shared__ unsigned long long sc[256], sk[256], sp[kNumPaths + 1][256];
    __shared__ double ss[256];
    __shared__ unsigned long long stc[256];
    unsigned long long c = 0, k = 0, pth[kNumPaths + 1] = {0, 0, 0, 0, 0, 0}, tcc = 0;
    double s = 0.0;
    for (int q = threadIdx.x; q < nslots; q += blockDim.x) {
        c += slots[q].count;
        k += slots[q].checks;
        s += slots[q].sum;
        for (int u = 0; u < kNumPaths; ++u) pth[u] += slots[q].path[u];
        pth[kNumPaths] += slots[q].rescans;
        tcc += slots[q].pad[0];
    }
    if (claims_hold_sums)
        for (int q = threadIdx.x; q < nclaims; q += blockDim.x) s += claims[q];
    sc[threadIdx.x] = c; sk[threadIdx.x] = k; ss[threadIdx.x] = s; stc[threadIdx.x] = tcc;
    for (int u = 0; u <= kNumPaths; ++u) sp[u][threadIdx.x] = pth[u];
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
            sc[threadIdx.x] += sc[threadIdx.x + h];
            stc[threadIdx.x] += stc[threadIdx.x + h];
            sk[threadIdx.x] += sk[threadIdx.x + h];
            ss[threadIdx.x] += ss[threadIdx.x + h];
            for (int u = 0; u <= kNumPaths; ++u) sp[u][threadIdx.x] += sp[u][threadIdx.x + h];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pc_pairs_result r;
        r.count = (long long)sc[0];
        r.sum = ss[0];
        r.pairs = pairs;
        r.exact_checks = (long long)sk[0];
        // counts: a non-finite coordinate is InteractionDomainError (collision_indicator,
        // spi_engine.py:70-71); sums: the float64 kernel evaluated the reference's terms and a
        // NaN among them is AccumulationError (spi_engine.py:93-95)
        r.error = direct ? (isnan(ss[0]) ? PC_ERR_DOMAIN : PC_OK) : (st->nonfinite ? PC_ERR_DOMAIN : PC_OK);
        if (kernel_id == kKernKey && st->pad) r.error = PC_ERR_ARG;  // span > 1023: no 30-bit key
        r.reserved = 0;
        *out = r;
        prof->chunks_gram += (long long)sp[kPathGram][0];
        prof->chunks_main += (long long)sp[kPathMain][0];
        prof->chunks_near += (long long)sp[kPathNear][0];
        prof->chunks_far += (long long)sp[kPathFar][0];
        prof->chunks_edge += (long long)sp[kPathEdge][0];
        prof->chunks_tc += (long long)stc[0];
        prof->rows_rescanned += (long long)sp[kNumPaths][0];
        prof->exact_checks += (long long)sk[0];
        prof->claims += claims_total;
        prof->pairs += pairs;
        prof->pairs_per_chunk = pairs_per_chunk;
        prof->kernel = kernel_id;
        if (direct && f64_takes(*st, dtype, direct == 2)) prof->f64_taken = 1;
    }
}

// Sum + count in float64 for the calls f64_takes() routes here (non-finite
// coordinates, |c| >= 1e18, or a non-f32 span the compensated staging cannot hold):
// every owned pair with the reference's own arithmetic -- the count as
// collision_indicator (spi_engine.py:68-73), the term 1/(1+d2) as the softened
// inverse square.  Always launched after the fp32 kernel of a sum call; exactly one
// of the two does the work (both read the prep statistics), the other writes zero
// slots.  Rows follow the fp32 kernel's tiles (tile_rows, tstride, toff).
__global__ void __launch_bounds__(256) pairs_f64_kernel(const PairsArgs a, int comp, Slot* __restrict__ slots) {
    __shared__ unsigned long long s_c[8];
    __shared__ double s_s[8];
    const bool wide = f64_takes(*a.st, a.dtype, comp != 0);
    unsigned long long cnt = 0;
    double sum = 0.0;
    if (wide) {
        const bool bal = a.sched == PC_BALANCED;
        for (long long i = a.lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.hi;
             i += (long long)gridDim.x * blockDim.x) {
            if (a.tstride > 1 && ((i - a.lo) / a.tile_rows / kTcsOrgG) % a.tstride != a.toff) continue;
            const long long m = bal ? steps_for_dev(a.n, (int)i) : (long long)a.n - 1 - i;
            const double xi = coord_f64(a.xyz, a.dtype, i, 0), yi = coord_f64(a.xyz, a.dtype, i, 1),
                         zi = coord_f64(a.xyz, a.dtype, i, 2);
            for (long long s = 1; s <= m; ++s) {
                long long j = i + s;
                if (j >= a.n) j -= a.n;
                PC_CHECK(j >= 0 && j < a.n && i < a.n);
                const double dx = __dsub_rn(xi, coord_f64(a.xyz, a.dtype, j, 0));
                const double dy = __dsub_rn(yi, coord_f64(a.xyz, a.dtype, j, 1));
                const double dz = __dsub_rn(zi, coord_f64(a.xyz, a.dtype, j, 2));
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                cnt += d2 < 1.0 ? 1ull : 0ull;
                sum += 1.0 / (1.0 + d2);
            }
        }
    }
    cnt = warp_sum(cnt);
    sum = warp_sum(sum);
    if ((threadIdx.x & 31) == 0) {
        s_c[threadIdx.x >> 5] = cnt;
        s_s[threadIdx.x >> 5] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Slot sl{};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            sl.count += s_c[w];
            sl.sum += s_s[w];
        }
        sl.checks = sl.count;
        slots[blockIdx.x] = sl;
    }
}

// ------------------------------------------------------------------------
// host side of the all-pairs path
// ------------------------------------------------------------------------
struct KernelCfg {
    int warps, r, w;
};
#ifndef PC_BIG_R
#define PC_BIG_R 8
#endif
#ifndef PC_BIG_W
#define PC_BIG_W 256
#endif
constexpr KernelCfg kBig{4, PC_BIG_R, PC_BIG_W};  // direct (sum) kernel: warp tile 32*R rows (256 by default)
#ifndef PC_SORTED_SUM
#define PC_SORTED_SUM 1  // whole-range fp32 balanced sums: spatial sort + tile-local Gram chunks
#endif
#ifndef PC_SORTED_COUNT
#define PC_SORTED_COUNT 1  // whole-range fp32 balanced contact counts: spatial sort + box pruning
#endif
#ifndef PC_TC_AUTO
#define PC_TC_AUTO 1  // balanced counts with kTcMinN <= n < kTcMaxN (rows >= n/8) take the tensor-core kernel
#endif
#ifndef PC_GRAM_R
#define PC_GRAM_R 12
#endif
#ifndef PC_GRAM_W
#define PC_GRAM_W 192  // 4 CTAs per SM fit in shared memory (256: 3); +4% at N = 65,536
#endif
#ifndef PC_COMP_W
#define PC_COMP_W 192
#endif
constexpr KernelCfg kBigGram{4, PC_GRAM_R, PC_GRAM_W};  // count kernel: 384-row warp tiles measured 6% faster than 256
constexpr KernelCfg kBigComp{4, 4, PC_COMP_W};          // compensated sum kernel (non-f32 input): 6 row registers per row
#ifndef PC_COMP_SORTED_R
#define PC_COMP_SORTED_R 6
#endif
#ifndef PC_COMP_SORTED_W
#define PC_COMP_SORTED_W 192
#endif
constexpr KernelCfg kBigCompSorted{4, PC_COMP_SORTED_R, PC_COMP_SORTED_W};  // float64 points, sorted
constexpr KernelCfg kBigCompSortedTc{4, 8, 256};  // ... beside the tensor-core kernel (its tile and chunk)
constexpr KernelCfg kSmall{4, 2, 64};  // warp tile 64 rows, for n < kSmallN
constexpr int kSmallN = 16384;


size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

long long max_slots(long long n) { return 148LL * 64 + n / (32 * kSmall.r * kSmall.warps) + 64; }

// ---- spatial (Morton) sort for the whole-range fp32 sum: permuting the points leaves
// the all-pairs total unchanged and makes row tiles and column chunks compact boxes,
// which the SORTED kernel uses for its tile-local Gram form (pairs_kernel.cuh).
inline size_t kSortTempBytes(size_t n) { return ((size_t)16 << 20) + 4 * n; }
constexpr long long kSortedMinN = 1 << 15;

__device__ __forceinline__ unsigned spread10(unsigned v) {  // 10 bits -> every third bit
    v &= 1023u;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
template <typename T>  // float (sums and counts) or double (pruned counts of float64 points)
__global__ void morton_kernel(const T* __restrict__ xyz, long long n, const PrepStats* __restrict__ st,
                              unsigned* __restrict__ keys, unsigned* __restrict__ idx) {
    T lo[3], sc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double mn = dec_f64(st->mn[k]), mx = dec_f64(st->mx[k]);
        lo[k] = (T)mn;
        sc[k] = mx > mn ? (T)(1023.0 / (mx - mn)) : (T)0;
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned c[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float v = (float)((xyz[3 * i + k] - lo[k]) * sc[k]);
            c[k] = (unsigned)fminf(fmaxf(v, 0.f), 1023.f);
        }
        keys[i] = spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2);
        idx[i] = (unsigned)i;
    }
}
template <typename T>
__global__ void gather_sorted_kernel(const T* __restrict__ xyz, const unsigned* __restrict__ idx, long long n,
                                     T* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long s = idx[i];
        out[3 * i] = xyz[3 * s];
        out[3 * i + 1] = xyz[3 * s + 1];
        out[3 * i + 2] = xyz[3 * s + 2];
    }
}
// one thread per 32-point block of sorted float64 points: the box of their centred fp32 high
// parts fl32(p - c) (c the bounding-box centre), the coordinates the compensated sum kernel
// holds in its row registers and stages as column highs
__global__ void blk_box_centred_kernel(const double* __restrict__ xyz, long long n, int nblk,
                                       const PrepStats* __restrict__ st, float4* __restrict__ box) {
    double c[3];
    long long ci[3];
    bbox_centre(*st, PC_F64, c, ci);
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nblk; b += (long long)gridDim.x * blockDim.x) {
        float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
        const long long e = min(n, 32 * b + 32);
        for (long long i = 32 * b; i < e; ++i) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float h = (float)(xyz[3 * i + k] - c[k]);
                mn[k] = fminf(mn[k], h);
                mx[k] = fmaxf(mx[k], h);
            }
        }
        box[2 * b] = make_float4(mn[0], mn[1], mn[2], 0.f);
        box[2 * b + 1] = make_float4(mx[0], mx[1], mx[2], 0.f);
    }
}
// one thread per 1024-point block: the union of its 32 per-32-point boxes
__global__ void blk2_box_kernel(const float4* __restrict__ box, int nblk, int nblk2, float4* __restrict__ box2) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblk2; b += gridDim.x * blockDim.x) {
        float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.f), hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
        for (int q = 32 * b; q < min(nblk, 32 * b + 32); ++q) {
            const float4 l = box[2 * q], h = box[2 * q + 1];
            lo = make_float4(fminf(lo.x, l.x), fminf(lo.y, l.y), fminf(lo.z, l.z), 0.f);
            hi = make_float4(fmaxf(hi.x, h.x), fmaxf(hi.y, h.y), fmaxf(hi.z, h.z), 0.f);
        }
        box2[2 * b] = lo;
        box2[2 * b + 1] = hi;
    }
}
// one thread per 32-point block: (min x, y, z, 0), (max x, y, z, 0)
__device__ __forceinline__ float round_down_f(float v) { return v; }
__device__ __forceinline__ float round_up_f(float v) { return v; }
__device__ __forceinline__ float round_down_f(double v) { return __double2float_rd(v); }
__device__ __forceinline__ float round_up_f(double v) { return __double2float_ru(v); }
// float64 points: boxes rounded outward to fp32, so they still contain their points
template <typename T>
__global__ void blk_box_kernel(const T* __restrict__ xyz, long long n, int nblk, float4* __restrict__ box) {
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nblk; b += (long long)gridDim.x * blockDim.x) {
        float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
        const long long e = min(n, 32 * b + 32);
        for (long long i = 32 * b; i < e; ++i) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                mn[k] = fminf(mn[k], round_down_f(xyz[3 * i + k]));
                mx[k] = fmaxf(mx[k], round_up_f(xyz[3 * i + k]));
            }
        }
        box[2 * b] = make_float4(mn[0], mn[1], mn[2], 0.f);
        box[2 * b + 1] = make_float4(mx[0], mx[1], mx[2], 0.f);
    }
}

struct WsLayout {
    size_t pts, stats, prof, red, slots, claims, claims_tc, tc_bits, tc_bits_cap, tc_cbox, tc_a, tc_b, tc_cand, tc_cnt, srt, srt_temp, total;
};
WsLayout ws_layout(long long n) {
    WsLayout l;
    const size_t pair_bytes = align_up((size_t)(n / 2 + 1) * 3 * sizeof(float4), 256);  // up to 3 float4 per pair
    l.pts = 0;  // even pairs, then odd pairs
    l.stats = 2 * pair_bytes;
    l.prof = l.stats + 256;  // pc_pairs_profile of the last call
    l.red = l.prof + 256;    // kRedBlocks float64 partials of the claim sums
    l.slots = l.red + 2 * kRedBlocks * sizeof(double);  // FFMA claims, then tensor-core claims
    l.claims = align_up(l.slots + (size_t)max_slots(n) * sizeof(Slot), 256);
    l.claims_tc = align_up(l.claims + (size_t)kClaimsCap * sizeof(double), 256);
    l.tc_bits = align_up(l.claims_tc + (size_t)kClaimsCap * sizeof(double), 256);
    l.tc_bits_cap = tcs_bits_bytes(n < 0 ? 0 : n);  // the whole-range bitmap, up to kTcsBitsMax
    l.tc_cbox = align_up(l.tc_bits + l.tc_bits_cap, 256);  // per-256 chunk boxes, 32 B each
    l.tc_a = align_up(l.tc_cbox + (size_t)((n < 0 ? 0 : n) / 256 + 1) * 32, 1024);
    const TcGeom g = tc_geom(n < 0 ? 0 : n);  // tensor-core count kernel operands (64 B per staged point)
    l.tc_b = align_up(l.tc_a + (size_t)g.n_rows * 64, 1024);
    l.tc_cand = align_up(l.tc_b + (size_t)g.n_ext * 64, 256);
    l.tc_cnt = align_up(l.tc_cand + (size_t)tc_cand_cap(n) * sizeof(uint2), 256);
    // spatial sort for the whole-range fp32 sum: keys + indices (double-buffered), the
    // sorted points, per-32-point boxes, radix-sort scratch
    l.srt = align_up(l.tc_cnt + 4 * 1024, 256);
    const size_t nn = (size_t)(n < 0 ? 0 : n);
    l.srt_temp = align_up(l.srt + 4 * align_up(nn * 4, 256) + align_up(nn * 24, 256) +
                          align_up((nn / 32 + 1) * 32, 256) + align_up((nn / 1024 + 1) * 32, 256), 256);
    l.total = align_up(l.srt_temp + kSortTempBytes(nn), 256);
    return l;
}

long long row_pairs(long long n, long long lo, long long hi, int sched) {
    if (hi <= lo) return 0;
    if (sched == PC_STANDARD) return ((n - 1 - lo) + (n - 1 - (hi - 1))) * (hi - lo) / 2;
    if (n & 1) return (hi - lo) * ((n - 1) / 2);
    long long h = n / 2;
    long long first = std::max(0LL, std::min(hi, h) - lo);
    return first * h + (hi - lo - first) * (h - 1);
}

int g_num_sms[64] = {0};
int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!g_num_sms[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        g_num_sms[dev] = v > 0 ? v : 148;
    }
    return g_num_sms[dev];
}

template <int WARPS, int R, int W, bool DIRECT, bool FLAT, bool COMP, bool SORTED = false>
int launch_pairs(PairsArgs args, long long n_slots_cap, int* nslots_out, int* nclaims_out, cudaStream_t s) {
    auto kern = pairs_kernel<WARPS, R, W, DIRECT, FLAT, COMP, SORTED>;
    constexpr int smem = WARPS * pairs_smem_per_warp<R, W, COMP>();
    {
        static thread_local bool attr_set[64] = {false};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!attr_set[dev & 63]) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr_set[dev & 63] = true;
        }
    }
    int grid;
    *nclaims_out = 0;
    if (FLAT) {
        static thread_local int occ_cache[64] = {0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!occ_cache[dev & 63]) {
            int occ = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WARPS * 32, smem));
            occ_cache[dev & 63] = occ > 0 ? occ : 1;
        }
        const long long want = (long long)num_sms() * occ_cache[dev & 63];
        const long long chunks = (args.total + W - 1) / W;
        grid = (int)std::max(1LL, std::min(want, (chunks + WARPS - 1) / WARPS));
        // claim stages over the block-transposed (tile, column) space (pairs_kernel.cuh claim()):
        // uniform claims of S chunks (one block, S a power of two <= PC_CLAIM_MAX, larger only to
        // keep the claim count within kClaimsCap) for the bulk, then a guided tail -- P claims of
        // about (remaining / 2P) chunks, a power of two, halving down to single chunks
        const long long P = (long long)grid * WARPS;
        auto pow2_floor = [](long long v) { long long p2 = 1; while (p2 * 2 <= v) p2 *= 2; return p2; };
        long long S = pow2_floor(std::max(1LL, std::min((long long)PC_CLAIM_MAX, chunks / (8 * P))));
        while (S * (kClaimsCap / 2) < chunks) S *= 2;
        args.blk_cols = S * W;
        const long long nb = (args.L + args.blk_cols - 1) / args.blk_cols;  // blocks per window
        args.win_blks = nb;
        const long long vchunks = (long long)args.n_tiles * nb * S;         // incl. the windows' ragged ends
        long long rem = vchunks, c0 = 0, b0 = 0;
        int ns = 0;
        auto add_stage = [&](long long sz, long long k) {
            args.st_c0[ns] = c0;
            args.st_b0[ns] = b0;
            args.st_s[ns] = sz * W;
            c0 += k;
            b0 += k * sz * W;
            rem -= k * sz;
            ++ns;
        };
        const long long bulk = PC_GUIDED ? (vchunks - std::min(vchunks, 2 * P * S)) / S : vchunks / S;
        if (bulk > 0) add_stage(S, bulk);
        while (rem > 0) {
            if (ns == kMaxStages) return arg_fail("too many claim stages");
            const long long sz = pow2_floor(std::max(1LL, std::min(S, rem / (2 * P))));
            add_stage(sz, sz == 1 ? rem : std::min(P, rem / sz));
        }
        args.st_c0[ns] = c0;
        args.nstage = ns;
        if (c0 > kClaimsCap) return arg_fail("workspace too small for the claim partials");
        *nclaims_out = (int)c0;
        if (DIRECT) CK(cudaMemsetAsync(args.claim_sums, 0, (size_t)c0 * sizeof(double), s));
    } else {
        grid = (args.n_tiles + WARPS - 1) / WARPS;
    }
    if (grid > n_slots_cap) return arg_fail("workspace too small for the CTA slots");
    if (FLAT) CK(cudaMemsetAsync(args.work_ctr, 0, sizeof(unsigned long long), s));
    EvPair* ev = nullptr;
    if (g_timing && g_ev_used < 4096) {
        if (g_ev_used == g_ev_made) {
            CK(cudaEventCreate(&g_ev[g_ev_made].a));
            CK(cudaEventCreate(&g_ev[g_ev_made].b));
            ++g_ev_made;
        }
        ev = &g_ev[g_ev_used++];
        ev->kind = 0;
        CK(cudaEventRecord(ev->a, s));
    }
    kern<<<grid, WARPS * 32, smem, s>>>(args);
    CK_LAUNCH("pairs_kernel");
    if (ev) CK(cudaEventRecord(ev->b, s));
    *nslots_out = grid;
    return PC_OK;
}

// Row tiles of one call: all tiles of [lo, hi) when tstride = 1, else the blocks of kTcsOrgG tiles
// toff, toff + tstride, ... -- pc_pairs_part_async deals a range's tile blocks round-robin over nparts
// calls; the call's i-th tile is absolute tile tile_abs(i) (pairs_kernel.cuh).
struct TileSel {
    int tstride, toff;
};
inline int tiles_of(long long lo, long long hi, int T, TileSel ts) {
    const long long all = (hi - lo + T - 1) / T;
    if (ts.tstride == 1) return (int)all;
    const long long blocks = (all + kTcsOrgG - 1) / kTcsOrgG;  // the last one may be partial
    if (blocks <= ts.toff) return 0;
    const long long nb = (blocks - ts.toff + ts.tstride - 1) / ts.tstride, last = ts.toff + (nb - 1) * ts.tstride;
    return (int)((nb - 1) * kTcsOrgG + std::min<long long>(kTcsOrgG, all - last * kTcsOrgG));
}
// pairs owned by the selected tiles' rows
long long tile_sel_pairs(long long n, long long lo, long long hi, int T, TileSel ts, int sched) {
    if (ts.tstride == 1) return row_pairs(n, lo, hi, sched);
    long long p = 0;
    const int nt = tiles_of(lo, hi, T, ts);
    for (int i = 0; i < nt; ++i) {
        const long long t = tile_abs(i, ts.tstride, ts.toff);
        p += row_pairs(n, lo + t * T, std::min(hi, lo + (t + 1) * T), sched);
    }
    return p;
}

template <int WARPS, int R, int W, bool DIRECT, bool COMP = false, bool SORTED = false>
int dispatch_cfg(PairsArgs args, bool flat, TileSel ts, long long cap, int* nslots, int* nclaims, int* tile_rows,
                 long long* pairs_per_chunk, cudaStream_t s) {
    constexpr int T = 32 * R;
    args.tstride = ts.tstride;
    args.toff = ts.toff;
    args.tile_rows = T;
    args.n_tiles = tiles_of(args.lo, args.hi, T, ts);
    *tile_rows = T;
    *pairs_per_chunk = (long long)T * W;
    *nclaims = 0;
    if (args.n_tiles == 0) {  // a tile part with no tiles (more parts than tiles)
        *nslots = 0;
        return PC_OK;
    }
    if (flat) {
        args.L = (long long)(T - 1) + (args.n >> 1);
        args.total = (long long)args.n_tiles * args.L;
        return launch_pairs<WARPS, R, W, DIRECT, true, COMP, SORTED>(args, cap, nslots, nclaims, s);
    }
    return launch_pairs<WARPS, R, W, DIRECT, false, COMP>(args, cap, nslots, nclaims, s);
}

// The tensor-core Gram chunks of a sorted fp32 sum (pairs_tcsum.cuh): launched after the
// FFMA sorted kernel (which left these chunks alone) over the same tiles.  PAIRCOUNT_TCSUM=0
// in the environment keeps every chunk on the FFMA kernel (A/B runs).
#ifndef PC_TCSUM
#define PC_TCSUM 1
#endif
// PAIRCOUNT_TCS_BITMAP=0: classify chunks in-loop in both kernels (the path beyond the bitmap's size
// cap), for tests at sizes where the bitmap would fit
bool tcs_bitmap_enabled() {
    static const bool on = [] {
        const char* e = getenv("PAIRCOUNT_TCS_BITMAP");
        return !(e && e[0] == '0');
    }();
    return on;
}
// PAIRCOUNT_TCS2=1: the SM-pair kernel (pairs_tcs2.cuh) for fp32 points -- correct, but measured
// 110.6 ms against 66.2 for pairs_tcs_kernel at 2^20, so off by default
bool tcs2_enabled() {
    static const bool on = [] {
        const char* e = getenv("PAIRCOUNT_TCS2");
        return e && e[0] == '1';
    }();
    return on;
}
bool tcs_enabled() {
    static const bool on = [] {
        const char* e = getenv("PAIRCOUNT_TCSUM");
        return PC_TCSUM && !(e && e[0] == '0');
    }();
    return on && 32 * kBig.r == kTcsT && kBig.w == kTcsW;
}
// The chunk bitmap of one range's tiles into `bits` (capacity cap_bytes); *cpw_pad stays 0 when it does
// not fit (the kernels then classify in-loop).
int classify_tcs(const PairsArgs& p, TileSel ts, unsigned* bits, size_t cap_bytes, long long* cpw_pad,
                 cudaStream_t s, float4* cbox_area = nullptr) {
    TcsArgs a{};
    a.blk_box = p.blk_box;
    a.n = p.n;
    a.lo = p.lo;
    a.hi = p.hi;
    a.tstride = ts.tstride;
    a.toff = ts.toff;
    a.n_tiles = tiles_of(p.lo, p.hi, kTcsT, ts);
    a.L = (long long)(kTcsT - 1) + (p.n >> 1);
    a.cpw = tcs_cpw(p.n);
    a.cpw_pad = tcs_cpw_pad(p.n);
    a.bits = bits;
    *cpw_pad = 0;
    if (a.n_tiles == 0 || !bits || (size_t)a.n_tiles * (size_t)a.cpw_pad / 8 > cap_bytes) return PC_OK;
    if (cbox_area && p.n % 256 == 0 && p.lo % 256 == 0) {  // every chunk starts at 256 m + 1
        const int nchunk = p.n / 256;
        tcs_chunk_box_kernel<<<(nchunk + 255) / 256, 256, 0, s>>>(p.blk_box, p.n / 32, nchunk, cbox_area);
        CK_LAUNCH("tcs_chunk_box_kernel");
        a.cbox = cbox_area;
    }
    tcs_classify_kernel<<<(int)(((long long)a.n_tiles * (a.cpw_pad / 32) + 7) / 8), 256, 0, s>>>(a);
    CK_LAUNCH("tcs_classify_kernel");
    *cpw_pad = a.cpw_pad;
    return PC_OK;
}

int launch_tcs(const PairsArgs& p, TileSel ts, double* claims_tc, Slot* slots, long long cap, int* nslots,
               int* nparts, cudaStream_t s, unsigned* bits = nullptr, long long cpw_pad = 0) {
    TcsArgs a{};
    a.xyz = p.xyz;
    a.blk_box = p.blk_box;
    a.st = p.st;
    a.slots = slots;
    a.claim_sums = claims_tc;
    a.work_ctr = p.work_ctr;
    a.dtype = p.dtype;
    a.n = p.n;
    a.lo = p.lo;
    a.hi = p.hi;
    a.tstride = ts.tstride;
    a.toff = ts.toff;
    a.n_tiles = tiles_of(p.lo, p.hi, kTcsT, ts);
    a.L = (long long)(kTcsT - 1) + (p.n >> 1);
    a.cpw = (a.L + kTcsW - 1) / kTcsW;
    a.bits = bits;
    a.cpw_pad = cpw_pad;
    // fp32 points with the bitmap and PAIRCOUNT_TCS2=1: the SM-pair kernel (pairs_tcs2.cuh)
    const bool pair = tcs2_enabled() && p.dtype == PC_F32 && bits != nullptr && num_sms() >= 2;
    // work units: the diagonals of groups of G consecutive tiles (one column operand for up to G
    // items; tile parts deal whole groups); the SM-pair kernel: one item per unit
    a.G = pair ? 1 : kTcsOrgG;
    a.upg = a.cpw + a.G - 1;
    a.items = (long long)((a.n_tiles + a.G - 1) / a.G) * a.upg;
    // units per claim: a power of two keeping the float64 partials (kTcsParts per claim) within
    // kClaimsCap, and as large as ~128 claims per CTA allows (up to 128 units): a claim's units are
    // consecutive diagonals of one group, so small claims rebuild the row operands often (tile parts)
    const long long parts = pair ? kTc2Parts : kTcsParts;
    const int grid = pair ? num_sms() & ~1 : num_sms();
    long long S = 1;
    while (S * (kClaimsCap / parts) < a.items) S *= 2;
#ifndef PC_TCS_SMAX
#define PC_TCS_SMAX 128  // (2^20: 32 / 64 / 128 / 256 units -> 58.1 / 57.6 / 57.5 / 57.5 ms)
#endif
#ifndef PC_TCS_CPC
#define PC_TCS_CPC 32  // claims per CTA the claim size keeps at least (8 tile parts at 2^20: 128 -> 8.67, 32 -> 8.56 ms)
#endif
    while (S < PC_TCS_SMAX && S * 2 * (long long)grid * PC_TCS_CPC <= a.items) S *= 2;
    a.S = S;
    a.nclaims = (a.items + S - 1) / S;
    *nslots = 0;
    *nparts = 0;
    if (a.n_tiles == 0) return PC_OK;
    if (grid > cap) return arg_fail("workspace too small for the CTA slots");
    static thread_local bool attr_set[64] = {false};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!attr_set[dev & 63]) {
        CK(cudaFuncSetAttribute(pairs_tcs_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcsSmem));
        CK(cudaFuncSetAttribute(pairs_tcs_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcsSmem));
        CK(cudaFuncSetAttribute(pairs_tcs2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTc2Smem));
        attr_set[dev & 63] = true;
    }
    CK(cudaMemsetAsync(a.work_ctr, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(claims_tc, 0, (size_t)a.nclaims * parts * sizeof(double), s));
    EvPair* ev = nullptr;
    if (g_timing && g_ev_used < 4096) {
        if (g_ev_used == g_ev_made) {
            CK(cudaEventCreate(&g_ev[g_ev_made].a));
            CK(cudaEventCreate(&g_ev[g_ev_made].b));
            ++g_ev_made;
        }
        ev = &g_ev[g_ev_used++];
        ev->kind = 1;
        CK(cudaEventRecord(ev->a, s));
    }
    if (pair) pairs_tcs2_kernel<<<grid, kTc2Warps * 32, kTc2Smem, s>>>(a);
    else if (p.dtype == PC_F64) pairs_tcs_kernel<double><<<grid, kTcsWarps * 32, kTcsSmem, s>>>(a);
    else pairs_tcs_kernel<float><<<grid, kTcsWarps * 32, kTcsSmem, s>>>(a);
    CK_LAUNCH("pairs_tcs_kernel");
    if (ev) CK(cudaEventRecord(ev->b, s));
    *nslots = grid;
    *nparts = (int)(a.nclaims * parts);
    return PC_OK;
}

// Balanced counts on the tensor cores (pairs_tc.cuh): operands staged once per call,
// then per row range the persistent kernel (one CTA per SM), the exact pass over its
// queued candidates and the fixed-order slot sum.
int run_pairs_tc(const PairsArgs& p, char* ws, const WsLayout& lay, long long n, long long cap, int nranges,
                 const long long* bounds, pc_pairs_result* dres, pc_pairs_profile* prof, cudaStream_t s) {
    const TcGeom g = tc_geom(n);
    const long long npts = std::max(g.n_rows, g.n_ext);
    const int pblocks = (int)std::min<long long>((npts + 255) / 256, (long long)num_sms() * 8);
    prep_tc_kernel<<<pblocks, 256, 0, s>>>(p.xyz, p.dtype, n, p.st, g.n_rows, g.n_ext, ws + lay.tc_a, ws + lay.tc_b);
    CK_LAUNCH("prep_tc_kernel");
    static thread_local bool attr_set[64] = {false};
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!attr_set[dev & 63]) {
        CK(cudaFuncSetAttribute(pairs_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
        attr_set[dev & 63] = true;
    }
    TcArgs a{};
    a.aop = (const float4*)(ws + lay.tc_a);
    a.bop = (const float4*)(ws + lay.tc_b);
    a.pts_even = p.pts_even;
    a.pts_odd = p.pts_odd;
    a.xyz = p.xyz;
    a.st = p.st;
    a.slots = p.slots;
    a.work_ctr = p.work_ctr;
    a.dtype = p.dtype;
    a.pred = p.pred;
    a.n = (int)n;
    a.thr = p.thr;
    a.chunks = g.chunks;
    a.cand = (uint2*)(ws + lay.tc_cand);
    a.cand_counts = (unsigned*)(ws + lay.tc_cnt);
    for (int k = 0; k < nranges; ++k) {
        const long long lo = bounds[k], hi = bounds[k + 1];
        int nslots = 0;
        if (hi > lo) {
            a.lo = (int)lo;
            a.hi = (int)hi;
            a.lo8 = (int)(lo & ~7LL);
            a.n_tiles = (hi - a.lo8 + kTcM - 1) / kTcM;
            a.items = a.n_tiles * g.chunks;
            const int grid = (int)std::min<long long>(std::min(num_sms(), 1024), a.items);
            a.cand_per_cta = tc_cand_cap(n) / grid;
            a.group = (int)std::max(1LL, std::min(16LL, a.items / ((long long)grid * 16)));
            if (2 * grid > cap) return arg_fail("workspace too small for the CTA slots");
            CK(cudaMemsetAsync(p.work_ctr, 0, sizeof(unsigned long long), s));
            EvPair* ev = nullptr;
            if (g_timing && g_ev_used < 4096) {
                if (g_ev_used == g_ev_made) {
                    CK(cudaEventCreate(&g_ev[g_ev_made].a));
                    CK(cudaEventCreate(&g_ev[g_ev_made].b));
                    ++g_ev_made;
                }
                ev = &g_ev[g_ev_used++];
                ev->kind = 0;
                CK(cudaEventRecord(ev->a, s));
            }
            pairs_tc_kernel<<<grid, kTcWarps * 32, kTcSmem, s>>>(a);
            CK_LAUNCH("pairs_tc_kernel");
            tc_exact_kernel<<<grid, 256, 0, s>>>(a, p.slots + grid);
            CK_LAUNCH("tc_exact_kernel");
            if (ev) CK(cudaEventRecord(ev->b, s));
            nslots = 2 * grid;
        }
        finalize_kernel<<<1, 256, 0, s>>>(p.slots, nslots, nullptr, 0, 0, 0, p.st, p.dtype, row_pairs(n, lo, hi, PC_BALANCED),
                                          0, dres + k, prof, kKernTc, (long long)kTcM * kTcN);
        CK_LAUNCH("finalize_kernel");
    }
    return PC_OK;
}

// Exact coincidence counts by 30-bit key compare (pairs_key.cuh; PC_TILE_KEY).
int run_pairs_key(const PairsArgs& p, char* ws, const WsLayout& lay, long long n, long long cap, int nranges,
                  const long long* bounds, pc_pairs_result* dres, pc_pairs_profile* prof, cudaStream_t s) {
    constexpr int T = 32 * kKeyR;
    unsigned* ext = (unsigned*)(ws + lay.tc_b);
    const long long e = 2 * n + 2 * T;
    if ((size_t)e * 4 > lay.tc_cand - lay.tc_b) return arg_fail("workspace too small for the key array");
    const int pblocks = (int)std::min<long long>((e + 255) / 256, (long long)num_sms() * 8);
    if (n > 0) {
        prep_key_kernel<<<pblocks, 256, 0, s>>>(p.xyz, p.dtype, n, e, const_cast<PrepStats*>(p.st), ext);
        CK_LAUNCH("prep_key_kernel");
    }
    KeyArgs a{};
    a.ext = ext;
    a.st = p.st;
    a.slots = p.slots;
    a.work_ctr = p.work_ctr;
    a.n = (int)n;
    a.L = T - 1 + (int)(n >> 1);
    a.cpt = (a.L + kKeyW - 1) / kKeyW;
    for (int k = 0; k < nranges; ++k) {
        const long long lo = bounds[k], hi = bounds[k + 1];
        int nslots = 0;
        if (hi > lo && n >= 2) {
            a.lo = (int)lo;
            a.hi = (int)hi;
            a.n_tiles = (int)((hi - lo + T - 1) / T);
            a.units = (long long)a.n_tiles * a.cpt;
            const long long want = (long long)num_sms() * 4;
            const int grid = (int)std::max(1LL, std::min(want, (a.units + kKeyWarps - 1) / kKeyWarps));
            a.group = (int)std::max(1LL, std::min(16LL, a.units / ((long long)grid * kKeyWarps * 8)));
            if (grid > cap) return arg_fail("workspace too small for the CTA slots");
            CK(cudaMemsetAsync(p.work_ctr, 0, sizeof(unsigned long long), s));
            EvPair* ev = nullptr;
            if (g_timing && g_ev_used < 4096) {
                if (g_ev_used == g_ev_made) {
                    CK(cudaEventCreate(&g_ev[g_ev_made].a));
                    CK(cudaEventCreate(&g_ev[g_ev_made].b));
                    ++g_ev_made;
                }
                ev = &g_ev[g_ev_used++];
                ev->kind = 0;
                CK(cudaEventRecord(ev->a, s));
            }
            pairs_key_kernel<<<grid, kKeyWarps * 32, 0, s>>>(a);
            CK_LAUNCH("pairs_key_kernel");
            if (ev) CK(cudaEventRecord(ev->b, s));
            nslots = grid;
        }
        finalize_kernel<<<1, 256, 0, s>>>(p.slots, nslots, nullptr, 0, 0, 0, p.st, p.dtype,
                                          row_pairs(n, lo, hi, PC_BALANCED), 0, dres + k, prof, kKernKey,
                                          (long long)T * kKeyW);
        CK_LAUNCH("finalize_kernel");
    }
    return PC_OK;
}

int run_pairs(const void* xyz, int dtype, long long n, int interaction, int schedule, int tiling,
              int nranges, const long long* bounds, void* workspace, size_t wsb,
              pc_pairs_result* dres, cudaStream_t s, TileSel ts = TileSel{1, 0}) {
    g_launches = 0;
    if (ts.tstride < 1 || ts.toff < 0 || ts.toff >= ts.tstride) return arg_fail("bad tile part (0 <= part < nparts)");
    if (dtype < PC_F32 || dtype > PC_I64) return arg_fail("unknown dtype");
    if (schedule != PC_STANDARD && schedule != PC_BALANCED) return arg_fail("unknown schedule");
    if (interaction < PC_COLLISION || interaction > PC_MANHATTAN1) return arg_fail("unknown interaction");
    if ((interaction == PC_COINCIDE || interaction == PC_MANHATTAN1) && dtype < PC_I32)
        return arg_fail("integer interactions need integer coordinates");
    if (n < 0 || n >= (1LL << 30)) return arg_fail("n out of range (0 <= n < 2^30)");
    if (nranges < 1 || !bounds) return arg_fail("need at least one row range");
    for (int k = 0; k < nranges; ++k)
        if (bounds[k] < 0 || bounds[k] > bounds[k + 1] || bounds[k + 1] > n) return arg_fail("bad row range bounds");
    const bool tc_ok = interaction != PC_COLLISION_INVSQ && schedule == PC_BALANCED && n >= 2;
    if (tiling == PC_TILE_TC && !tc_ok)
        return arg_fail("PC_TILE_TC needs a count interaction and the balanced schedule");
    long long rows = 0;  // AUTO: ranges of a few tiles stay on the FFMA kernel (the staging is per call)
    for (int k = 0; k < nranges; ++k) rows += std::max(0LL, (long long)(bounds[k + 1] - bounds[k]));
    if (tiling == PC_TILE_TC && ts.tstride != 1) return arg_fail("PC_TILE_TC does not take tile parts");
    const bool whole = nranges == 1 && bounds[0] == 0 && bounds[1] == n;
    const bool prune_auto = PC_SORTED_COUNT && tiling == PC_TILE_AUTO && whole && interaction == PC_COLLISION &&
                            (dtype == PC_F32 || dtype == PC_F64) && schedule == PC_BALANCED && n >= kSortedMinN;
    const bool use_tc = tc_ok && ts.tstride == 1 && !prune_auto &&
                        (tiling == PC_TILE_TC || (tiling == PC_TILE_AUTO && PC_TC_AUTO && n >= kTcMinN &&
                                                  n < kTcMaxN && rows * 8 >= n));
    const bool auto_tiling = tiling == PC_TILE_AUTO, sorted_req = tiling == PC_TILE_SORTED;
    const bool use_key = tiling == PC_TILE_KEY;
    const bool use_row = tiling == PC_TILE_THREAD_ROW;
    if (use_row && (dtype != PC_F32 || (interaction != PC_COLLISION && interaction != PC_COLLISION_INVSQ) ||
                    ts.tstride != 1))
        return arg_fail("PC_TILE_THREAD_ROW needs fp32 spheres (collision count or inverse-square sum), no tile parts");
    if (use_key && (interaction != PC_COINCIDE || schedule != PC_BALANCED || ts.tstride != 1))
        return arg_fail("PC_TILE_KEY needs the coincidence count, the balanced schedule and no tile parts");
    if (sorted_req && ((interaction == PC_COLLISION_INVSQ && dtype != PC_F32 && dtype != PC_F64) ||
                       (interaction == PC_COLLISION && dtype != PC_F32 && dtype != PC_F64) ||
                       (interaction != PC_COLLISION_INVSQ && interaction != PC_COLLISION) || schedule != PC_BALANCED))
        return arg_fail("PC_TILE_SORTED needs spheres -- the inverse-square sum or the contact count on fp32 / fp64 "
                        "points -- and the balanced schedule");
    if (tiling == PC_TILE_AUTO || tiling == PC_TILE_TC || tiling == PC_TILE_SORTED || use_key || use_row)
        tiling = schedule == PC_BALANCED ? PC_TILE_FLAT : PC_TILE_PER_ROW_TILE;
    if (tiling == PC_TILE_FLAT && schedule != PC_BALANCED)
        return arg_fail("PC_TILE_FLAT needs the balanced schedule (equal windows per row tile)");
    if (tiling != PC_TILE_FLAT && tiling != PC_TILE_PER_ROW_TILE) return arg_fail("unknown tiling");
    const WsLayout lay = ws_layout(n);
    if (!workspace || wsb < lay.total) return arg_fail("workspace too small (see pc_pairs_workspace_bytes)");
    char* ws = (char*)workspace;
    float4* pts_even = (float4*)(ws + lay.pts);
    float4* pts_odd = (float4*)(ws + lay.pts + lay.stats / 2);
    PrepStats* st = (PrepStats*)(ws + lay.stats);
    pc_pairs_profile* prof = (pc_pairs_profile*)(ws + lay.prof);
    Slot* slots = (Slot*)(ws + lay.slots);
    double* claims = (double*)(ws + lay.claims);
    const bool direct = interaction == PC_COLLISION_INVSQ;
    const bool comp = direct && dtype != PC_F32;  // f32 coordinates are exact as staged

    // bbox init: minima to the largest ordered code, maxima to the smallest
    CK(cudaMemsetAsync(st, 0xff, offsetof(PrepStats, mx), s));
    CK(cudaMemsetAsync((char*)st + offsetof(PrepStats, mx), 0, sizeof(PrepStats) - offsetof(PrepStats, mx), s));
    CK(cudaMemsetAsync(prof, 0, sizeof(pc_pairs_profile), s));
    // whole-range fp32 sums over the balanced schedule run on spatially sorted points
    // (PC_TILE_AUTO on the whole range, or PC_TILE_SORTED for row ranges of the sorted
    // order; PC_TILE_FLAT keeps the input order, the plain kernel)
    const bool whole_range = nranges == 1 && bounds[0] == 0 && bounds[1] == n;
    const bool sorted = PC_SORTED_SUM && direct && (!comp || dtype == PC_F64) && schedule == PC_BALANCED &&
                        n >= kSortedMinN && ((auto_tiling && whole_range) || sorted_req);
    // whole-range fp32 contact counts: the same sort, then the Gram count with box pruning (pairs_kernel.cuh)
    const bool sorted_count = PC_SORTED_COUNT && interaction == PC_COLLISION && (dtype == PC_F32 || dtype == PC_F64) &&
                              schedule == PC_BALANCED && n >= kSortedMinN && ts.tstride >= 1 &&
                              ((auto_tiling && whole_range) || sorted_req);
    const float4* blk_box = nullptr;
    const float4* blk2_box = nullptr;
    const int nblk = (int)((n + 31) / 32);
    if (n > 0) {
        const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 8);
        prep_bbox_kernel<<<blocks, 256, 0, s>>>(xyz, dtype, n, st);
        CK_LAUNCH("prep_bbox_kernel");
        if (sorted || sorted_count) {
            const size_t kb = align_up((size_t)n * 4, 256);
            unsigned* k0 = (unsigned*)(ws + lay.srt);
            unsigned* k1 = (unsigned*)(ws + lay.srt + kb);
            unsigned* v0 = (unsigned*)(ws + lay.srt + 2 * kb);
            unsigned* v1 = (unsigned*)(ws + lay.srt + 3 * kb);
            void* xs = ws + lay.srt + 4 * kb;  // sorted copy of the points (12 or 24 B each)
            float4* box = (float4*)(ws + lay.srt + 4 * kb + align_up((size_t)n * 24, 256));
            const bool f64 = dtype == PC_F64;
            if (f64) morton_kernel<double><<<blocks, 256, 0, s>>>((const double*)xyz, n, st, k0, v0);
            else morton_kernel<float><<<blocks, 256, 0, s>>>((const float*)xyz, n, st, k0, v0);
            CK_LAUNCH("morton_kernel");
            cub::DoubleBuffer<unsigned> dk(k0, k1), dv(v0, v1);
            size_t tb = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)n, 0, 30, s));
            if (tb > kSortTempBytes((size_t)n)) return arg_fail("radix-sort scratch exceeds its reservation");
            CK(cub::DeviceRadixSort::SortPairs(ws + lay.srt_temp, tb, dk, dv, (int)n, 0, 30, s));
            // (the radix sort's kernels are CUB's, not counted in g_launches)
            if (f64) gather_sorted_kernel<double><<<blocks, 256, 0, s>>>((const double*)xyz, dv.Current(), n, (double*)xs);
            else gather_sorted_kernel<float><<<blocks, 256, 0, s>>>((const float*)xyz, dv.Current(), n, (float*)xs);
            CK_LAUNCH("gather_sorted_kernel");
            if (f64 && comp)  // the compensated sum works on centred high parts
                blk_box_centred_kernel<<<(nblk + 255) / 256, 256, 0, s>>>((const double*)xs, n, nblk, st, box);
            else if (f64) blk_box_kernel<double><<<(nblk + 255) / 256, 256, 0, s>>>((const double*)xs, n, nblk, box);
            else blk_box_kernel<float><<<(nblk + 255) / 256, 256, 0, s>>>((const float*)xs, n, nblk, box);
            CK_LAUNCH("blk_box_kernel");
            if (sorted_count) {
                // the per-1024 boxes follow the (n/32+1)*32 B of per-32 boxes
                float4* box2 = (float4*)(ws + lay.srt + 4 * kb + align_up((size_t)n * 24, 256) +
                                         align_up((size_t)(n / 32 + 1) * 32, 256));
                const int nblk2 = (int)((n + 1023) / 1024);
                blk2_box_kernel<<<(nblk2 + 255) / 256, 256, 0, s>>>(box, nblk, nblk2, box2);
                CK_LAUNCH("blk2_box_kernel");
                blk2_box = box2;
            }
            xyz = xs;  // from here on the call works on the sorted points
            blk_box = box;
        }
        if (comp) prep_stage_kernel<true, true><<<blocks, 256, 0, s>>>(xyz, dtype, n, st, pts_even, pts_odd);
        else if (direct) prep_stage_kernel<true, false><<<blocks, 256, 0, s>>>(xyz, dtype, n, st, pts_even, pts_odd);
        else prep_stage_kernel<false, false><<<blocks, 256, 0, s>>>(xyz, dtype, n, st, pts_even, pts_odd);
        CK_LAUNCH("prep_stage_kernel");
    }
    PairsArgs args{};
    args.pts_even = pts_even;
    args.pts_odd = pts_odd;
    args.xyz = xyz;
    args.st = st;
    args.blk_box = blk_box;
    args.blk2_box = blk2_box;
    args.nblk = nblk;
    args.slots = slots;
    args.claim_sums = claims;
    args.work_ctr = &st->work_ctr;
    args.dtype = dtype;
    args.pred = interaction == PC_COINCIDE ? kPredCoincide : interaction == PC_MANHATTAN1 ? kPredManhattan1 : kPredSphere;
    args.thr = interaction == PC_COINCIDE ? 0.5f : interaction == PC_MANHATTAN1 ? 1.5f : 1.0f;
    args.sched = schedule;
    args.n = (int)n;
    const long long cap = max_slots(n);
    if (use_tc) return run_pairs_tc(args, ws, lay, n, cap, nranges, bounds, dres, prof, s);
    if (use_key) return run_pairs_key(args, ws, lay, n, cap, nranges, bounds, dres, prof, s);
    if (use_row) {  // the paper's thread-per-row schemes (pairs_row.cuh), a baseline
        for (int k = 0; k < nranges; ++k) {
            const long long lo = bounds[k], hi = bounds[k + 1];
            int nslots = 0;
            if (hi > lo && n >= 2) {
                args.lo = (int)lo;
                args.hi = (int)hi;
                const int grid = (int)((hi - lo + kRowThreads - 1) / kRowThreads);
                if (grid + num_sms() * 4 > cap) return arg_fail("workspace too small for the CTA slots");
                EvPair* ev = nullptr;
                if (g_timing && g_ev_used < 4096) {
                    if (g_ev_used == g_ev_made) {
                        CK(cudaEventCreate(&g_ev[g_ev_made].a));
                        CK(cudaEventCreate(&g_ev[g_ev_made].b));
                        ++g_ev_made;
                    }
                    ev = &g_ev[g_ev_used++];
                    ev->kind = 0;
                    CK(cudaEventRecord(ev->a, s));
                }
                pairs_row_kernel<<<grid, kRowThreads, 0, s>>>(args, direct ? 1 : 0);
                CK_LAUNCH("pairs_row_kernel");
                if (ev) CK(cudaEventRecord(ev->b, s));
                nslots = grid;
                if (direct) {
                    args.tstride = 1;
                    args.toff = 0;
                    args.tile_rows = kRowThreads;
                    const int g2 = (int)std::min<long long>((hi - lo + 255) / 256, (long long)num_sms() * 4);
                    pairs_f64_kernel<<<g2, 256, 0, s>>>(args, 0, slots + nslots);
                    CK_LAUNCH("pairs_f64_kernel");
                    nslots += g2;
                }
            }
            finalize_kernel<<<1, 256, 0, s>>>(slots, nslots, nullptr, 0, 0, 0, st, dtype,
                                              row_pairs(n, lo, hi, schedule), direct ? 1 : 0, dres + k, prof,
                                              kKernRow, 0);
            CK_LAUNCH("finalize_kernel");
        }
        return PC_OK;
    }
    // sorted fp32 sums: the Gram chunks the tensor cores can take go to pairs_tcs_kernel (ranges
    // starting on a 32-point block, so both kernels see the same per-32 boxes of every tile)
    const bool use_tcs_call = sorted && (!comp || dtype == PC_F64) && n >= kSmallN && tcs_enabled();
    double* claims_tc = (double*)(ws + lay.claims_tc);
    for (int k = 0; k < nranges; ++k) {
        const long long lo = bounds[k], hi = bounds[k + 1];
        const bool use_tcs = use_tcs_call && lo % 32 == 0;
        args.tc_split = use_tcs ? 1 : 0;
        args.tc_bits = nullptr;
        args.tc_cpw_pad = 0;
        const int kern_id = !direct ? (sorted_count ? kKernSortedCount : kKernGram)
                                    : comp ? (sorted ? (use_tcs ? kKernCompSortedTc : kKernCompSorted) : kKernComp)
                                           : sorted ? (use_tcs ? kKernSortedTc : kKernSorted) : kKernDirect;
        int nslots = 0, nclaims = 0, trows = 1, ntcparts = 0;
        long long ppc = 0;
        if (hi > lo && n >= 2) {
            args.lo = (int)lo;
            args.hi = (int)hi;
            const bool flat = tiling == PC_TILE_FLAT;
            int rc;
            if (use_tcs) {  // the chunk bitmap both kernels follow (when it fits the workspace)
                long long cpw_pad = 0;
                unsigned* bits = (unsigned*)(ws + lay.tc_bits);
                rc = lay.tc_bits_cap && tcs_bitmap_enabled()
                         ? classify_tcs(args, ts, bits, lay.tc_bits_cap, &cpw_pad, s, (float4*)(ws + lay.tc_cbox))
                         : PC_OK;
                if (rc) return rc;
                if (cpw_pad) {
                    args.tc_bits = bits;
                    args.tc_cpw_pad = cpw_pad;
                }
            }
#define PC_DISPATCH(CFG, ...) dispatch_cfg<CFG.warps, CFG.r, CFG.w, __VA_ARGS__>(args, flat, ts, cap, &nslots, &nclaims, \
                                                                                &trows, &ppc, s)
            if (n < kSmallN)
                rc = comp     ? PC_DISPATCH(kSmall, true, true)
                     : direct ? PC_DISPATCH(kSmall, true)
                              : PC_DISPATCH(kSmall, false);
            else
                rc = comp     ? (sorted ? (use_tcs ? PC_DISPATCH(kBigCompSortedTc, true, true, true)
                                          : PC_DISPATCH(kBigCompSorted, true, true, true))
                                : PC_DISPATCH(kBigComp, true, true))
                     : sorted ? PC_DISPATCH(kBig, true, false, true)
                     : direct ? PC_DISPATCH(kBig, true)
                     : sorted_count ? PC_DISPATCH(kBigGram, false, false, true)
                              : PC_DISPATCH(kBigGram, false);
#undef PC_DISPATCH
            if (rc) return rc;
            if (direct) {  // the float64 path (does nothing unless f64_takes: non-finite, huge, wide span)
                args.tstride = ts.tstride;
                args.toff = ts.toff;
                args.tile_rows = trows;
                const int g2 = (int)std::min<long long>((hi - lo + 255) / 256, (long long)num_sms() * 4);
                if (nslots + g2 > cap) return arg_fail("workspace too small for the CTA slots");
                pairs_f64_kernel<<<g2, 256, 0, s>>>(args, comp ? 1 : 0, slots + nslots);
                CK_LAUNCH("pairs_f64_kernel");
                nslots += g2;
            }
            if (use_tcs) {
                int ntc = 0;
                rc = launch_tcs(args, ts, claims_tc, slots + nslots, cap - nslots, &ntc, &ntcparts, s,
                                const_cast<unsigned*>(args.tc_bits), args.tc_cpw_pad);
                if (rc) return rc;
                nslots += ntc;
            }
        }
        const long long pr = hi > lo && n >= 2 ? tile_sel_pairs(n, lo, hi, trows, ts, schedule) : 0;
        const double* csum = claims;
        int ncs = nclaims;
        if (direct && (nclaims > 8 * kRedBlocks || ntcparts > 0)) {
            // fixed-order two-stage reduction: FFMA claims into red[0, 128), tensor-core claim
            // partials into red[128, 256)
            double* red = (double*)(ws + lay.red);
            claims_reduce_kernel<<<kRedBlocks, 256, 0, s>>>(claims, nclaims, red);
            CK_LAUNCH("claims_reduce_kernel");
            csum = red;
            ncs = kRedBlocks;
            if (ntcparts > 0) {
                claims_reduce_kernel<<<kRedBlocks, 256, 0, s>>>(claims_tc, ntcparts, red + kRedBlocks);
                CK_LAUNCH("claims_reduce_kernel");
                ncs = 2 * kRedBlocks;
            }
        }
        finalize_kernel<<<1, 256, 0, s>>>(slots, nslots, csum, ncs, direct ? 1 : 0, nclaims + ntcparts / (int)kTcsParts, st, dtype, pr,
                                          direct ? (comp ? 2 : 1) : 0,
                                          dres + k, prof, kern_id, ppc);
        CK_LAUNCH("finalize_kernel");
    }
    return PC_OK;
}

// ------------------------------------------------------------------------
// library-owned per-device scratch for the *_host entry points
// ------------------------------------------------------------------------
struct Arena {
    std::mutex mu;
    void* dev = nullptr;
    size_t cap = 0;
    cudaStream_t stream = nullptr;
};
Arena g_arena[64];

// PAIRCOUNT_POISON=<byte>: fill the scratch with that byte before every call (debug: a kernel that
// reads scratch it did not write then gives different results for different poison bytes)
int poison_byte() {
    static const int v = [] {
        const char* e = getenv("PAIRCOUNT_POISON");
        return e && *e ? (int)(strtol(e, nullptr, 0) & 0xff) : -1;
    }();
    return v;
}

int arena_get(size_t bytes, Arena** out) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    Arena& ar = g_arena[dev & 63];
    if (!ar.stream) CK(cudaStreamCreateWithFlags(&ar.stream, cudaStreamNonBlocking));
    if (ar.cap < bytes) {
        if (ar.dev) CK(cudaFree(ar.dev));
        ar.dev = nullptr;
        ar.cap = 0;
        size_t want = align_up(bytes + bytes / 8, 1 << 20);
        CK(cudaMalloc(&ar.dev, want));
        ar.cap = want;
    }
    if (poison_byte() >= 0) {  // synchronous: callers may run the scratch on their own stream
        CK(cudaMemsetAsync(ar.dev, poison_byte(), ar.cap, ar.stream));
        CK(cudaStreamSynchronize(ar.stream));
    }
    *out = &ar;
    return PC_OK;
}

size_t dtype_bytes(int dtype) { return dtype == PC_F32 || dtype == PC_I32 ? 4 : 8; }

// Pinned host staging for pc_lattice_collisions_vectors / pc_pairs_batch (per device, guarded
// by the arena lock).  Not used by pc_pairs_host: staging 12 MB through it measured ~1 ms
// slower than one pageable cudaMemcpy (scripts/time_e2e.py, r2).
struct Pinned {
    void* p = nullptr;
    size_t cap = 0;
};
Pinned g_pinned[64];

int pinned_get(int dev, size_t bytes, void** out) {
    Pinned& pn = g_pinned[dev & 63];
    if (pn.cap < bytes) {
        if (pn.p) CK(cudaFreeHost(pn.p));
        pn.p = nullptr;
        pn.cap = 0;
        const size_t want = align_up(bytes + bytes / 4, 1 << 20);
        CK(cudaHostAlloc(&pn.p, want, cudaHostAllocDefault));
        pn.cap = want;
    }
    *out = pn.p;
    return PC_OK;
}



#include "lattice.cuh"

// ------------------------------------------------------------------------
// micro-benchmarks for the roofline denominator
// ------------------------------------------------------------------------
__global__ void mb_ffma_kernel(float* out, int iters, float b, float c) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = threadIdx.x * 1e-3f + k;
    const float bb = b * (1.0f + threadIdx.x * 1e-9f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = fmaf(v[k], c, bb);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += v[k];
    if (s == 1234.5f) out[0] = s;
}

__global__ void mb_pairs_kernel(float* out, int iters, float4 c0, float4 c1) {
    constexpr int R = 8;
    float rx[R], ry[R], rz[R], m[R];
#pragma unroll
    for (int r = 0; r < R; ++r) { rx[r] = threadIdx.x * 1e-3f + r; ry[r] = rx[r] * 0.5f; rz[r] = rx[r] * 0.25f; m[r] = -1e30f; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            float t0 = fmaf(rx[r], c0.x, c0.w), t1 = fmaf(rx[r], c1.x, c1.w);
            t0 = fmaf(ry[r], c0.y, t0); t1 = fmaf(ry[r], c1.y, t1);
            t0 = fmaf(rz[r], c0.z, t0); t1 = fmaf(rz[r], c1.z, t1);
            m[r] = max3f(m[r], t0, t1);
        }
        c0.w += 1e-7f;
        c1.w -= 1e-7f;
    }
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) s += m[r];
    if (s == 1234.5f) out[0] = s;
}

}  // namespace

// ==========================================================================
// C ABI
// ==========================================================================
extern "C" {

const char* pc_last_error(void) { return g_err.c_str(); }
const char* pc_version(void) { return "paircount-b200 0.1 (sm_100a)"; }

int pc_device_count(int32_t* count) {
    int c = 0;
    CK(cudaGetDeviceCount(&c));
    *count = c;
    return PC_OK;
}
int pc_set_device(int32_t device) {
    CK(cudaSetDevice(device));
    return PC_OK;
}
int pc_device_alloc(size_t bytes, void** ptr) {
    *ptr = nullptr;
    if (bytes == 0) bytes = 256;
    CK(cudaMalloc(ptr, bytes));
    CK(cudaMemset(*ptr, 0, bytes));
    return PC_OK;
}
int pc_device_free(void* ptr) {
    CK(cudaFree(ptr));
    return PC_OK;
}
int pc_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    return PC_OK;
}
int pc_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    return PC_OK;
}
int pc_stream_sync(void* stream) {
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    return PC_OK;
}

size_t pc_pairs_workspace_bytes(int64_t n, int32_t nranges) {
    (void)nranges;
    return ws_layout(n < 0 ? 0 : n).total;
}

int pc_pairs_async(const void* xyz, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule, int32_t tiling,
                   int32_t nranges, const int64_t* bounds, void* workspace, size_t workspace_bytes,
                   pc_pairs_result* results_device, void* stream) {
    return run_pairs(xyz, dtype, n, interaction, schedule, tiling, nranges, (const long long*)bounds, workspace,
                     workspace_bytes, results_device, (cudaStream_t)stream);
}

int pc_pairs(const void* xyz, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule, int32_t tiling,
             int32_t nranges, const int64_t* bounds, void* workspace, size_t workspace_bytes,
             pc_pairs_result* results, void* stream) {
    if (nranges < 1) return arg_fail("need at least one row range");
    // results live at the tail of the workspace's slot area: use a separate small allocation instead
    pc_pairs_result* dres = nullptr;
    CK(cudaMallocAsync((void**)&dres, sizeof(pc_pairs_result) * nranges, (cudaStream_t)stream));
    int rc = run_pairs(xyz, dtype, n, interaction, schedule, tiling, nranges, (const long long*)bounds, workspace,
                       workspace_bytes, dres, (cudaStream_t)stream);
    if (rc == PC_OK) {
        CK(cudaMemcpyAsync(results, dres, sizeof(pc_pairs_result) * nranges, cudaMemcpyDeviceToHost,
                           (cudaStream_t)stream));
    }
    CK(cudaFreeAsync(dres, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    return rc;
}

}  // extern "C"
namespace {
thread_local pc_pairs_profile g_last_prof;

int pairs_host_run(const void* xyz_host, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                   int32_t tiling, int32_t nranges, const int64_t* bounds, pc_pairs_result* results, TileSel ts) {
    if (dtype < PC_F32 || dtype > PC_I64) return arg_fail("unknown dtype");
    if (n < 0) return arg_fail("negative n");
    if (nranges < 1) return arg_fail("need at least one row range");
    const size_t in_bytes = align_up((size_t)n * 3 * dtype_bytes(dtype), 256);
    const size_t ws_bytes = ws_layout(n).total;
    const size_t res_bytes = align_up(sizeof(pc_pairs_result) * nranges, 256);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_arena[dev & 63].mu);
    Arena* ar = nullptr;
    int rc = arena_get(in_bytes + ws_bytes + res_bytes, &ar);
    if (rc) return rc;
    char* base = (char*)ar->dev;
    cudaStream_t s = ar->stream;
    if (n > 0) CK(cudaMemcpyAsync(base, xyz_host, (size_t)n * 3 * dtype_bytes(dtype), cudaMemcpyHostToDevice, s));
    pc_pairs_result* dres = (pc_pairs_result*)(base + in_bytes + ws_bytes);
    rc = run_pairs(base, dtype, n, interaction, schedule, tiling, nranges, (const long long*)bounds,
                   base + in_bytes, ws_bytes, dres, s, ts);
    const int launches = g_launches;
    if (rc == PC_OK) {
        CK(cudaMemcpyAsync(results, dres, sizeof(pc_pairs_result) * nranges, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&g_last_prof, base + in_bytes + ws_layout(n).prof, sizeof g_last_prof,
                           cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    g_launches = launches;
    return rc;
}
}  // namespace
extern "C" {

int pc_pairs_host(const void* xyz_host, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                  int32_t tiling, int32_t nranges, const int64_t* bounds, pc_pairs_result* results) {
    return pairs_host_run(xyz_host, dtype, n, interaction, schedule, tiling, nranges, bounds, results, TileSel{1, 0});
}

int pc_pairs_part_host(const void* xyz_host, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                       int32_t tiling, int64_t lo, int64_t hi, int32_t part, int32_t nparts, pc_pairs_result* result) {
    const int64_t b[2] = {lo, hi};
    return pairs_host_run(xyz_host, dtype, n, interaction, schedule, tiling, 1, b, result, TileSel{nparts, part});
}

int pc_pairs_part_async(const void* xyz, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                        int32_t tiling, int64_t lo, int64_t hi, int32_t part, int32_t nparts, void* workspace,
                        size_t workspace_bytes, pc_pairs_result* result_device, void* stream) {
    const long long b[2] = {lo, hi};
    return run_pairs(xyz, dtype, n, interaction, schedule, tiling, 1, b, workspace, workspace_bytes, result_device,
                     (cudaStream_t)stream, TileSel{nparts, part});
}

int pc_pairs_last_profile(pc_pairs_profile* out) {
    *out = g_last_prof;
    return PC_OK;
}

int pc_pairs_profile_read(const void* workspace, int64_t n, pc_pairs_profile* out, void* stream) {
    CK(cudaMemcpyAsync(out, (const char*)workspace + ws_layout(n < 0 ? 0 : n).prof, sizeof *out,
                       cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    return PC_OK;
}

int pc_pairs_multi(const void* xyz_host, int32_t dtype, int64_t n, int32_t interaction, int32_t schedule,
                   int32_t tiling, int32_t ndev, const int32_t* devices, const int64_t* bounds,
                   pc_pairs_result* per_device, pc_pairs_result* total) {
    if (ndev < 1 || !devices || !bounds || !per_device || !total) return arg_fail("bad device list");
    if (n < 0) return arg_fail("negative n");
    if (bounds[0] != 0 || bounds[ndev] != n) return arg_fail("device slabs must cover rows [0, n)");
    for (int d = 0; d < ndev; ++d)
        if (bounds[d] > bounds[d + 1]) return arg_fail("device slab bounds must be non-decreasing");
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    for (int d = 0; d < ndev; ++d)
        if (devices[d] < 0 || devices[d] >= count) return arg_fail("device ordinal out of range");
    std::vector<int> rcs((size_t)ndev, PC_OK), launches((size_t)ndev, 0);
    std::vector<std::string> errs((size_t)ndev);
    auto work = [&](int d) {
        int prev = 0;
        cudaGetDevice(&prev);
        if (cudaSetDevice(devices[d]) != cudaSuccess) {
            rcs[d] = PC_ERR_CUDA;
            errs[d] = "cudaSetDevice failed";
            return;
        }
        rcs[d] = pc_pairs_host(xyz_host, dtype, n, interaction, schedule, tiling, 1, bounds + d, per_device + d);
        launches[d] = g_launches;  // thread-local state of this worker thread
        if (rcs[d] != PC_OK) errs[d] = g_err;
        cudaSetDevice(prev);
    };
    // one host thread per slab; slabs on the same device serialise on its arena lock
    std::vector<std::thread> pool;
    for (int d = 1; d < ndev; ++d) pool.emplace_back(work, d);
    work(0);
    for (auto& th : pool) th.join();
    g_launches = 0;
    for (int d = 0; d < ndev; ++d) g_launches += launches[d];
    for (int d = 0; d < ndev; ++d)
        if (rcs[d] != PC_OK) {
            g_err = errs[d];
            return rcs[d];
        }
    // the exchange step: partials combined in ascending device order (deterministic float64 sum)
    pc_pairs_result t;
    memset(&t, 0, sizeof t);
    for (int d = 0; d < ndev; ++d) {
        t.count += per_device[d].count;
        t.sum += per_device[d].sum;
        t.pairs += per_device[d].pairs;
        t.exact_checks += per_device[d].exact_checks;
        if (!t.error) t.error = per_device[d].error;
    }
    *total = t;
    return PC_OK;
}

int pc_lattice_collisions_multi(const void* xyz_host, int32_t dtype, int64_t n, int64_t half_extent, int32_t ndev,
                                const int32_t* devices, pc_lattice_result* per_device, pc_lattice_result* total) {
    if (ndev < 1 || !devices || !per_device || !total) return arg_fail("bad device list");
    if (n < 0 || (n > 0 && !xyz_host)) return arg_fail("bad bead array");
    if (half_extent < 0 || half_extent >= (1LL << 30)) return arg_fail("half_extent out of range");
    if (dtype != PC_I32 && dtype != PC_I64) return arg_fail("lattice beads must be int32 or int64");
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    for (int d = 0; d < ndev; ++d)
        if (devices[d] < 0 || devices[d] >= count) return arg_fail("device ordinal out of range");
    const long long a = half_extent, side = 2 * a + 3, planes = 2 * a + 1;
    std::vector<int> rcs((size_t)ndev, PC_OK);
    std::vector<std::string> errs((size_t)ndev);
    auto work = [&](int d) {
        pc_lattice_result& r = per_device[d];
        memset(&r, 0, sizeof r);
        const long long xlo = -a + planes * d / ndev, xhi = -a + planes * (d + 1) / ndev;
        auto fail = [&](int rc) {
            rcs[d] = rc;
            errs[d] = g_err;
        };
        int prev = 0;
        cudaGetDevice(&prev);
        if (cudaSetDevice(devices[d]) != cudaSuccess) return fail(cuda_fail("cudaSetDevice", cudaGetLastError()));
        MultiLat& ml = g_multilat[devices[d] & 63];
        std::lock_guard<std::mutex> lock(ml.mu);
        auto body = [&]() -> int {
            if (!ml.stream) CK(cudaStreamCreateWithFlags(&ml.stream, cudaStreamNonBlocking));
            cudaStream_t s = ml.stream;
            const size_t in_b = align_up((size_t)n * 3 * dtype_bytes(dtype), 256);
            // slab grids of >= 2^32 cells (a >= 812 on one device, a >= 1024 on two) take 8-byte keys
            const unsigned long long cells = (unsigned long long)(xhi - xlo + 2) * side * side;
            const bool wide_keys = cells >= (1ull << 32);
            const size_t cmp_b = align_up((size_t)n * 12 + 16, 256),
                         key_b = align_up((size_t)n * (wide_keys ? 8 : 4) + 64, 256);
            const size_t need = in_b + cmp_b + key_b + 256;
            if (ml.cap < need) {
                if (ml.buf) CK(cudaFree(ml.buf));
                ml.buf = nullptr;
                ml.cap = 0;
                CK(cudaMalloc(&ml.buf, need + need / 8));
                ml.cap = need + need / 8;
            }
            if (ml.grid_cells < cells) {
                if (ml.grid) CK(cudaFree(ml.grid));
                ml.grid = nullptr;
                ml.grid_cells = 0;
                CK(cudaMalloc(&ml.grid, cells * 4));
                CK(cudaMemsetAsync(ml.grid, 0, cells * 4, s));
                ml.grid_cells = cells;
            }
            char* base = (char*)ml.buf;
            int* cmp = (int*)(base + in_b);
            void* keys = base + in_b + cmp_b;
            unsigned long long* ctr = (unsigned long long*)(base + in_b + cmp_b + key_b);  // [0] kept, [1] bad
            if (n > 0) CK(cudaMemcpyAsync(base, xyz_host, (size_t)n * 3 * dtype_bytes(dtype), cudaMemcpyHostToDevice, s));
            CK(cudaMemsetAsync(ctr, 0, 8, s));
            CK(cudaMemsetAsync(ctr + 1, 0xff, 8, s));
            if (n > 0) {
                const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)num_sms() * 8);
                lat_compact_slab_kernel<<<blocks, 256, 0, s>>>(base, dtype, n, a, xlo, xhi, cmp, ctr, ctr + 1);
                CK_LAUNCH("lat_compact_slab_kernel");
            }
            unsigned long long hc[2] = {0, kNoBad};
            CK(cudaMemcpyAsync(hc, ctr, 16, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            r.beads_processed = n;
            if (hc[1] != kNoBad) {
                r.error = PC_ERR_RANGE;
                r.detail = (long long)hc[1];
                return PC_OK;
            }
            pc_lattice_result sub;
            const int rc = wide_keys ? lattice_run<unsigned long long>(cmp, PC_I32, 1, (long long)hc[0], a, ml.grid,
                                                                       keys, 1, 0, &sub, s, cells)
                                     : lattice_run<unsigned>(cmp, PC_I32, 1, (long long)hc[0], a, ml.grid, keys, 1, 0,
                                                             &sub, s, cells);
            CK(cudaMemsetAsync(ml.grid, 0, cells * 4, s));  // keep the slab grid clean for the next call
            CK(cudaStreamSynchronize(s));
            if (rc == PC_ERR_OVERFLOW) {
                r.error = PC_ERR_OVERFLOW;
                return PC_OK;
            }
            if (rc != PC_OK) return rc;
            r.count = sub.count;
            r.cells_touched = sub.cells_touched;
            return PC_OK;
        };
        const int rc = body();
        if (rc != PC_OK) fail(rc);
        cudaSetDevice(prev);
    };
    std::vector<std::thread> pool;
    for (int d = 1; d < ndev; ++d) pool.emplace_back(work, d);
    work(0);
    for (auto& th : pool) th.join();
    for (int d = 0; d < ndev; ++d)
        if (rcs[d] != PC_OK) {
            g_err = errs[d];
            return rcs[d];
        }
    pc_lattice_result t;
    memset(&t, 0, sizeof t);
    t.beads_processed = n;
    for (int d = 0; d < ndev; ++d) {
        const pc_lattice_result& r = per_device[d];
        if (r.error && !t.error) {
            t.error = r.error;
            t.detail = r.detail;
        }
        t.count += r.count;
        t.cells_touched += r.cells_touched;
    }
    *total = t;
    return PC_OK;
}

int32_t pc_last_launch_count(void) { return g_launches; }

int pc_kernel_timing(int32_t enable) {
    g_timing = enable != 0;
    g_ev_used = 0;
    return PC_OK;
}

int pc_kernel_timing_read_split(double* ms, int32_t* launches) {
    ms[0] = ms[1] = 0.0;
    launches[0] = launches[1] = 0;
    for (int k = 0; k < g_ev_used; ++k) {
        CK(cudaEventSynchronize(g_ev[k].b));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, g_ev[k].a, g_ev[k].b));
        const int kd = g_ev[k].kind == 1 ? 1 : 0;
        ms[kd] += t;
        ++launches[kd];
    }
    g_ev_used = 0;
    return PC_OK;
}

int pc_kernel_timing_read(double* total_ms, int32_t* launches) {
    double t = 0.0;
    for (int k = 0; k < g_ev_used; ++k) {
        CK(cudaEventSynchronize(g_ev[k].b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, g_ev[k].a, g_ev[k].b));
        t += ms;
    }
    *total_ms = t;
    *launches = g_ev_used;
    g_ev_used = 0;
    return PC_OK;
}

int64_t pc_lattice_grid_cells(int64_t half_extent) {
    const int64_t side = 2 * half_extent + 3;
    return side * side * side;
}
int32_t pc_lattice_key_bytes(int64_t half_extent) {
    return pc_lattice_grid_cells(half_extent) < (1LL << 32) ? 4 : 8;
}

int pc_lattice_collisions(const void* xyz, int32_t dtype, int32_t xyz_on_device, int64_t n, int64_t half_extent,
                          uint32_t* grid, void* keys, int32_t assume_clean, pc_lattice_result* result,
                          void* stream) {
    if (half_extent < 0) return arg_fail("half_extent must be >= 0");
    return pc_lattice_key_bytes(half_extent) == 4
               ? lattice_run<unsigned>(xyz, dtype, xyz_on_device, n, half_extent, grid, keys, assume_clean, 0, result,
                                       (cudaStream_t)stream)
               : lattice_run<unsigned long long>(xyz, dtype, xyz_on_device, n, half_extent, grid, keys, assume_clean,
                                                 0, result, (cudaStream_t)stream);
}

int pc_lattice_contacts(const void* xyz, int32_t dtype, int32_t xyz_on_device, int64_t n, int64_t half_extent,
                        uint32_t* grid, void* keys, int32_t assume_clean, pc_lattice_result* result, void* stream) {
    if (half_extent < 0) return arg_fail("half_extent must be >= 0");
    return pc_lattice_key_bytes(half_extent) == 4
               ? lattice_run<unsigned>(xyz, dtype, xyz_on_device, n, half_extent, grid, keys, assume_clean, 1, result,
                                       (cudaStream_t)stream)
               : lattice_run<unsigned long long>(xyz, dtype, xyz_on_device, n, half_extent, grid, keys, assume_clean,
                                                 1, result, (cudaStream_t)stream);
}

int pc_lattice_reset_keys(uint32_t* grid, int64_t half_extent, const void* keys, int64_t nkeys, void* stream) {
    g_launches = 0;
    if (nkeys <= 0) return PC_OK;
    const int nb = lattice_blocks(nkeys);
    cudaStream_t s = (cudaStream_t)stream;
    if (pc_lattice_key_bytes(half_extent) == 4) lat_zero_keys_kernel<unsigned><<<nb, 256, 0, s>>>((const unsigned*)keys, nkeys, grid);
    else lat_zero_keys_kernel<unsigned long long><<<nb, 256, 0, s>>>((const unsigned long long*)keys, nkeys, grid);
    CK_LAUNCH("lat_zero_keys_kernel");
    return PC_OK;
}

}  // extern "C" (reopened below)

namespace {
#include "batch.cuh"
}  // namespace

extern "C" {

int pc_lattice_collisions_batch(const void* xyz, int32_t dtype, int32_t xyz_on_device, const int64_t* offsets,
                                int32_t nvec, int64_t half_extent, pc_lattice_result* results, void* stream) {
    g_launches = 0;
    if (nvec < 0 || !offsets) return arg_fail("bad vector offsets");
    if (half_extent < 0) return arg_fail("half_extent must be >= 0");
    if (dtype != PC_I32 && dtype != PC_I64) return arg_fail("lattice beads must be int32 or int64");
    for (int v = 0; v < nvec; ++v)
        if (offsets[v] < 0 || offsets[v] > offsets[v + 1]) return arg_fail("vector offsets must be non-decreasing");
    if (nvec == 0) return PC_OK;
    const long long n = offsets[nvec];
    const size_t cbytes = xyz_on_device ? 0 : align_up((size_t)n * 3 * dtype_bytes(dtype), 256);
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_arena[dev & 63].mu);
    Arena* ar = nullptr;
    int rc = arena_get(cbytes + batch_tail_bytes(nvec), &ar);
    if (rc) return rc;
    char* base = (char*)ar->dev;
    const void* dxyz = xyz;
    if (!xyz_on_device) {
        if (n > 0) CK(cudaMemcpyAsync(base, xyz, (size_t)n * 3 * dtype_bytes(dtype), cudaMemcpyHostToDevice, s));
        dxyz = base;
    }
    return lat_batch_run(dxyz, dtype, offsets, nvec, half_extent, base + cbytes, results, s);
}

int pc_lattice_collisions_vectors(const void* const* vectors, const int64_t* lengths, int32_t dtype, int32_t nvec,
                                  int64_t half_extent, pc_lattice_result* results, void* stream) {
    g_launches = 0;
    if (nvec < 0 || (nvec > 0 && (!vectors || !lengths))) return arg_fail("bad vector list");
    if (half_extent < 0 || half_extent >= INT32_MAX) return arg_fail("half_extent out of range");
    if (dtype != PC_I32 && dtype != PC_I64) return arg_fail("lattice beads must be int32 or int64");
    if (nvec == 0) return PC_OK;
    std::vector<int64_t> offs((size_t)nvec + 1, 0);
    for (int v = 0; v < nvec; ++v) {
        if (lengths[v] < 0) return arg_fail("vector lengths must be >= 0");
        if (lengths[v] > 0 && !vectors[v]) return arg_fail("null vector pointer");
        offs[v + 1] = offs[v] + lengths[v];
    }
    const long long n = offs[nvec];
    const size_t bbytes = (size_t)n * 3 * 4, cbytes = align_up(bbytes, 256);
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_arena[dev & 63].mu);
    Arena* ar = nullptr;
    int rc = arena_get(cbytes + batch_tail_bytes(nvec), &ar);
    if (rc) return rc;
    char* base = (char*)ar->dev;
    if (n > 0) {
        void* stage = nullptr;
        rc = pinned_get(dev, bbytes, &stage);
        if (rc) return rc;
        split_vectors(nvec, offs.data(), bbytes, [&](int v0, int v1) {
            gather_narrow(vectors, offs.data(), dtype, (int64_t)half_extent, v0, v1, (int32_t*)stage);
        });
        CK(cudaMemcpyAsync(base, stage, bbytes, cudaMemcpyHostToDevice, s));
    }
    return lat_batch_run(base, PC_I32, offs.data(), nvec, half_extent, base + cbytes, results, s);
}

int pc_pairs_batch(const void* const* vectors, const int64_t* lengths, int32_t dtype, int32_t nvec,
                   int32_t interaction, pc_pairs_result* results, void* stream) {
    g_launches = 0;
    if (nvec < 0 || (nvec > 0 && (!vectors || !lengths || !results))) return arg_fail("bad vector list");
    if (dtype < PC_F32 || dtype > PC_I64) return arg_fail("unknown dtype");
    if (interaction < PC_COLLISION || interaction > PC_MANHATTAN1) return arg_fail("unknown interaction");
    if ((interaction == PC_COINCIDE || interaction == PC_MANHATTAN1) && dtype < PC_I32)
        return arg_fail("integer interactions need integer coordinates");
    if (nvec == 0) return PC_OK;
    std::vector<int64_t> offs((size_t)nvec + 1, 0);
    for (int v = 0; v < nvec; ++v) {
        if (lengths[v] < 0) return arg_fail("vector lengths must be >= 0");
        if (lengths[v] > 0 && !vectors[v]) return arg_fail("null vector pointer");
        offs[v + 1] = offs[v] + lengths[v];
    }
    const long long n = offs[nvec];
    const size_t pb = 3 * dtype_bytes(dtype), bbytes = (size_t)n * pb, cbytes = align_up(bbytes, 256);
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_arena[dev & 63].mu);
    Arena* ar = nullptr;
    int rc = arena_get(cbytes + batch_tail_bytes(nvec), &ar);
    if (rc) return rc;
    char* base = (char*)ar->dev;
    if (n > 0) {
        void* stage = nullptr;
        rc = pinned_get(dev, bbytes, &stage);
        if (rc) return rc;
        split_vectors(nvec, offs.data(), bbytes, [&](int v0, int v1) {
            for (int v = v0; v < v1; ++v)
                if (lengths[v]) memcpy((char*)stage + offs[v] * pb, vectors[v], (size_t)lengths[v] * pb);
        });
        CK(cudaMemcpyAsync(base, stage, bbytes, cudaMemcpyHostToDevice, s));
    }
    const size_t obytes = align_up((size_t)(nvec + 1) * 8, 256);
    long long* doffs = (long long*)(base + cbytes);
    unsigned long long* dout = (unsigned long long*)(base + cbytes + obytes);
    CK(cudaMemcpyAsync(doffs, offs.data(), (size_t)(nvec + 1) * 8, cudaMemcpyHostToDevice, s));
    static thread_local bool attr_set[64] = {false};
    if (!attr_set[dev & 63]) {
        CK(cudaFuncSetAttribute(pairs_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairsBatchSmem));
        attr_set[dev & 63] = true;
    }
    const int pred = interaction == PC_COINCIDE ? kPredCoincide : interaction == PC_MANHATTAN1 ? kPredManhattan1
                                                                                               : kPredSphere;
    const int grid = std::min(nvec, 2 * num_sms());
    pairs_batch_kernel<<<grid, 256, kPairsBatchSmem, s>>>(base, dtype, doffs, nvec, pred,
                                                          interaction == PC_COLLISION_INVSQ ? 1 : 0, dout);
    CK_LAUNCH("pairs_batch_kernel");
    std::vector<unsigned long long> host((size_t)nvec * 3);
    CK(cudaMemcpyAsync(host.data(), dout, host.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int v = 0; v < nvec; ++v) {
        pc_pairs_result& r = results[v];
        memset(&r, 0, sizeof r);
        const long long m = lengths[v];
        r.pairs = m * (m - 1) / 2;
        const unsigned long long st = host[3 * v + 2];
        if (st == ~1ull) {
            r.error = PC_ERR_ARG;  // more than kPairsBatchMax points: caller uses pc_pairs_host
        } else if (st) {
            r.error = PC_ERR_DOMAIN;
        } else {
            r.count = (long long)host[3 * v];
            memcpy(&r.sum, &host[3 * v + 1], sizeof r.sum);
            r.exact_checks = r.pairs;
        }
    }
    return PC_OK;
}

int pc_lattice_clear(uint32_t* grid, int64_t half_extent, void* stream) {
    g_launches = 0;
    if (half_extent < 0) return arg_fail("half_extent must be >= 0");
    CK(cudaMemsetAsync(grid, 0, (size_t)pc_lattice_grid_cells(half_extent) * sizeof(uint32_t), (cudaStream_t)stream));
    return PC_OK;
}

int pc_lattice_reset_beads(const void* xyz, int32_t dtype, int32_t xyz_on_device, int64_t n, int64_t half_extent,
                           uint32_t* grid, pc_lattice_result* result, void* stream) {
    g_launches = 0;
    memset(result, 0, sizeof *result);
    if (n <= 0) return PC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_arena[dev & 63].mu);
    Arena* ar = nullptr;
    LatScratch sc;
    int rc = lat_prepare(xyz, dtype, xyz_on_device, n, half_extent, &ar, &sc, &s);
    if (rc) return rc;
    const long long side = 2 * half_extent + 3;
    lat_keys_kernel<unsigned><<<sc.nslots, 256, 0, s>>>(sc.xyz, sc.dtype, n, half_extent, side, nullptr, sc.bad);
    CK_LAUNCH("lat_keys_kernel");
    lat_zero_beads_kernel<<<sc.nslots, 256, 0, s>>>(sc.xyz, sc.dtype, n, half_extent, side, grid, sc.bad);
    CK_LAUNCH("lat_zero_beads_kernel");
    unsigned long long bad = 0;
    CK(cudaMemcpyAsync(&bad, sc.bad, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bad != kNoBad) {
        result->error = PC_ERR_RANGE;
        result->detail = (long long)bad;
        return PC_ERR_RANGE;
    }
    return PC_OK;
}

int pc_grid_count_nonzero(const uint32_t* grid, int64_t cells, int64_t* nonzero, void* stream) {
    g_launches = 0;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* d = nullptr;
    CK(cudaMallocAsync((void**)&d, 8, s));
    CK(cudaMemsetAsync(d, 0, 8, s));
    const long long n4 = cells / 4;
    const int ntail = (int)(cells - n4 * 4);
    const int nb = (int)std::max(1LL, std::min<long long>((n4 + 255) / 256, (long long)num_sms() * 8));
    count_nonzero_kernel<<<nb, 256, 0, s>>>((const uint4*)grid, n4, grid + n4 * 4, ntail, d);
    CK_LAUNCH("count_nonzero_kernel");
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaFreeAsync(d, s));
    CK(cudaStreamSynchronize(s));
    *nonzero = (int64_t)h;
    return PC_OK;
}

int pc_microbench(int32_t kind, double* per_second, double* seconds) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    float* out = nullptr;
    CK(cudaMalloc(&out, 64));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = num_sms() * 8, threads = 256;
    const int iters = kind == 0 ? 65536 : 8192;
    double work;
    for (int rep = 0; rep < 2; ++rep) {  // first pass warms clocks up
        CK(cudaEventRecord(e0, s));
        if (kind == 0) mb_ffma_kernel<<<blocks, threads, 0, s>>>(out, iters, 0.5f, 0.999f);
        else mb_pairs_kernel<<<blocks, threads, 0, s>>>(out, iters, make_float4(0.1f, 0.2f, 0.3f, -1e6f),
                                                        make_float4(0.3f, 0.2f, 0.1f, -1e6f));
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
    }
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    work = (double)blocks * threads * iters * (kind == 0 ? 16.0 : 16.0);  // kind 0: lane-FFMA; kind 1: pairs
    *seconds = ms * 1e-3;
    *per_second = work / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaStreamDestroy(s);
    return PC_OK;
}

}  // extern "C"
