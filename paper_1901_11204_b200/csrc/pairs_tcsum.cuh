// Tensor-core Gram chunks of the sorted inverse-square sum (included by paircount.cu
// inside its anonymous namespace, after pairs_tc.cuh).  DESIGN.md §3 "pairs_tcs_kernel".
//
// The sorted sum kernel (pairs_kernel.cuh, SORTED + DIRECT) evaluates most of its
// chunks in tile-local Gram form, p = A_i + B_j - 2 a_i.b_j with a = q_i - o,
// b = q_j - o about the row tile's centre o: a matrix product plus a per-pair
// epilogue.  Here that product runs on the 5th-generation tensor cores and the
// FP32 pipes are left with the epilogue:
//   * tcgen05.mma.cta_group::1.kind::f16, M = 128 rows (a row half of the 256-row
//     tile), N = 256 columns (the chunk), K = 32 as two K = 16 steps: every coordinate
//     split three ways into exact bf16 pieces x = h + m + l, products
//       a_h.b_{h,m,l} + a_m.b_{h,m,l} + a_l.b_{h,m}    (the b side carries -2)
//       + (A_h + A_m + A_l + A_lo) + (B_h + B_m + B_l + B_lo)
//     with A = 1 + |a|^2, B = |b|^2 computed in float64 and carried as fp32 hi + lo: every
//     product exact in fp32, a_l.b_l (<= 2^-32 |a||b|) dropped.  What remains is the
//     rounding of a = q - o, b = q - o (2u (|a|+|b|)^2) and the tensor core's fp32
//     accumulation, measured at <= 3.2u (1 + (|a|+|b|)^2) over nine geometries
//     (scripts/tc_prec_proto.cu) and allowed 6u: the FFMA Gram form's 8u (|a|+|b|)^2 test.
//   * epilogue: eight terms per two reciprocals, packed: 1/a + 1/c + 1/e + 1/g =
//     ((a+c) eg + (e+g) ac) / (ac eg) in the x lanes (even columns) and the y lanes (odd
//     columns) -- 8 FFMA2/FMUL2/FADD2 + 2 MUFU per eight pairs.
// Which chunks: tcs_classify_kernel's bitmap (or, beyond its size cap, the same test
// in-loop): dense chunks of whole 256-row tiles whose boxes pass tcs_takes() -- the
// Gram test, dmin^2 > 4.5 (no contact in the chunk, so no contact test here), and
// |a|+|b| <= 3e4 (the four-term products stay finite).  The FFMA sorted kernel skips
// exactly these chunks: both form the boxes as unions of the per-32 boxes and evaluate
// chunk_geom() with explicit round-to-nearest operations, so every chunk has one owner.
//
// Work: items (row tile, chunk) of the FFMA kernel's 256 x 256 geometry in tile-major
// order, claimed S at a time from one counter.  An item is two accumulators of 128 x 256
// (the row halves), all 512 TMEM columns.  CTA = 12 warps, one per SM:
//   warp 0       MMA issuer (one elected thread)
//   warps 1-3    producers: claim items, read the bitmap, build the row operand A (256
//                rows, on a tile change) and the column operand B (256 columns, every
//                item, the next item's coordinates already in flight) in shared memory --
//                K-major no-swizzle layout, 512 B per 8 points
//   warps 4-11   drain: group h (4 warps, one per TMEM lane quadrant) reads accumulator h
//                in two rounds of 128 columns, releases it after the second round's loads,
//                and folds the values -- so the next MMA overlaps the last round's arithmetic.
// Sums: each drain warp keeps a float64 partial per claim (its rows and columns of the
// claim's items, in item order) and writes it to claim_sums[claim * 8 + warp]: the
// claim's composition is fixed by its index, so the float64 total is bit-reproducible.

constexpr int kTcsT = 256, kTcsW = 256;           // the FFMA sorted kernel's tile and chunk
constexpr int kTcsKC = 4;                          // K = 32 bf16: four 16-byte K-chunks per point
constexpr int kTcsGroup = kTcsKC * 128;            // bytes per 8 points
constexpr int kTcsOp = 256 / 8 * kTcsGroup;        // bytes per 256-point operand (16 KB)
constexpr int kTcsHalf = kTcsOp / 2;               // 128 points
#ifndef PC_TCS_NQ
#define PC_TCS_NQ 1  // column pieces per row half: accumulators of 256 / NQ columns, 2 NQ of them in TMEM
#endif
constexpr int kTcsNQ = PC_TCS_NQ, kTcsNP = 256 / kTcsNQ, kTcsNAcc = 2 * kTcsNQ;
#ifndef PC_TCS_ROUND
#define PC_TCS_ROUND 64  // accumulator columns per drain round (pipelined: 64 -> 50.3, 32 -> 50.7 ms)
#endif
constexpr int kTcsRound = PC_TCS_ROUND;
static_assert(kTcsNAcc * kTcsNP == 512 && kTcsNP % kTcsRound == 0 && kTcsRound % 32 == 0, "TMEM: 512 columns");
#ifndef PC_TCS_STAGES
#define PC_TCS_STAGES 3  // column stages (G = 4: 2 / 3 stages 61.5 / 61.4 ms; G = 3: 4 beat 3 and 5)
#endif
constexpr int kTcsStages = PC_TCS_STAGES;
#ifndef PC_TCS_KSTEPS  // K = 16 steps per accumulator; a debug knob for A/B of the MMA cost
#define PC_TCS_KSTEPS 2
#endif
#ifndef PC_TCS_PROD
#define PC_TCS_PROD 3  // producer warps: 12 warps in all (142 registers with the pipelined drain); three beat
                       // two by 0.5 ms (two beat three before the pipelined drain; 13 warps take 16 slots)
#endif
#ifndef PC_TCS_EPI
#define PC_TCS_EPI 8  // epilogue warps: 4 per accumulator (each all its columns) or 8 (half the columns each)
#endif
constexpr int kTcsMma = 1, kTcsProd = PC_TCS_PROD, kTcsEpi = PC_TCS_EPI,
              kTcsWarps = kTcsMma + kTcsProd + kTcsEpi;  // one MMA warp, producers, drain warps
constexpr int kTcsEpiG = kTcsEpi / 2, kTcsSpan = kTcsNP * 4 / kTcsEpiG;  // warps per accumulator, columns per warp
static_assert(kTcsNQ == 1 || kTcsEpi == 8, "column-split epilogue for whole-row-half accumulators only");
constexpr int kTcsPT = kTcsProd * 32, kTcsPR = (256 + kTcsPT - 1) / kTcsPT;  // producer threads, points per thread
constexpr int kTcsSmem = (2 * kTcsOrgG + kTcsStages) * kTcsOp + 1024;  // rows [2][G], columns [stages]
constexpr long long kTcsParts = kTcsEpi;           // float64 partials per claim
// instruction descriptor (kind::f16): D f32, A/B bf16, both K-major, N = kTcsNP, M = 128
constexpr uint32_t kTcsIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcsNP >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ bool mbar_test_wait(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}

// exact three-way bf16 split x = h + m + l (round to nearest even; 8 + 8 + 8 significant bits)
__device__ __forceinline__ float bf16r(float x) {  // round to nearest even on the integer pipe (finite x)
    const unsigned u = __float_as_uint(x);
    return __uint_as_float((u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u);
}
__device__ __forceinline__ void split3(float x, float& h, float& m, float& l) {
    h = bf16r(x);
    const float r = __fsub_rn(x, h);
    m = bf16r(r);
    l = bf16r(__fsub_rn(r, m));  // exact: <= 8 significant bits left
}
__device__ __forceinline__ unsigned bf2(float lo, float hi) {  // two exact bf16 values, lo at the lower address
    return (__float_as_uint(hi) & 0xffff0000u) | (__float_as_uint(lo) >> 16);
}
__device__ __forceinline__ unsigned tcs_off(int p, int kc) { return (unsigned)((p >> 3) * kTcsGroup + kc * 128 + (p & 7) * 16); }
// smem matrix descriptor, K-major no swizzle: K-chunks 128 B apart (LBO), 8-point groups kTcsGroup B apart (SBO)
__device__ __forceinline__ uint64_t tcs_desc(unsigned saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)((unsigned)kTcsGroup >> 4) << 32) |
           (1ull << 46);
}
// Two values split three ways at once, as packed bf16x2 words (x in the low half = the lower K
// index): cvt.rn.bf16x2.f32 rounds both to nearest even, the residuals are exact in fp32.
__device__ __forceinline__ unsigned pk2(float lo, float hi) {
    unsigned r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ float lo_f(unsigned w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_f(unsigned w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ void split3x2(float x, float y, unsigned& h, unsigned& m, unsigned& l) {
    h = pk2(x, y);
    const float rx = __fsub_rn(x, lo_f(h)), ry = __fsub_rn(y, hi_f(h));
    m = pk2(rx, ry);
    l = pk2(__fsub_rn(rx, lo_f(m)), __fsub_rn(ry, hi_f(m)));  // exact: <= 8 significant bits left
}
// halves of two words: (lo a, lo b), (lo a, hi b), (hi a, lo b), (hi a, hi b)
__device__ __forceinline__ unsigned ll(unsigned a, unsigned b) { return __byte_perm(a, b, 0x5410); }
__device__ __forceinline__ unsigned lh(unsigned a, unsigned b) { return __byte_perm(a, b, 0x7610); }
__device__ __forceinline__ unsigned hl(unsigned a, unsigned b) { return __byte_perm(a, b, 0x5432); }
__device__ __forceinline__ unsigned hh(unsigned a, unsigned b) { return __byte_perm(a, b, 0x7632); }
constexpr unsigned kBf16One2 = 0x3F803F80u;  // (1, 1)
// The drain folds PC_TCS_FOLD terms per two reciprocals.  Sixteen: the column operand scales every
// p by S = 2^-16 (exact; its ones become S), so for the tensor-core chunks' p in [5.5, 9e8] (dmin^2 >
// 4.5, |a| + |b| <= 3e4) every product of eight S p and its reciprocal stay normal fp32; the sums
// take the factor back (exact).
#ifndef PC_TCS_PIPE
#define PC_TCS_PIPE 1  // drain: the next round's TMEM loads in flight while a round folds (57.5 -> 50.3 ms)
#endif
static_assert(!PC_TCS_PIPE || PC_TCS_ROUND < 256, "a pipelined drain needs two rounds or more");
#ifndef PC_TCS_FOLD
#define PC_TCS_FOLD 8  // (sixteen, scaled: 58.6 vs 57.5 ms at 2^20 -- the drain is latency-, not MUFU-bound)
#endif
static_assert(PC_TCS_FOLD == 8 || PC_TCS_FOLD == 16, "eight or sixteen terms per two reciprocals");
constexpr float kTcsS = PC_TCS_FOLD == 16 ? 1.52587890625e-05f : 1.f;  // 2^-16 or 1
constexpr unsigned kBf16S2 = PC_TCS_FOLD == 16 ? 0x37803780u : kBf16One2;  // (S, S) in bf16

// Row p of the A operand: a = q - o and A = 1 + |a|^2 (float64, carried as fp32 hi + lo), split.
// K order (bf16, 32):  a_h a_h a_h a_m a_m a_m a_l a_l | A_h A_m A_l A_lo | 1 1 1 1
// against the B order  b_h b_m b_l b_h b_m b_l b_h b_m | 1 1 1 1 | B_h B_m B_l B_lo   (each a_*, b_* three
// coordinates): a_h.b_{h,m,l} + a_m.b_{h,m,l} + a_l.b_{h,m} + A + B -- every product exact in fp32, only
// a_l.b_l (<= 2^-32 |a||b|) dropped, and A, B within 2^-32 relative of |a|^2 + 1, |b|^2 of the fp32 a, b.
__device__ __forceinline__ void tcs_write_row(unsigned char* d, int p, float ax, float ay, float az) {
#ifdef PC_TCS_DBG_F32NORM  // debug (timing only): fp32 norms
    const float A = 1.f + ax * ax + ay * ay + az * az, Alo = 0.f;
#else
    const double Ad = 1.0 + (double)ax * ax + (double)ay * ay + (double)az * az;  // products exact in float64
    const float A = (float)Ad, Alo = (float)(Ad - (double)A);
#endif
    unsigned XYh, XYm, XYl, ZAh, ZAm, ZAl;
    split3x2(ax, ay, XYh, XYm, XYl);
    split3x2(az, A, ZAh, ZAm, ZAl);
    const unsigned lo2 = pk2(Alo, Alo);
    *reinterpret_cast<uint4*>(d + tcs_off(p, 0)) = make_uint4(XYh, ll(ZAh, XYh), hl(XYh, ZAh), XYh);
    *reinterpret_cast<uint4*>(d + tcs_off(p, 1)) = make_uint4(ll(ZAh, XYm), hl(XYm, ZAm), XYm, ll(ZAm, XYm));
    *reinterpret_cast<uint4*>(d + tcs_off(p, 2)) = make_uint4(hl(XYm, ZAm), XYl, ll(ZAl, XYl), hl(XYl, ZAl));
    *reinterpret_cast<uint4*>(d + tcs_off(p, 3)) = make_uint4(hh(ZAh, ZAm), hl(ZAl, lo2), kBf16One2, kBf16One2);
}
// Column p of the B operand from b = q - o: the products carry -2b (exact), B = |b|^2 (float64 hi + lo)
__device__ __forceinline__ void tcs_write_col(unsigned char* d, int p, float bx, float by, float bz) {
#ifdef PC_TCS_DBG_F32NORM
    const float B = bx * bx + by * by + bz * bz, Blo = 0.f;
#else
    const double Bd = (double)bx * bx + (double)by * by + (double)bz * bz;
    const float B = (float)Bd, Blo = (float)(Bd - (double)B);
#endif
    unsigned XYh, XYm, XYl, ZBh, ZBm, ZBl;
    constexpr float m2 = -2.f * kTcsS;
    split3x2(m2 * bx, m2 * by, XYh, XYm, XYl);
    split3x2(m2 * bz, kTcsS * B, ZBh, ZBm, ZBl);
    const unsigned lo2 = pk2(kTcsS * Blo, kTcsS * Blo);
    *reinterpret_cast<uint4*>(d + tcs_off(p, 0)) = make_uint4(XYh, ll(ZBh, XYm), hl(XYm, ZBm), XYl);
    *reinterpret_cast<uint4*>(d + tcs_off(p, 1)) = make_uint4(ll(ZBl, XYh), hl(XYh, ZBh), XYm, ll(ZBm, XYl));
    *reinterpret_cast<uint4*>(d + tcs_off(p, 2)) = make_uint4(hl(XYl, ZBl), XYh, ll(ZBh, XYm), hl(XYm, ZBm));
    *reinterpret_cast<uint4*>(d + tcs_off(p, 3)) = make_uint4(kBf16S2, kBf16S2, hh(ZBh, ZBm), hh(ZBl, lo2));
}

// Chunk bitmap: bit t * cpw_pad + c set when pairs_tcs_kernel evaluates chunk c of row tile t (whole
// 32-bit words per tile, so one warp writes a tile's row with ballots).  Sized for the whole range;
// beyond kTcsBitsMax (n > ~2^23) both kernels classify in-loop instead.
constexpr size_t kTcsBitsMax = (size_t)64 << 20;
__host__ __device__ inline long long tcs_cpw(long long n) { return ((long long)(kTcsT - 1) + n / 2 + kTcsW - 1) / kTcsW; }
__host__ __device__ inline long long tcs_cpw_pad(long long n) { return (tcs_cpw(n) + 31) / 32 * 32; }
inline size_t tcs_bits_bytes(long long n) {
    const size_t b = (size_t)((n + kTcsT - 1) / kTcsT) * (size_t)tcs_cpw_pad(n) / 8;
    return b <= kTcsBitsMax ? (b + 255) / 256 * 256 : 0;
}

struct TcsArgs {
    const void* xyz;   // sorted points (fp32, or float64 for the compensated path)
    const float4* blk_box;
    const PrepStats* st;
    Slot* slots;
    double* claim_sums;  // kTcsParts per claim
    unsigned long long* work_ctr;
    int dtype, n, lo, hi;
    int tstride, toff, n_tiles;
    long long L;       // window length (T - 1 + n/2)
    long long cpw;     // chunks per window
    int G;             // tiles per work unit: kTcsOrgG (pairs_tcs2_kernel: 1)
    long long upg;     // units per group of G tiles: cpw + G - 1 diagonals
    long long items;   // work units: ceil(n_tiles / G) * upg (pairs_tcs2_kernel: G = 1, n_tiles * cpw)
    long long S;       // units per claim
    long long nclaims;
    unsigned* bits;    // chunk bitmap (tcs_classify_kernel writes it, the kernels read it), or null
    long long cpw_pad;
    const float4* cbox;  // classify: the box of the chunk starting at 256 m + 1 (n, lo multiples of 256), or null
};

// In-loop classification of item (call tile i, chunk c) by one thread (no bitmap: n > ~2^23): the same
// boxes tcs_classify_kernel unions across its lanes, so the same decision.
__device__ __noinline__ bool tcs_item_takes(const float4* __restrict__ blk_box, int n, int lo, int hi, int tabs,
                                            long long L, long long c) {
    const int steps_min = (n & 1) ? (n - 1) >> 1 : (n >> 1) - 1;
    const int i0 = lo + tabs * kTcsT;
    const long long off = c * kTcsW;
    if (!(off + kTcsW <= L && i0 + kTcsT <= hi && off + 1 >= kTcsT && off + kTcsW <= steps_min)) return false;
    auto add = [&](int b, float (&mn)[3], float (&mx)[3]) {
        const float4 lo4 = __ldg(blk_box + 2 * b), hi4 = __ldg(blk_box + 2 * b + 1);
        mn[0] = fminf(mn[0], lo4.x); mn[1] = fminf(mn[1], lo4.y); mn[2] = fminf(mn[2], lo4.z);
        mx[0] = fmaxf(mx[0], hi4.x); mx[1] = fmaxf(mx[1], hi4.y); mx[2] = fmaxf(mx[2], hi4.z);
    };
    float tmin[3] = {INFINITY, INFINITY, INFINITY}, tmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = 0; q < kTcsT / 32; ++q) add((i0 >> 5) + q, tmin, tmax);
    float gmin[3] = {INFINITY, INFINITY, INFINITY}, gmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = 0; k < kTcsOrgG; ++k) {  // tcs_group_box, one thread
        const int tq = tabs / kTcsOrgG * kTcsOrgG + k;
        if ((long long)lo + 256ll * (tq + 1) > hi) continue;
        for (int q = 0; q < 8; ++q) add((lo >> 5) + 8 * tq + q, gmin, gmax);
    }
    // the chunk's box: one or two runs of per-32 boxes (the FFMA kernel's blocks)
    int jw = i0 + (int)off + 1;
    if (jw >= n) jw -= n;
    const int jend = jw + kTcsW - 1;
    const int nb1 = (min(jend, n - 1) >> 5) - (jw >> 5) + 1;
    const int nb2 = jend >= n ? ((jend - n) >> 5) + 1 : 0;
    float cl[3] = {INFINITY, INFINITY, INFINITY}, ch[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = 0; q < nb1 + nb2; ++q) add(q < nb1 ? (jw >> 5) + q : q - nb1, cl, ch);
    return tcs_takes(chunk_geom_g(tmin, tmax, gmin, gmax, cl, ch));
}

// Per-chunk boxes when every chunk starts at 256 m + 1 (n and lo multiples of 256): chunk m covers the
// per-32 blocks 8m .. 8m+8 (mod n / 32), the blocks the FFMA kernel unions for it.
__global__ void __launch_bounds__(256) tcs_chunk_box_kernel(const float4* __restrict__ box, int nblk, int nchunk,
                                                            float4* __restrict__ cbox) {
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < nchunk; m += gridDim.x * blockDim.x) {
        float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.f), hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
#pragma unroll
        for (int q = 0; q <= kTcsW / 32; ++q) {
            int b = 8 * m + q;
            if (b >= nblk) b -= nblk;
            const float4 l = box[2 * b], h = box[2 * b + 1];
            lo = make_float4(fminf(lo.x, l.x), fminf(lo.y, l.y), fminf(lo.z, l.z), 0.f);
            hi = make_float4(fmaxf(hi.x, h.x), fmaxf(hi.y, h.y), fmaxf(hi.z, h.z), 0.f);
        }
        cbox[2 * m] = lo;
        cbox[2 * m + 1] = hi;
    }
}

// The chunk bitmap: one warp per 32-chunk word of a row tile, a lane per chunk (the tile's box from its
// eight per-32 boxes, each chunk's from its nine -- the unions the FFMA kernel forms, min / max exact).
__global__ void __launch_bounds__(256) tcs_classify_kernel(const TcsArgs a) {
    const int lane = threadIdx.x & 31;
    const long long wg = (long long)blockIdx.x * 8 + (threadIdx.x >> 5), words = a.cpw_pad / 32;
    const long long t = wg / words, c0 = (wg - t * words) * 32;  // one warp per 32-chunk word of a tile
    if (t >= a.n_tiles) return;
    const int n = a.n;
    const int steps_min = (n & 1) ? (n - 1) >> 1 : (n >> 1) - 1;
    const int i0 = a.lo + tile_abs((int)t, a.tstride, a.toff) * kTcsT;
    const bool rows_ok = i0 + kTcsT <= a.hi;
    float tmin[3] = {INFINITY, INFINITY, INFINITY}, tmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    if (rows_ok) {
        float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
        if (lane < kTcsT / 32) {
            const float4 lo4 = a.blk_box[2 * ((i0 >> 5) + lane)], hi4 = a.blk_box[2 * ((i0 >> 5) + lane) + 1];
            mn[0] = lo4.x; mn[1] = lo4.y; mn[2] = lo4.z;
            mx[0] = hi4.x; mx[1] = hi4.y; mx[2] = hi4.z;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            tmin[k] = warp_min_f(mn[k]);
            tmax[k] = warp_max_f(mx[k]);
        }
    }
    float gmin[3] = {0.f, 0.f, 0.f}, gmax[3] = {0.f, 0.f, 0.f};  // the origin group's box
    if (rows_ok) tcs_group_box(a.blk_box, a.lo, a.hi, tile_abs((int)t, a.tstride, a.toff), lane, gmin, gmax);
    {
        const long long c = c0 + lane;
        const long long off = c * kTcsW;
        bool take = false;
        if (rows_ok && c < a.cpw && off + kTcsW <= a.L && off + 1 >= kTcsT && off + kTcsW <= steps_min) {
            int jw = i0 + (int)off + 1;
            if (jw >= n) jw -= n;
            const int jend = jw + kTcsW - 1;
            const int nb1 = (min(jend, n - 1) >> 5) - (jw >> 5) + 1;
            const int nb2 = jend >= n ? ((jend - n) >> 5) + 1 : 0;
            float cl[3] = {INFINITY, INFINITY, INFINITY}, ch[3] = {-INFINITY, -INFINITY, -INFINITY};
            if (a.cbox) {  // the same union, precomputed (aligned chunk starts)
                PC_CHECK(((jw - 1) & 255) == 0);
                const float4 lo4 = __ldg(a.cbox + 2 * ((jw - 1) >> 8)), hi4 = __ldg(a.cbox + 2 * ((jw - 1) >> 8) + 1);
                cl[0] = lo4.x; cl[1] = lo4.y; cl[2] = lo4.z;
                ch[0] = hi4.x; ch[1] = hi4.y; ch[2] = hi4.z;
            } else
#pragma unroll
            for (int q = 0; q < kTcsW / 32 + 2; ++q) {  // <= 9 blocks, 10 when the window wraps
                if (q < nb1 + nb2) {
                    const int bq = q < nb1 ? (jw >> 5) + q : q - nb1;
                    const float4 lo4 = __ldg(a.blk_box + 2 * bq), hi4 = __ldg(a.blk_box + 2 * bq + 1);
                    cl[0] = fminf(cl[0], lo4.x); cl[1] = fminf(cl[1], lo4.y); cl[2] = fminf(cl[2], lo4.z);
                    ch[0] = fmaxf(ch[0], hi4.x); ch[1] = fmaxf(ch[1], hi4.y); ch[2] = fmaxf(ch[2], hi4.z);
                }
            }
            take = tcs_takes(chunk_geom_g(tmin, tmax, gmin, gmax, cl, ch));
        }
        const unsigned w = __ballot_sync(0xffffffffu, take);
        PC_CHECK(t * a.cpw_pad + c0 + 32 <= (long long)a.n_tiles * a.cpw_pad);
        if (lane == 0) a.bits[(t * a.cpw_pad + c0) >> 5] = w;
    }
}

// T = float: fp32 points, a = fl32(q - o); T = double: float64 points (the sorted compensated path),
// a = fl32((q - c) - o) with c the bounding-box centre the FFMA kernel's centred boxes use -- one
// rounding either way, so the same error bound holds.
template <typename T>
__global__ void __launch_bounds__(kTcsWarps * 32) pairs_tcs_kernel(const TcsArgs a) {
    constexpr bool kF64 = sizeof(T) == 8;
    extern __shared__ __align__(1024) unsigned char tcs_smem[];
    unsigned char* base = (unsigned char*)(((uintptr_t)tcs_smem + 1023) & ~(uintptr_t)1023);
    unsigned char* sA = base;                         // [2][kTcsOrgG][kTcsOp]: a group's row operands
    unsigned char* sB = base + 2 * kTcsOrgG * kTcsOp; // [kTcsStages][kTcsOp]: column operands
    __shared__ __align__(8) unsigned long long bar_bfull[kTcsStages], bar_bempty[kTcsStages];
    __shared__ __align__(8) unsigned long long bar_afull[2], bar_aempty[2];
    __shared__ __align__(8) unsigned long long bar_accfull[kTcsNAcc], bar_accempty[kTcsNAcc];  // index h NQ + q
    __shared__ long long s_item[kTcsStages];  // claim << 8 | item mask << 2 | abuf << 1 | new group; -1 = done
    __shared__ long long s_meta[kTcsNAcc];    // MMA -> epilogue: the accumulator's claim (-1 = done)
    __shared__ long long s_pclaim[2];
    __shared__ unsigned s_tmem;
    __shared__ unsigned s_items;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool skip = f64_takes(*a.st, a.dtype, kF64);  // the float64 kernel takes this call
    if (skip || a.n_tiles == 0) {
        if (threadIdx.x == 0) a.slots[blockIdx.x] = Slot{};
        return;
    }
    const unsigned b_full = (unsigned)__cvta_generic_to_shared(bar_bfull);
    const unsigned b_empty = (unsigned)__cvta_generic_to_shared(bar_bempty);
    const unsigned a_full = (unsigned)__cvta_generic_to_shared(bar_afull);
    const unsigned a_empty = (unsigned)__cvta_generic_to_shared(bar_aempty);
    const unsigned acc_full = (unsigned)__cvta_generic_to_shared(bar_accfull);
    const unsigned acc_empty = (unsigned)__cvta_generic_to_shared(bar_accempty);
    if (threadIdx.x == 0) {
        for (int k = 0; k < kTcsStages; ++k) {
            mbar_init(b_full + 8 * k, kTcsProd);
            mbar_init(b_empty + 8 * k, kTcsMma);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(a_full + 8 * k, kTcsProd);
            mbar_init(a_empty + 8 * k, kTcsMma);
        }
        for (int k = 0; k < kTcsNAcc; ++k) {
            mbar_init(acc_full + 8 * k, 2);  // the MMA thread's hand-off + the MMAs' commit
            mbar_init(acc_empty + 8 * k, kTcsEpiG);
        }
        mbar_init_fence();
        s_items = 0;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (unsigned)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = s_tmem;
    const int n = a.n;
    const int steps_min = (n & 1) ? (n - 1) >> 1 : (n >> 1) - 1;
    double sum = 0.0;

    if (warp == 0) {
        // ---------------- MMA issuer (one elected thread): per stage, the unit's items -- tile k of
        // the group against the stage's column operand, for each bit k of the unit's item mask
        if (lane == 0) {
            long long it = 0, fills = 0;  // stages consumed, items issued (each fills both accumulators)
            long long aloads[2] = {0, 0};
            int cur_abuf = -1, sg = 0;
            // (the operands stay inside the 256 KB window of the 14-bit address field: offsets add)
            const uint64_t dA0 = tcs_desc((unsigned)__cvta_generic_to_shared(sA));
            const uint64_t dB0 = tcs_desc((unsigned)__cvta_generic_to_shared(sB));
            for (;; ++it, sg = sg + 1 == kTcsStages ? 0 : sg + 1) {
                mbar_wait(b_full + 8 * sg, (unsigned)((it / kTcsStages) & 1));
                const long long tag = s_item[sg];
                if (tag < 0) {
                    for (int k = 0; k < kTcsNAcc; ++k) {
                        if (fills >= 1) mbar_wait(acc_empty + 8 * k, (unsigned)((fills - 1) & 1));
                        s_meta[k] = -1;
                        mbar_arrive_plain(acc_full + 8 * k);
                        mbar_arrive_plain(acc_full + 8 * k);
                    }
                    break;
                }
                const int ab = (int)((tag >> 1) & 1);
                if (tag & 1) {  // first unit of a group: its rows landed; the previous rows are free after the MMAs so far
                    if (cur_abuf >= 0) tc_commit(a_empty + 8 * cur_abuf);
                    mbar_wait(a_full + 8 * ab, (unsigned)(aloads[ab] & 1));
                    ++aloads[ab];
                    cur_abuf = ab;
                }
                const uint64_t db0 = dB0 + (uint64_t)((sg * kTcsOp) >> 4);
                for (unsigned km = (unsigned)((tag >> 2) & 0xF); km; km &= km - 1) {
                    const int g = __ffs(km) - 1;
                    // descriptors: the base descriptor plus the 16-byte-unit offset (start address field)
                    const uint64_t da0 = dA0 + (uint64_t)(((ab * kTcsOrgG + g) * kTcsOp) >> 4);
#pragma unroll
                    for (int kk = 0; kk < kTcsNAcc; ++kk) {
                        // accumulator k = (row half h, column piece q) = h NQ + q, in the order the two
                        // epilogue groups release them: (0,0), (1,0), (0,1), (1,1), ...
                        const int h = kk & 1, q = kk >> 1, k = h * kTcsNQ + q;
                        if (fills >= 1) mbar_wait(acc_empty + 8 * k, (unsigned)((fills - 1) & 1));
                        s_meta[k] = tag >> 8;
                        mbar_arrive_plain(acc_full + 8 * k);  // release: the epilogue reads s_meta after its wait
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint64_t da = da0 + (uint64_t)((h * kTcsHalf) >> 4),
                                       db = db0 + (uint64_t)((q * (kTcsNP / 8) * kTcsGroup) >> 4);
#pragma unroll
                        for (int ks = 0; ks < PC_TCS_KSTEPS; ++ks) {
                            asm volatile(
                                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                                " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + (unsigned)(k * kTcsNP)),
                                "l"(da + (uint64_t)(16 * ks)), "l"(db + (uint64_t)(16 * ks)), "r"(kTcsIdesc), "r"(ks));
                        }
                        tc_commit(acc_full + 8 * k);
                    }
                    ++fills;
                }
                tc_commit(b_empty + 8 * sg);
            }
            s_items = (unsigned)fills;
        }
    } else if (warp < 1 + kTcsProd) {
        // ---------------- producers: claims, item masks, operands
        // Work units: (call group gc, diagonal d) -> the items (tile gc G + k, chunk d - k), k < G, which
        // all cover the columns from row0(gc G) + 256 d + 1.  Per claim the units are examined 32 at a
        // time (lane l: unit ub + l, its items' bitmap bits or in-loop tests), and the units with items
        // are built in order -- the group's G row operands on a group change, then ONE column operand
        // for the unit's items -- with the next unit's column coordinates already in flight.
        const int pw = warp - 1, tid = pw * 32 + lane;
        long long it = 0, nclaim = 0;
        int sg = 0, abuf = 1, o_grp = -1;
        long long aloads[2] = {0, 0};
        long long a_grp = -1;
        float o[3] = {0.f, 0.f, 0.f};
        const long long C = a.cpw, UPG = a.upg;
        const int G = a.G;
        auto row0t = [&](int tt) -> int { return a.lo + tile_abs(tt, a.tstride, a.toff) * kTcsT; };
        auto unit_col = [&](long long u, long long& gc) -> int {  // the unit's group and first column, wrapped
            gc = u / UPG;
            const int j0 = row0t((int)(gc * G)) + (int)(u - gc * UPG) * kTcsW + 1;
            return j0 >= n ? j0 - n : j0;
        };
        auto unit_mask = [&](long long u) -> unsigned {  // bit k: item (gc G + k, d - k) is a tensor-core chunk
            const long long gc = u / UPG, d = u - gc * UPG;
            unsigned km = 0;
            for (int k = 0; k < G; ++k) {
                const long long i = gc * G + k, ch = d - k;
                if (i >= a.n_tiles || ch < 0 || ch >= C) continue;
                bool take;
                if (a.bits) {
                    const long long b = i * a.cpw_pad + ch;
                    take = (__ldg(a.bits + (b >> 5)) >> (b & 31)) & 1u;
                } else {
                    take = tcs_item_takes(a.blk_box, n, a.lo, a.hi, tile_abs((int)i, a.tstride, a.toff), a.L, ch);
                }
                km |= (take ? 1u : 0u) << k;
            }
            return km;
        };
        const T* xyz = (const T*)a.xyz;
        double cc[3] = {0.0, 0.0, 0.0};  // float64 points: the bounding-box centre of the centred boxes
        if (kF64) {
            long long ci[3];
            bbox_centre(*a.st, PC_F64, cc, ci);
        }
        auto load_cols = [&](int jw, T (&q)[3 * kTcsPR]) {
#pragma unroll
            for (int h = 0; h < kTcsPR; ++h) {
                int j = jw + min(tid + kTcsPT * h, 255);
                if (j >= n) j -= n;
                PC_CHECK(j >= 0 && j < n);
                const T* src = xyz + 3ll * j;
                q[3 * h] = __ldg(src);
                q[3 * h + 1] = __ldg(src + 1);
                q[3 * h + 2] = __ldg(src + 2);
            }
        };
        auto rel = [&](T q, int k) -> float {  // the coordinate relative to the group centre o, one rounding
            if constexpr (kF64) return (float)(((double)q - cc[k]) - (double)o[k]);
            else return __fsub_rn((float)q, o[k]);
        };
        for (;; ++nclaim) {
            if (tid == 0) s_pclaim[nclaim & 1] = (long long)atomicAdd(a.work_ctr, 1ull);
            asm volatile("bar.sync 1, %0;" ::"r"(kTcsProd * 32) : "memory");
            const long long c = s_pclaim[nclaim & 1];
            if (c >= a.nclaims) break;
            const long long u0 = c * a.S, u1 = min(u0 + a.S, a.items);
            for (long long ub = u0; ub < u1; ub += 32) {
                const unsigned km = ub + lane < u1 ? unit_mask(ub + lane) : 0u;
                unsigned mask = __ballot_sync(0xffffffffu, km != 0u);
                if (!mask) continue;
                // ---- the units with items, in order, one ahead in flight
                T cur[3 * kTcsPR], nxt[3 * kTcsPR];
                int e = __ffs(mask) - 1;
                mask &= mask - 1;
                long long egc;
                load_cols(unit_col(ub + e, egc), cur);
                for (;;) {
                    const int e2 = mask ? __ffs(mask) - 1 : -1;
                    if (mask) mask &= mask - 1;
                    long long ngc = 0;
                    if (e2 >= 0) load_cols(unit_col(ub + e2, ngc), nxt);
                    const unsigned ekm = __shfl_sync(0xffffffffu, km, e);
                    long long flag = 0;
                    if (egc != a_grp) {
                        // the origin: the centre of the origin group's box (chunk_geom_g's o)
                        const int tabs = tile_abs((int)(egc * G), a.tstride, a.toff);
                        if (tabs / kTcsOrgG != o_grp) {
                            o_grp = tabs / kTcsOrgG;
                            float gmn[3], gmx[3];
                            tcs_group_box(a.blk_box, a.lo, a.hi, tabs, lane, gmn, gmx);
#pragma unroll
                            for (int k = 0; k < 3; ++k) o[k] = __fmul_rn(0.5f, __fadd_rn(gmn[k], gmx[k]));
                        }
                        // the row operands of the group's full tiles: a = q - o, A = 1 + |a|^2, three-way splits
                        abuf ^= 1;
                        if (aloads[abuf] > 0) mbar_wait(a_empty + 8 * abuf, (unsigned)((aloads[abuf] - 1) & 1));
                        for (int k = 0; k < G; ++k) {
                            const long long i = egc * G + k;
                            const int i0 = row0t((int)i);
                            if (i >= a.n_tiles || i0 + kTcsT > a.hi) continue;
                            unsigned char* dA = sA + (abuf * kTcsOrgG + k) * kTcsOp;
#pragma unroll
                            for (int h = 0; h < kTcsPR; ++h) {
                                const int p = tid + kTcsPT * h;
                                if (p >= 256) break;
                                PC_CHECK(i0 + p >= a.lo && i0 + p < a.hi);
                                const T* q = xyz + 3ll * (i0 + p);
                                const float ax = rel(q[0], 0), ay = rel(q[1], 1), az = rel(q[2], 2);
                                tcs_write_row(dA, p, ax, ay, az);
                            }
                        }
                        fence_proxy_async_shared();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_plain(a_full + 8 * abuf);
                        ++aloads[abuf];
                        a_grp = egc;
                        flag = 1;
                    }
                    // the column operand: b = q - o (carrying -2), B = |b|^2
                    if (it >= kTcsStages) mbar_wait(b_empty + 8 * sg, (unsigned)(((it / kTcsStages) - 1) & 1));
                    unsigned char* dB = sB + sg * kTcsOp;
#ifdef PC_TCS_DBG_NOBUILD  // debug (timing only): keep whatever the stage holds
                    if (it < kTcsStages)
#endif
#pragma unroll
                    for (int h = 0; h < kTcsPR; ++h) {
                        const int p = tid + kTcsPT * h;
                        if (p >= 256) break;
                        const float bx = rel(cur[3 * h], 0), by = rel(cur[3 * h + 1], 1), bz = rel(cur[3 * h + 2], 2);
                        tcs_write_col(dB, p, bx, by, bz);
                    }
                    fence_proxy_async_shared();
                    __syncwarp();
                    if (tid == 0) s_item[sg] = (c << 8) | ((long long)ekm << 2) | ((long long)abuf << 1) | flag;
                    if (lane == 0) mbar_arrive_plain(b_full + 8 * sg);
                    ++it;
                    sg = sg + 1 == kTcsStages ? 0 : sg + 1;
                    if (e2 < 0) break;
                    e = e2;
                    egc = ngc;
#pragma unroll
                    for (int k = 0; k < 3 * kTcsPR; ++k) cur[k] = nxt[k];
                }
            }
        }
        // end of the work: a sentinel item
        if (it >= kTcsStages) mbar_wait(b_empty + 8 * sg, (unsigned)(((it / kTcsStages) - 1) & 1));
        if (tid == 0) s_item[sg] = -1;
        if (lane == 0) mbar_arrive_plain(b_full + 8 * sg);
    } else {
        // ---------------- epilogue: group h drains accumulators (h, 0) and (h, 1), lane quadrant warp % 4
        const int ew = warp - kTcsMma - kTcsProd, h = ew / kTcsEpiG, quad = warp & 3, cpart = (ew % kTcsEpiG) >> 2;
        long long cur = -1;
        for (long long it = 0;; ++it) {
            bool done = false;
#pragma unroll 1
            for (int q = 0; q < kTcsNQ; ++q) {
                const int k = h * kTcsNQ + q;
                mbar_wait(acc_full + 8 * k, (unsigned)(it & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const long long claim = s_meta[k];
                if (claim < 0) {
                    done = true;
                    break;
                }
                if (claim != cur) {
                    if (cur >= 0) {
                        const double cs = warp_sum(sum);
                        PC_CHECK(cur < a.nclaims);
                        if (lane == 0) a.claim_sums[cur * kTcsParts + ew] = cs;
                        sum = 0.0;
                    }
                    cur = claim;
                }
                // the accumulator in rounds of kTcsRound columns; released after the last round's loads
                const unsigned tbase = tmem + ((unsigned)(quad * 32) << 16) + (unsigned)(k * kTcsNP + cpart * kTcsSpan);
                float2 acc = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);  // two chains
                // the fold of one round's values: eight (or sixteen) terms per two reciprocals, two chains
                auto fold = [&](unsigned (&v)[kTcsRound / 32][32]) {
#pragma unroll
                    for (int w = 0; w < kTcsRound / 32; ++w) {
#pragma unroll
                        for (int e = 0; e < 32; e += PC_TCS_FOLD) {
                            // four terms (x lanes: even columns, y lanes: odd) -> numerator and denominator
                            auto quad = [&](int f, float2& Nq, float2& Pq) {
                                const float2 p1 = make_float2(__uint_as_float(v[w][f]), __uint_as_float(v[w][f + 1]));
                                const float2 p2 = make_float2(__uint_as_float(v[w][f + 2]), __uint_as_float(v[w][f + 3]));
                                const float2 p3 = make_float2(__uint_as_float(v[w][f + 4]), __uint_as_float(v[w][f + 5]));
                                const float2 p4 = make_float2(__uint_as_float(v[w][f + 6]), __uint_as_float(v[w][f + 7]));
                                const float2 m12 = __fmul2_rn(p1, p2), s12 = __fadd2_rn(p1, p2);
                                const float2 m34 = __fmul2_rn(p3, p4), s34 = __fadd2_rn(p3, p4);
                                Pq = __fmul2_rn(m12, m34);
                                Nq = __ffma2_rn(s34, m12, __fmul2_rn(s12, m34));
                            };
                            float2 Nn, P;
                            quad(e, Nn, P);
                            if (PC_TCS_FOLD == 16) {  // 1/a + ... + 1/h = (N1 P2 + N2 P1) / (P1 P2)
                                float2 N2, P2;
                                quad(e + 8, N2, P2);
                                Nn = __ffma2_rn(Nn, P2, __fmul2_rn(N2, P));
                                P = __fmul2_rn(P, P2);
                            }
                            if (PC_TCS_FOLD == 8 ? (e & 8) : (e & 16))  // two chains
                                acc2 = __ffma2_rn(Nn, make_float2(rcp_approx(P.x), rcp_approx(P.y)), acc2);
                            else acc = __ffma2_rn(Nn, make_float2(rcp_approx(P.x), rcp_approx(P.y)), acc);
                        }
                    }
                };
#if PC_TCS_PIPE
                // two buffers of kTcsRound columns: the next round's loads in flight while this one folds
                // (released after the last round's loads, as below)
                {
                    constexpr int NR = kTcsSpan / kTcsRound;
                    unsigned va[kTcsRound / 32][32], vb[kTcsRound / 32][32];
#pragma unroll
                    for (int w = 0; w < kTcsRound / 32; ++w) PC_TC_LD32(va[w], tbase + 32u * w);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int rd = 0; rd < NR; ++rd) {
                        unsigned(&vc)[kTcsRound / 32][32] = (rd & 1) ? vb : va;
                        unsigned(&vn)[kTcsRound / 32][32] = (rd & 1) ? va : vb;
                        if (rd + 1 < NR) {
#pragma unroll
                            for (int w = 0; w < kTcsRound / 32; ++w)
                                PC_TC_LD32(vn[w], tbase + (unsigned)(kTcsRound * (rd + 1)) + 32u * w);
                        }
                        fold(vc);
                        if (rd + 1 < NR) {
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                            for (int w = 0; w < kTcsRound / 32; ++w)
#pragma unroll
                                for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(vn[w][i]));  // (after the wait)
                            if (rd + 1 == NR - 1) {
                                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                                __syncwarp();
                                if (lane == 0) mbar_arrive_plain(acc_empty + 8 * k);
                            }
                        }
                    }
                }
#else
#pragma unroll 1
                for (int rd = 0; rd < kTcsSpan / kTcsRound; ++rd) {
                    unsigned v[kTcsRound / 32][32];
#pragma unroll
                    for (int w = 0; w < kTcsRound / 32; ++w) PC_TC_LD32(v[w], tbase + (unsigned)(kTcsRound * rd) + 32u * w);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (rd == kTcsSpan / kTcsRound - 1) {
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive_plain(acc_empty + 8 * k);
                    }
#ifdef PC_TCS_DBG_LIGHT  // debug (timing only): the drain without the arithmetic
#pragma unroll
                    for (int w = 0; w < kTcsRound / 32; ++w) acc.x += __uint_as_float(v[w][w]);
#else
                    fold(v);
#endif
                }
#endif
                acc = __fadd2_rn(acc, acc2);
                sum += (double)(acc.x + acc.y) * (double)kTcsS;
            }
            if (done) break;
        }
        if (cur >= 0) {
            const double cs = warp_sum(sum);
            PC_CHECK(cur < a.nclaims);
            if (lane == 0) a.claim_sums[cur * kTcsParts + ew] = cs;
        }
        sum = 0.0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        Slot sl{};
        sl.pad[0] = s_items;  // items (chunks) evaluated on the tensor cores
        a.slots[blockIdx.x] = sl;
    }
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}
