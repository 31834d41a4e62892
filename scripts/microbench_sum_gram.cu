// Would a Gram-form d^2 pay for the inverse-square SUM?  Same harness for both loops:
// R = 8 rows per lane in registers, W = 256 columns per pass from shared memory
// (pair layout as the library stages it), 4 CTAs x 4 warps per SM.
//   DIRECT: p = 1 + (x_i-x_j)^2 + (y_i-y_j)^2 + (z_i-z_j)^2   3 FADD2 + 3 FFMA2 per 2 pairs
//   GRAM:   p = A_i + (B_j - 2 a_i.b_j), A_i = 1 + |a_i|^2     3 FFMA2 + 1 FADD2 per 2 pairs
//   DIRECT-ASM: DIRECT with the library's inline-asm broadcast subtract (f2_rsub)
//   DIRECT+EPI: DIRECT-ASM plus the library's per-chunk epilogue (fp64 row sums, flags)
// and for both: 1/pa + 1/pc = (pa + pc) * rcp(pa * pc)       FMUL2 + FADD2 + 2 MUFU + FFMA2 per 4 pairs
// Prints Tpair/s (the library's sum kernel: 4.41 at N = 2^20).  (The Gram form needs local origins to be accurate; this measures
// only the instruction cost.)
//
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mbsg scripts/microbench_sum_gram.cu && ./mbsg
#include <cuda_runtime.h>

#include <cstdio>

constexpr int W = 256, R = 8;

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 f2_rsub(float a, float2 b) {  // the library's a - b, a broadcast (inline asm)
    unsigned long long bb = *reinterpret_cast<unsigned long long*>(&b), dd;
    asm("{.reg .b64 t; mov.b64 t, {%1, %1}; sub.rn.f32x2 %0, t, %2;}" : "=l"(dd) : "f"(a), "l"(bb));
    return *reinterpret_cast<float2*>(&dd);
}

template <int GRAM>
__global__ void __launch_bounds__(128, 4) k(const float4* __restrict__ cols, float* out, int reps,
                                            long long* cyc) {
    const long long c0 = clock64();
    __shared__ float4 s[W];  // W/2 column pairs x 2 float4: (x, x1, y, y1)(z, z1, w, w1)
    for (int q = threadIdx.x; q < W; q += blockDim.x) s[q] = cols[q];
    __syncthreads();
    float rx[R], ry[R], rz[R], ra[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {  // runtime row values (constants would fold into immediates)
        const float4 rv = cols[(threadIdx.x * R + r) % W];
        rx[r] = rv.x + 0.01f * r;
        ry[r] = rv.y - 0.02f * r;
        rz[r] = rv.z + 0.03f * threadIdx.x;
        ra[r] = 1.0f + rx[r] * rx[r] + ry[r] * ry[r] + rz[r] * rz[r];
        if (GRAM == 1) {
            rx[r] *= -2.f;
            ry[r] *= -2.f;
            rz[r] *= -2.f;
        }
    }
    float2 acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = make_float2(0.f, 0.f);
    double dsum = 0.0;
    unsigned flags = 0;
    for (int it = 0; it < reps; ++it) {
#pragma unroll 2
        for (int k2 = 0; k2 < W; k2 += 4) {  // two column pairs per step
            const float4 A0 = s[k2], B0 = s[k2 + 1], A1 = s[k2 + 2], B1 = s[k2 + 3];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                float2 pa, pc;
                if (GRAM == 1) {
                    pa = __ffma2_rn(f2(rz[r]), make_float2(B0.x, B0.y),
                                    __ffma2_rn(f2(ry[r]), make_float2(A0.z, A0.w),
                                               __ffma2_rn(f2(rx[r]), make_float2(A0.x, A0.y), make_float2(B0.z, B0.w))));
                    pc = __ffma2_rn(f2(rz[r]), make_float2(B1.x, B1.y),
                                    __ffma2_rn(f2(ry[r]), make_float2(A1.z, A1.w),
                                               __ffma2_rn(f2(rx[r]), make_float2(A1.x, A1.y), make_float2(B1.z, B1.w))));
                    pa = __fadd2_rn(pa, f2(ra[r]));
                    pc = __fadd2_rn(pc, f2(ra[r]));
                } else if (GRAM == 2 || GRAM == 3) {
                    float2 dx = f2_rsub(rx[r], make_float2(A0.x, A0.y));
                    float2 dy = f2_rsub(ry[r], make_float2(A0.z, A0.w));
                    float2 dz = f2_rsub(rz[r], make_float2(B0.x, B0.y));
                    pa = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, f2(1.f))));
                    dx = f2_rsub(rx[r], make_float2(A1.x, A1.y));
                    dy = f2_rsub(ry[r], make_float2(A1.z, A1.w));
                    dz = f2_rsub(rz[r], make_float2(B1.x, B1.y));
                    pc = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, f2(1.f))));
                } else {
                    const float2 dxa = __fadd2_rn(f2(rx[r]), make_float2(-A0.x, -A0.y));
                    const float2 dya = __fadd2_rn(f2(ry[r]), make_float2(-A0.z, -A0.w));
                    const float2 dza = __fadd2_rn(f2(rz[r]), make_float2(-B0.x, -B0.y));
                    const float2 dxc = __fadd2_rn(f2(rx[r]), make_float2(-A1.x, -A1.y));
                    const float2 dyc = __fadd2_rn(f2(ry[r]), make_float2(-A1.z, -A1.w));
                    const float2 dzc = __fadd2_rn(f2(rz[r]), make_float2(-B1.x, -B1.y));
                    pa = __ffma2_rn(dza, dza, __ffma2_rn(dya, dya, __ffma2_rn(dxa, dxa, f2(1.f))));
                    pc = __ffma2_rn(dzc, dzc, __ffma2_rn(dyc, dyc, __ffma2_rn(dxc, dxc, f2(1.f))));
                }
                const float2 pr = __fmul2_rn(pa, pc), sm = __fadd2_rn(pa, pc);
                acc[r] = __ffma2_rn(sm, make_float2(rcp_approx(pr.x), rcp_approx(pr.y)), acc[r]);
            }
        }
        if (GRAM == 3) {  // the library's per-chunk epilogue: fp64 row sums + conservative contact flags
            unsigned fl = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float cs = acc[r].x + acc[r].y;
                dsum += (double)cs;
                fl |= (cs > 0.4999f ? 1u : 0u) << r;
                acc[r] = make_float2(0.f, 0.f);
            }
            if (__any_sync(0xffffffffu, fl != 0)) flags |= fl;
        }
    }
    if (GRAM == 3) acc[0].x += (float)dsum + (float)flags;
    float t = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) t += acc[r].x + acc[r].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = clock64() - c0;
}

template <int GRAM>
void run(const float4* d, float* o, int sms, long long* cyc) {
    const int grid = sms * 4, reps = 2000;
    k<GRAM><<<grid, 128>>>(d, o, 10, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<GRAM><<<grid, 128>>>(d, o, reps, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * 128 * R * W * reps;
    printf("%s: %.3f ms, %.3f Tpair/s\n", GRAM == 1 ? "gram      " : GRAM == 2 ? "direct-asm" : GRAM == 3 ? "direct+epi" : "direct    ", ms,
           pairs / (ms * 1e-3) / 1e12);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float4 h[W];
    for (int q = 0; q < W; ++q) h[q] = make_float4(0.1f * q, 0.2f, 0.3f * (q & 7), 1.5f + q);
    float4* d;
    float* o;
    long long* cyc;
    cudaMalloc(&cyc, 8);
    cudaMalloc(&d, sizeof h);
    cudaMalloc(&o, sms * 4 * 128 * 4);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
        run<0>(d, o, sms, cyc);
        run<1>(d, o, sms, cyc);
        run<2>(d, o, sms, cyc);
        run<3>(d, o, sms, cyc);
    }
    return 0;
}
