// l2dir.cu -- does alternating the row-streaming direction between SCG phases let a phase re-read
// the previous phase's most recent rows from L2?  Emulates the loop kernel's access pattern at C3
// size: one wave of 148 x 16 warps, each warp a 128-column strip x S-row segment, phases alternate
// update-like (read x,p,r,Y; write x',p') and value+gradient-like (read x',p',Y,r; write r').
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2dir l2dir.cu && ./l2dir
#include <cstdio>
#include <cuda_runtime.h>

constexpr int H = 4096, W = 4096, WPB = 16, SCOL = 128;
constexpr int NSTRIP = W / SCOL;   // 32 strips, no overlap in this emulation

template <int NIN, int NOUT>
__global__ void __launch_bounds__(WPB * 32, 1) k_phase(const float* __restrict__ i0, const float* __restrict__ i1,
                                                       const float* __restrict__ i2, const float* __restrict__ i3,
                                                       float* o0, float* o1, int S, int rev, float* sink) {
    const int gw = blockIdx.x * WPB + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    const int strip = gw % NSTRIP, seg = gw / NSTRIP;
    const int r0 = seg * S;
    if (r0 >= H) return;
    const int r1 = min(r0 + S, H);
    const int col = strip * SCOL + 4 * lane;
    float acc = 0.f;
    const int n = r1 - r0;
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
        const int row = rev ? r1 - 1 - k : r0 + k;
        const size_t o = (size_t)row * W + col;
        float4 a = __ldg((const float4*)(i0 + o));
        float4 b = __ldg((const float4*)(i1 + o));
        float4 c = __ldg((const float4*)(i2 + o));
        float4 d = __ldg((const float4*)(i3 + o));
        float4 v = make_float4(a.x + b.x * 0.5f, a.y + b.y * 0.5f, a.z + c.z, a.w + d.w);
        acc += v.x + v.y + c.x + d.y;
        *(float4*)(o0 + o) = v;
        if (NOUT > 1) *(float4*)(o1 + o) = make_float4(b.x + c.y, b.y, b.z, b.w + d.x);
    }
    if (acc == 12345.f) *sink = acc;
}

// same pattern through cp.async.bulk (the loop kernel's loads): per-warp 3-stage shared-memory ring
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int NOUT>
__global__ void __launch_bounds__(WPB * 32, 1) k_bulk(const float* __restrict__ i0, const float* __restrict__ i1,
                                                      const float* __restrict__ i2, const float* __restrict__ i3,
                                                      float* o0, float* o1, int S, int rev, float* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = __shfl_sync(~0u, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int gw = blockIdx.x * WPB + warp;
    const int strip = gw % NSTRIP, seg = gw / NSTRIP;
    const int r0 = seg * S;
    if (r0 >= H) return;
    const int r1 = min(r0 + S, H);
    const int n = r1 - r0;
    float* ring = reinterpret_cast<float*>(sm + warp * (3 * 4 * 512 + 64));
    const unsigned bars = su32(ring + 3 * 4 * 128);
    if (lane == 0) {
        for (int s = 0; s < 3; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int c0 = strip * SCOL;
    auto issue = [&](int s, int k) {
        const int row = rev ? r1 - 1 - k : r0 + k;
        const size_t o = (size_t)row * W + c0;
        const unsigned d = su32(ring + s * 512), bar = bars + 8 * s;
        asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
            "@P mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 2048;\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%2], 512, [%0];\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%3], [%4], 512, [%0];\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%5], [%6], 512, [%0];\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%7], [%8], 512, [%0];\n\t}"
            ::"r"(bar), "r"(d), "l"(i0 + o), "r"(d + 512), "l"(i1 + o), "r"(d + 1024), "l"(i2 + o), "r"(d + 1536), "l"(i3 + o)
            : "memory");
    };
    for (int k = 0; k < 3 && k < n; ++k) issue(k, k);
    float acc = 0.f;
    unsigned par = 0;
    for (int k = 0; k < n; ++k) {
        const int s = k % 3;
        unsigned ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(bars + 8 * s), "r"(par) : "memory");
        if (s == 2) par ^= 1;
        const float4 a = reinterpret_cast<const float4*>(ring + s * 512)[lane];
        const float4 b = reinterpret_cast<const float4*>(ring + s * 512 + 128)[lane];
        const float4 c = reinterpret_cast<const float4*>(ring + s * 512 + 256)[lane];
        const float4 d = reinterpret_cast<const float4*>(ring + s * 512 + 384)[lane];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (k + 3 < n) issue(s, k + 3);
        const int row = rev ? r1 - 1 - k : r0 + k;
        const size_t o = (size_t)row * W + c0 + 4 * lane;
        float4 v = make_float4(a.x + b.x * 0.5f, a.y + b.y * 0.5f, a.z + c.z, a.w + d.w);
        acc += v.x + v.y + c.x + d.y;
        *(float4*)(o0 + o) = v;
        if (NOUT > 1) *(float4*)(o1 + o) = make_float4(b.x + c.y, b.y, b.z, b.w + d.x);
    }
    if (acc == 12345.f) *sink = acc;
}

int main() {
    const size_t N = (size_t)H * W;
    float* buf;
    cudaMalloc(&buf, 8 * N * sizeof(float));
    float *x[2], *p[2], *r[2], *Y = buf + 6 * N, *sink = buf + 7 * N;
    for (int k = 0; k < 2; ++k) { x[k] = buf + k * N; p[k] = buf + (2 + k) * N; r[k] = buf + (4 + k) * N; }
    cudaMemset(buf, 0, 8 * N * sizeof(float));
    float* flush;
    cudaMalloc(&flush, 512u << 20);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nwarps = sms * WPB;
    const int nseg = nwarps / NSTRIP;
    const int S = (H + nseg - 1) / nseg;
    const int grid = (NSTRIP * ((H + S - 1) / S) + WPB - 1) / WPB;
    printf("SMs %d, warps %d, segments %d x %d rows, grid %d\n", sms, nwarps, nseg, S, grid);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int smem = WPB * (3 * 4 * 512 + 64);
    cudaFuncSetAttribute(k_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_bulk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int bulk = 0; bulk < 2; ++bulk)
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(flush, rep, 512u << 20);
            cudaEventRecord(e0);
            int xc = 0, rc = 0;
            for (int ph = 0; ph < 40; ++ph) {
                const int rev = mode == 0 ? 0 : (mode == 1 ? (ph & 1) : 1);
                if ((ph & 1) == 0) {   // update: x,p,r,Y -> x',p'
                    if (bulk) k_bulk<2><<<grid, WPB * 32, smem>>>(x[xc], p[xc], r[rc], Y, x[xc ^ 1], p[xc ^ 1], S, rev, sink);
                    else k_phase<4, 2><<<grid, WPB * 32>>>(x[xc], p[xc], r[rc], Y, x[xc ^ 1], p[xc ^ 1], S, rev, sink);
                    xc ^= 1;
                } else {               // value+gradient: x',p',Y,r -> r'
                    if (bulk) k_bulk<1><<<grid, WPB * 32, smem>>>(x[xc], p[xc], Y, r[rc], r[rc ^ 1], nullptr, S, rev, sink);
                    else k_phase<4, 1><<<grid, WPB * 32>>>(x[xc], p[xc], Y, r[rc], r[rc ^ 1], nullptr, S, rev, sink);
                    rc ^= 1;
                }
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = 20.0 * (4 * 4 + 4 * 2) * N + 20.0 * (4 * 4 + 4) * N;
            printf("%s mode %s rep %d: %.3f ms, %.1f us/phase, algorithmic %.0f GB/s\n",
                   bulk ? "bulk" : "ldg ", mode == 0 ? "down    " : (mode == 1 ? "alternate" : "up      "), rep, ms, ms * 1e3 / 40,
                   bytes / (ms * 1e-3) / 1e9);
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
