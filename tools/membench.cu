// membench.cu -- memory-pipeline microbenchmark for the streaming-kernel access pattern
// (warp strips of 128 columns x row segments, 4 loads + 1 store of 512 B per warp per step).
// Measures achieved HBM bandwidth vs per-step compute and prefetch strategy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu && ./membench
#include <cstdio>
#include <cuda_runtime.h>

constexpr int H = 4096, W = 4096, S = 61, SSTEP = 124, NSTRIP = 34, WPB = 8;

__device__ __forceinline__ float work(float a, int n) {
    float b = a, c = a * 0.5f, d = a + 1.f, e = a - 1.f;
    for (int i = 0; i < n; ++i) {
        b = fmaf(b, 0.999f, 0.001f); c = fmaf(c, 0.999f, 0.001f);
        d = fmaf(d, 0.999f, 0.001f); e = fmaf(e, 0.999f, 0.001f);
    }
    return b + c + d + e;
}

// depth-1 register prefetch (the current design)
template <int NW>
__global__ void __launch_bounds__(256, 2) k_reg(const float* x, const float* p, const float* y, const float* r,
                                                 float* o, int nseg) {
    int gw = blockIdx.x * WPB + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (gw >= NSTRIP * nseg) return;
    int strip = gw % NSTRIP, seg = gw / NSTRIP;
    int col = strip * SSTEP + 4 * lane;
    if (col + 3 >= W) col = W - 4;
    int r0 = seg * S;
    size_t off = (size_t)r0 * W + col;
    const float *qx = x + off, *qp = p + off, *qy = y + off, *qr = r + off;
    float* qo = o + off;
    float4 fx = *(const float4*)qx, fp = *(const float4*)qp, fy = *(const float4*)qy, fr = *(const float4*)qr;
    float acc = 0.f;
    int rows = min(S, H - r0 - 4);
    for (int t = 0; t < rows; ++t) {
        float v = fx.x + fx.y + fx.z + fx.w + fp.x + fp.y + fp.z + fp.w + fy.x + fy.y + fy.z + fy.w + fr.x + fr.y + fr.z + fr.w;
        qx += W; qp += W; qy += W; qr += W;
        fx = __ldg((const float4*)qx); fp = __ldg((const float4*)qp);
        fy = __ldg((const float4*)qy); fr = __ldg((const float4*)qr);
        acc += work(v, NW);
        *(float4*)qo = make_float4(acc, v, acc, v);
        qo += W;
    }
}

// cp.async.bulk (TMA 1D) into a per-warp shared-memory ring of NST stages, mbarrier completion
template <int NW, int NST>
__global__ void __launch_bounds__(256, 2) k_bulk(const float* x, const float* p, const float* y, const float* r,
                                                  float* o, int nseg) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* ring = reinterpret_cast<float*>(smem) + warp * NST * 4 * 128;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + WPB * NST * 4 * 128 * 4) + warp * NST;
    int gw = blockIdx.x * WPB + warp;
    bool live = gw < NSTRIP * nseg;
    int strip = live ? gw % NSTRIP : 0, seg = live ? gw / NSTRIP : 0;
    int col0 = strip * SSTEP;
    if (col0 + 128 > W) col0 = W - 128;
    int r0 = seg * S;
    int rows = live ? min(S, H - r0 - 4) : 0;
    const float* src[4] = {x, p, y, r};
    if (lane == 0)
        for (int s = 0; s < NST; ++s) {
            unsigned a = (unsigned)__cvta_generic_to_shared(&bars[s]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](int t) {
        int s = t % NST;
        unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4 * 512));
        for (int a = 0; a < 4; ++a) {
            const float* g = src[a] + (size_t)(r0 + t) * W + col0;
            unsigned dst = (unsigned)__cvta_generic_to_shared(ring + (s * 4 + a) * 128);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];"
                         ::"r"(dst), "l"(g), "r"(bar) : "memory");
        }
    };
    if (lane == 0)
        for (int t = 0; t < NST && t < rows; ++t) issue(t);
    float acc = 0.f;
    for (int t = 0; t < rows; ++t) {
        int s = t % NST;
        unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[s]);
        unsigned par = (t / NST) & 1;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"
                     ::"r"(bar), "r"(par) : "memory");
        float v = 0.f;
        for (int a = 0; a < 4; ++a) {
            float4 q = *reinterpret_cast<const float4*>(ring + (s * 4 + a) * 128 + 4 * lane);
            v += q.x + q.y + q.z + q.w;
        }
        acc += work(v, NW);
        __syncwarp();
        if (lane == 0 && t + NST < rows) issue(t + NST);
        *(float4*)(o + (size_t)(r0 + t) * W + col0 + 4 * lane) = make_float4(acc, v, acc, v);
    }
}

int main() {
    size_t n = (size_t)H * W;
    float *x, *p, *y, *r, *o, *fl;
    cudaMalloc(&x, n * 4); cudaMalloc(&p, n * 4); cudaMalloc(&y, n * 4); cudaMalloc(&r, n * 4);
    cudaMalloc(&o, n * 4); cudaMalloc(&fl, 512 << 20);
    cudaMemset(x, 0, n * 4); cudaMemset(p, 0, n * 4); cudaMemset(y, 0, n * 4); cudaMemset(r, 0, n * 4);
    int nseg = (H + S - 1) / S;
    int nblk = (NSTRIP * nseg + WPB - 1) / WPB;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    double bytes = 5.0 * n * 4;
    auto run = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaMemset(fl, it, 512 << 20);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (it > 0 && ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("%-28s %8.1f us  %7.0f GB/s  %s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(e));
    };
#define REG(NW) run("reg  work=" #NW, [&] { k_reg<NW><<<nblk, 256>>>(x, p, y, r, o, nseg); })
    REG(0); REG(16); REG(32); REG(64); REG(96);
#define BULK(NW, NST)                                                                                     \
    {                                                                                                     \
        size_t sm = WPB * NST * 4 * 128 * 4 + WPB * NST * 8;                                              \
        cudaFuncSetAttribute(k_bulk<NW, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);      \
        run("bulk work=" #NW " st=" #NST, [&] { k_bulk<NW, NST><<<nblk, 256, sm>>>(x, p, y, r, o, nseg); }); \
    }
    BULK(0, 2); BULK(0, 4); BULK(16, 4); BULK(32, 4); BULK(64, 4); BULK(96, 4); BULK(64, 6); BULK(96, 6);
    return 0;
}
