// flmisr_stream_common.cuh -- device building blocks shared by the register-streaming kernels
// (flmisr_stream.cu: common separable kappa; flmisr_stream4.cu: per-phase 4x4 kappa): packed fp32x2
// arithmetic, the per-warp bulk-copy ring, warp work-item geometry, border helpers, programmatic
// dependent launch and the persistent loop's grid barrier with its fixed-order fp64 sum.
// Each including translation unit gets its own copies (anonymous namespace).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "flmisr_common.cuh"
#include "flmisr_internal.h"

namespace flmisr {
namespace {

// Host: opt a kernel in to smem bytes of dynamic shared memory once per (kernel, device).  Thread-safe:
// plans may be created and launched from several host threads.
inline cudaError_t ensure_dyn_smem(const void* kernel, size_t smem) { return raise_dyn_smem(kernel, smem); }

// ---- packed fp32x2 helpers (PTX f32x2 -> SASS FFMA2 / FADD2 / FMUL2 on sm_100a) ----
__device__ __forceinline__ float2 F2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}\n"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}\n"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}\n"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}\n"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 fma2s(float s, float2 b, float2 c) { return fma2(F2(s, s), b, c); }
__device__ __forceinline__ float2 mul2s(float s, float2 b) { return mul2(F2(s, s), b); }
__device__ __forceinline__ float2 rsq2(float2 q) { return F2(rsq(q.x), rsq(q.y)); }
__device__ __forceinline__ float2 lo2(const float4& v) { return F2(v.x, v.y); }   // (c0, c2)
__device__ __forceinline__ float2 hi2(const float4& v) { return F2(v.z, v.w); }   // (c1, c3)

// ---- per-warp TMA ring: cp.async.bulk (1D bulk copy engine) row segments -> shared memory ----
constexpr int NARR = 4;           // rows per stage (4 arrays)
// ring data + mbarriers of NS stages, rounded to 128 B so every warp's ring (bulk-copy destination,
// 16-byte shared-memory vector reads) stays aligned
template <int NS, int WPB = SWPB>
struct RingDims {
    static constexpr int FLOATS = NS * NARR * SCOLS;
    static constexpr size_t BYTES_PER_WARP = ((size_t)FLOATS * 4 + NS * 8 + 127) / 128 * 128;
    static constexpr size_t SMEM = WPB * BYTES_PER_WARP;
};
constexpr int NST = 3;            // stages per warp of the common-kappa kernels (== their row-loop unroll)
constexpr size_t RING_SMEM = RingDims<NST>::SMEM;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}

template <int NS>
struct RingT {
    static constexpr int RING_FLOATS = RingDims<NS>::FLOATS;
    static constexpr size_t RING_BYTES_PER_WARP = RingDims<NS>::BYTES_PER_WARP;
    const float* ptr;   // this warp's ring (generic pointer into shared memory)
    uint32_t data;      // shared address of this warp's ring
    uint32_t bars;      // shared address of its NST mbarriers
    __device__ __forceinline__ void init(unsigned char* smem, int warp, int lane) {
        unsigned char* base = smem + (size_t)warp * RING_BYTES_PER_WARP;
        ptr = reinterpret_cast<const float*>(base);
        data = smem_u32(base);
        bars = smem_u32(base + (size_t)RING_FLOATS * 4);
        if (lane == 0) {
            for (int s = 0; s < NS; ++s) mbar_init(bars + 8 * s);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    // whole (converged) warp: one elected lane arms stage s and issues its four 512-byte row copies;
    // the addresses are warp-uniform, so no per-lane branch or register-to-uniform waterfall
    __device__ __forceinline__ void issue(int s, const float* a0, const float* a1, const float* a2,
                                          const float* a3) const {
        const uint32_t bar = bars + 8 * s;
        const uint32_t d = data + (uint32_t)(s * NARR * SCOLS * 4);
        asm volatile(
            "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\t"
            "@P mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], 512, [%0];\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%4], [%5], 512, [%0];\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%6], [%7], 512, [%0];\n\t"
            "@P cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%8], [%9], 512, [%0];\n\t}"
            ::"r"(bar), "r"(NARR * SCOLS * 4), "r"(d), "l"(a0), "r"(d + SCOLS * 4), "l"(a1), "r"(d + 2 * SCOLS * 4),
              "l"(a2), "r"(d + 3 * SCOLS * 4), "l"(a3)
            : "memory");
    }
    __device__ __forceinline__ void wait(int s, uint32_t parity) const {
        while (!mbar_try(bars + 8 * s, parity)) {
        }
    }
    __device__ __forceinline__ float4 get(int s, int a, int lane) const {
        return *reinterpret_cast<const float4*>(ptr + (s * NARR + a) * SCOLS + 4 * lane);
    }
    // all lanes: the stage's rows are consumed; order the generic-proxy reads before the async
    // proxy refills the stage
    __device__ __forceinline__ void release() const {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
    }
};
using Ring = RingT<NST>;

// FLMISR_BOUNDS builds (memory-safety check without compute-sanitizer): every row the streaming
// kernels stage or load directly and every row segment they store must lie inside the plan's HR
// allocation; a violation traps (the kernel fails loudly instead of touching foreign memory)
#ifdef FLMISR_BOUNDS
__device__ __forceinline__ void bchk(const Buffers& b, const float* p, int nfloats) {
    if (p < b.mem_lo || p + nfloats > b.mem_hi) __trap();
}
#define FL_BCHK(b, p, n) bchk((b), (p), (n))
#else
#define FL_BCHK(b, p, n) ((void)0)
#endif

__device__ __forceinline__ const float* rowp(const float* base, const StencilParams& sp, int row) {
    int r = min(max(row, sp.store_lo), sp.store_hi - 1);
    return base + (size_t)(r - sp.store_lo) * sp.pitch;
}

// r rows for the update kernel: rows outside the owned band come from the received halo buffers
// (inner-outer border exchange) when this rank has a neighbour on that side.
__device__ __forceinline__ const float* rrowp(const Buffers& b, const float* R, const StencilParams& sp, int row) {
    if (row < sp.row_lo && b.halo_top) {
        int k = min(max(row - (sp.row_lo - b.eta), 0), b.eta - 1);
        return b.halo_top + (size_t)k * sp.pitch;
    }
    if (row >= sp.row_hi && b.halo_bot) {
        int k = min(max(row - sp.row_hi, 0), b.eta - 1);
        return b.halo_bot + (size_t)k * sp.pitch;
    }
    return rowp(R, sp, row);
}

// Direct (non-ring) loads of the two warm-up rows of a segment.  Plain coherent loads, not
// ld.global.nc: in the persistent loop kernels these rows were written earlier in the SAME launch by
// other CTAs (x/p of the neighbouring segment) or by peer GPUs (r halo rows), and the non-coherent
// path is only defined for data that is read-only for the whole kernel.  The grid barrier's acquire
// orders them (PTX memory model: weak loads after an acquire observe the released stores).
template <bool BORDER>
__device__ __forceinline__ float4 ld4(const float* rp, int col, int W) {
    if (!BORDER || col + 3 < W) return *reinterpret_cast<const float4*>(rp + col);
    // right image border (W % 4 == 0): a group is either inside or wholly outside -> replicate col W-1
    // (column W-1 is the c3 slot of the last group, at the same physical place)
    float v = rp[W - 1];
    return make_float4(v, v, v, v);
}

// store a lane's 4 columns given as the pairs A = (c0, c2), B = (c1, c3) in the permuted layout;
// partial lanes (strip overlap) write only the output half (.x: c0,c1 / .y: c2,c3)
__device__ __forceinline__ void stp(float* rp, float2 A, float2 B, bool olo, bool ohi) {
    if (olo && ohi) {
        *reinterpret_cast<float4*>(rp) = make_float4(A.x, A.y, B.x, B.y);
    } else {
        if (olo) { rp[0] = A.x; rp[2] = B.x; }
        if (ohi) { rp[1] = A.y; rp[3] = B.y; }
    }
}

struct Geo {
    int lane, cbase, col0, r_lo, r_hi, w_lo, w_hi, llast;
    bool strip0, live, border, rstrip;
    bool olo, ohi;   // columns (c0, c1) / (c2, c3) of this lane are output columns of the strip
    bool cv0, cv4;   // the lane's group / the right neighbour group lies inside the image
};

// cta: this CTA's index among the CTAs that share the band's work items (blockIdx.x, or the CTA's
// index within its band in the peer loop)
// HALO: columns of overlap per strip side (the operator's column reach): SHALO = 2 for the common-kappa
// kernels, 4 for the per-phase 4x4 kernels; strips step by SCOLS - 2 HALO
// gw: the work item (warp-uniform); geometry() below takes the item of this warp of CTA cta.  DET: the
// det-mode layout (sp.det; a template flag so the default kernels carry none of its code)
template <int HALO = SHALO, bool DET = false>
__device__ __forceinline__ Geo geometry_item(const StencilParams& sp, int gw) {
    constexpr int STEP = SCOLS - 2 * HALO;
    Geo g;
    g.lane = threadIdx.x & 31;
    g.live = gw < sp.nitems;
    // work item -> (strip, rows [r_lo, r_hi)); see StencilParams: border pieces (band edges, edge
    // strips) are seg_b rows, interior pieces seg_rows rows
    int strip = 0, seg = 0, nseg = 1;
    g.r_lo = g.r_hi = sp.row_lo;
    if (DET && g.live) {
        // det mode: the same layout in units of the fixed tiles of T rows (from row_lo, a multiple of T; the
        // band's last tile is short when it ends at an image height H % T != 0), so every segment is a
        // union of whole tiles whatever its length
        const int T = sp.det_rows, nt = (sp.row_hi - sp.row_lo + T - 1) / T;
        const int m = sp.seg_rows / T, mb = sp.seg_b / T;
        int tlo, thi;
        if (gw < sp.n_int) {
            strip = 1 + gw % sp.ni;
            seg = gw / sp.ni;
            nseg = sp.nseg_i;
            if (seg == 0) { tlo = 0; thi = min(mb, nt); }
            else if (seg == nseg - 1) { tlo = max(nt - mb, mb); thi = nt; }
            else { tlo = mb + (seg - 1) * m; thi = min(tlo + m, nt - mb); }
        } else {
            const int e = gw - sp.n_int;
            strip = (sp.ne == 1 || (e & 1) == 0) ? 0 : sp.nstrips - 1;
            seg = e / sp.ne;
            nseg = sp.nseg_b;
            tlo = seg * mb;
            thi = min(tlo + mb, nt);
        }
        g.r_lo = min(sp.row_lo + tlo * T, sp.row_hi);
        g.r_hi = min(sp.row_lo + thi * T, sp.row_hi);
    } else if (g.live && gw < sp.n_int) {     // interior strip 1 .. ni: seg_b | seg_rows ... | seg_b
        strip = 1 + gw % sp.ni;
        seg = gw / sp.ni;
        nseg = sp.nseg_i;
        if (seg == 0) {
            g.r_hi = min(sp.row_lo + sp.seg_b, sp.row_hi);
        } else if (seg == nseg - 1) {
            g.r_lo = max(sp.row_hi - sp.seg_b, sp.row_lo + sp.seg_b);
            g.r_hi = sp.row_hi;
        } else {
            g.r_lo = sp.row_lo + sp.seg_b + (seg - 1) * sp.seg_rows;
            g.r_hi = min(g.r_lo + sp.seg_rows, sp.row_hi - sp.seg_b);
        }
    } else if (g.live) {                      // edge strip 0 / nstrips-1: seg_b rows each
        const int e = gw - sp.n_int;
        strip = (sp.ne == 1 || (e & 1) == 0) ? 0 : sp.nstrips - 1;
        seg = e / sp.ne;
        nseg = sp.nseg_b;
        g.r_lo = sp.row_lo + seg * sp.seg_b;
        g.r_hi = min(g.r_lo + sp.seg_b, sp.row_hi);
    }
    g.cbase = strip * STEP;
    g.col0 = g.cbase + 4 * g.lane;
    g.strip0 = strip == 0;
    const int oc_lo = g.strip0 ? 0 : g.cbase + HALO;
    const int oc_hi = (strip == sp.nstrips - 1) ? sp.W : min(g.cbase + SCOLS - HALO, sp.W);
    // strip bounds are at even offsets and W % 4 == 0, so (c0, c1) and (c2, c3) share their masks
    g.olo = g.live && g.col0 >= oc_lo && g.col0 + 1 < oc_hi;
    g.ohi = g.live && g.col0 + 2 >= oc_lo && g.col0 + 3 < oc_hi;
    g.cv0 = g.col0 < sp.W;
    g.cv4 = g.col0 + 4 < sp.W;
    g.rstrip = g.cbase + SCOLS > sp.W;
    g.llast = min(max((sp.W - 1 - g.cbase) >> 2, 0), 31);
    if (!g.live) g.r_hi = g.r_lo;
    // rows whose new x/p this segment writes: owned rows, plus the band's halo rows for the first /
    // last segment of a band with a neighbour on that side (bit-identical to the neighbour's owned
    // rows: same inputs, same fp32 operations)
    g.w_lo = g.r_lo;
    g.w_hi = g.r_hi;
    if (g.live && seg == 0 && sp.row_lo > 0) g.w_lo = sp.store_lo;
    if (g.live && seg == nseg - 1 && sp.row_hi < sp.H) g.w_hi = sp.store_hi;
    // interior warps: no image border, every row they touch (r_lo - 2 .. r_hi + 2) is an owned row of
    // the band, so they need no clamps, no halo buffers and no masks beyond the strip's output columns
    g.border = g.strip0 || g.rstrip || g.r_lo < sp.row_lo + 3 || g.r_hi > sp.row_hi - 3;
#ifdef FLMISR_ALL_BORDER   // tuning build: every warp takes the border instantiation
    g.border = true;
#endif
    return g;
}

template <int HALO = SHALO, int WPB = SWPB>
__device__ __forceinline__ Geo geometry(const StencilParams& sp, int cta) {
    // warp index through a lane-0 shuffle so the compiler sees it (and every row pointer and the
    // ring addresses derived from it) as warp-uniform: the bulk copies then take uniform-register
    // operands directly instead of a per-copy R2UR waterfall
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    return geometry_item<HALO>(sp, cta * WPB + warp);
}

// ---- det mode: exact sums in 128-bit fixed point (value = s 2^-64) ----
// Integer addition is associative, so a sum of fixed-point values does not depend on the order or the
// grouping of its terms: the per-tile fp64 values (bit-identical at every band count, same rows, same
// arithmetic) give the same total whether they are summed per CTA, per band or over all bands.  The
// conversion of a tile value truncates below 2^-64 (deterministic); |value| < 2^63 (the sums here are
// <= ~1e12); a non-finite tile value is counted instead (the total becomes NaN -> FLMISR_ERR_NUMERIC).
// m 2^(sh - 64) as a two's-complement 128-bit integer (truncated below 2^-64), without branches: the
// lanes of a warp convert different exponents, and a data-dependent branch here would diverge
// (mbits: the mantissa width; sh is clamped so that |value| < 2^62 -- saturation, never reached by the
// sums here, which stay below ~1e12)
template <int MBITS>
__device__ __forceinline__ __int128 fx_shift(unsigned long long m, int sh, bool neg) {
    sh = max(min(sh, 126 - MBITS), -127);
    const int r = -sh;                                        // right shift for sh < 0
    const unsigned long long lo_pos = sh < 64 ? m << (sh & 63) : 0ull;
    const unsigned long long hi_pos = sh == 0 ? 0ull : (sh < 64 ? m >> ((64 - sh) & 63) : m << ((sh - 64) & 63));
    const unsigned long long lo_neg = r < 64 ? m >> (r & 63) : 0ull;
    unsigned long long lo = sh >= 0 ? lo_pos : lo_neg, hi = sh >= 0 ? hi_pos : 0ull;
    const unsigned long long nlo = ~lo + 1ull, nhi = ~hi + (lo == 0ull ? 1ull : 0ull);
    lo = neg ? nlo : lo;
    hi = neg ? nhi : hi;
    return (__int128)(((unsigned __int128)hi << 64) | lo);
}
__device__ __forceinline__ __int128 fx_of(double v) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const int ex = (int)((bits >> 52) & 0x7ff);
    const unsigned long long m = ex ? ((bits & 0xFFFFFFFFFFFFFull) | (1ull << 52)) : 0ull;   // zero / subnormal: 0
    return fx_shift<53>(m, ex - 1075 + 64, (bits >> 63) != 0);   // v = m 2^(ex - 1075)
}
__device__ __forceinline__ __int128 fx_of(float v) {
    const unsigned bits = __float_as_uint(v);
    const int ex = (int)((bits >> 23) & 0xff);
    const unsigned long long m = ex ? ((bits & 0x7fffffu) | 0x800000u) : 0ull;
    return fx_shift<24>(m, ex - 150 + 64, (bits >> 31) != 0);     // v = m 2^(ex - 150)
}
__device__ __forceinline__ __int128 fx_shfl_xor(__int128 v, int o) {
    const long long hi = __shfl_xor_sync(0xffffffffu, (long long)(v >> 64), o);
    const unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, o);
    return (__int128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}
__device__ __forceinline__ __int128 fx_warp_sum(__int128 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += fx_shfl_xor(v, o);
    return v;
}
__device__ __forceinline__ __int128 ld_relaxed_fx(const __int128* p) {
    unsigned long long lo, hi;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
    return (__int128)(((unsigned __int128)hi << 64) | lo);
}

// per-lane exact accumulators of one phase (dynamic shared memory after the ring, det kernels only):
// every lane adds its own tile partials -- no cross-lane dependency at a tile boundary, so the warps of
// an SM, which reach their tile boundaries together, do not stall on shuffle trees there; the lanes
// are reduced once per phase (fx_cta_reduce)
template <int WPB>
struct FxCta {
    __int128 s[WPB][FXW][32];
    __int128 red[WPB][FXW];
};
constexpr size_t FX_SMEM = sizeof(FxCta<SWPB>);
// every lane: this lane's tile partial of slot k, exactly (a non-finite value is counted instead)
template <int WPB, typename V>
__device__ __forceinline__ void fx_lane_add(FxCta<WPB>& fc, int k, V v) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool ok = isfinite(v);
    fc.s[warp][k][lane] += ok ? fx_of(v) : (__int128)0;
    if (!ok) fc.s[warp][NSLOT][lane] += 1;
}
// all threads: zero the accumulators (before a phase; a __syncthreads must separate it from any use)
template <int WPB>
__device__ __forceinline__ void fx_zero(FxCta<WPB>& fc) {
    for (int i = threadIdx.x; i < WPB * FXW * 32; i += blockDim.x) (&fc.s[0][0][0])[i] = 0;
}
// all threads, after a __syncthreads: each warp's lanes -> red[warp][k] (exact)
template <int WPB>
__device__ __forceinline__ void fx_cta_reduce(FxCta<WPB>& fc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < FXW; ++k) {
        const __int128 v = fx_warp_sum(fc.s[warp][k][lane]);
        if (lane == 0) fc.red[warp][k] = v;
    }
}
// after fx_cta_reduce and a __syncthreads: this CTA's exact sum k
template <int WPB>
__device__ __forceinline__ __int128 fx_cta(const FxCta<WPB>& fc, int k) {
    __int128 t = 0;
    for (int w = 0; w < WPB; ++w) t += fc.red[w][k];
    return t;
}
// all threads: exact sum of n slots of FXW words at slot[i * FXW + k] -> t (128-bit totals)
__device__ __forceinline__ void fx_sum_raw(const __int128* slot, int n, __int128 (&t)[FXW]) {
    __shared__ __int128 sred[32][FXW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __int128 loc[FXW];
#pragma unroll
    for (int k = 0; k < FXW; ++k) loc[k] = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
#pragma unroll
        for (int k = 0; k < FXW; ++k) loc[k] += ld_relaxed_fx(slot + (size_t)i * FXW + k);
#pragma unroll
    for (int k = 0; k < FXW; ++k) {
        const __int128 v = fx_warp_sum(loc[k]);
        if (lane == 0) sred[warp][k] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < FXW; ++k) {
        t[k] = 0;
        for (int w = 0; w < nw; ++w) t[k] += sred[w][k];
    }
    __syncthreads();   // sred is reused by the next call
}
// ... converted (scaled and offset by the caller); the count of non-finite tile values makes every
// total NaN
__device__ __forceinline__ void fx_sum_slots(const __int128* slot, int n, double (&tot)[NSLOT]) {
    __int128 t[FXW];
    fx_sum_raw(slot, n, t);
    const bool bad = t[NSLOT] != 0;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) tot[k] = bad ? __longlong_as_double(0x7ff8000000000000ll) : fx_to_double(t[k]);
}

__device__ __forceinline__ float shup(float v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ float shdn(float v) { return __shfl_down_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ float msum(float2 a, const Geo& g) { return (g.olo ? a.x : 0.f) + (g.ohi ? a.y : 0.f); }

// right-border strip: lanes past the image take the replicated column W-1 (clamp, reading 4)
template <bool BORDER>
__device__ __forceinline__ float4 fixr(float4 v, const Geo& g) {
    if (BORDER && g.rstrip) {
        const float r = __shfl_sync(0xffffffffu, v.w, g.llast);
        if (!g.cv0) v = make_float4(r, r, r, r);
    }
    return v;
}

// Programmatic dependent launch: the streaming kernels are launched with programmatic stream
// serialization, so the next kernel's CTAs may be scheduled onto SMs this grid has already left;
// every kernel waits for its predecessor's completion (and memory flush) before touching any data.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

#ifdef FLMISR_TIMING
// diagnostic build only: per (phase, CTA): CTA work end, arrival, release, scalars done (globaltimer ns)
__device__ unsigned long long g_loop_time[64 * 256 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define FL_TMARK(ep, k) \
    if (threadIdx.x == 0 && (ep) < 64 && blockIdx.x < 256) g_loop_time[((ep) * 256 + blockIdx.x) * 4 + (k)] = gtimer();
#else
#define FL_TMARK(ep, k)
#endif

__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// grid_sum_fx: grid-wide sum of acc over all threads of all CTAs; result in tot (all threads).  Each CTA's fp64
// partial (fixed shuffle tree + fixed cross-warp order) is converted to 192-bit fixed point (value =
// X 2^-128: |value| < 2^63, truncation below 2^-128 ~ 3e-39, so the sums keep full fp64 precision from
// the first pass down to a converged <r,r>) and added as six 32-bit chunks with red.add.u64 into one
// of three accumulator sets (by epoch mod 3): integer adds commute, so the total does not depend on
// the order of the CTAs' arrivals, and after the barrier every CTA reads 25 words instead of summing
// all G slots (the per-phase tail after the last arrival: one L2 round trip).  Set (e + 2) mod 3 is
// zeroed by CTA 0 right after barrier e -- it was last read before barrier e and is next written after
// barrier e + 1, which CTA 0 releases after the zeroing; sets 0 and 1 are zeroed by k_state_init.
constexpr int FXCH = 6, FXA = NSLOT * FXCH + 1;   // chunks per sum; words per set (+ non-finite count)
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// 32-bit chunk c of the 192-bit two's-complement fixed-point image of a finite v (chunks from c = 0)
__device__ __forceinline__ void fx192_chunks(double v, unsigned (&ch)[FXCH]) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const int ex = (int)((bits >> 52) & 0x7ff);
    const unsigned long long m = ex ? ((bits & 0xFFFFFFFFFFFFFull) | (1ull << 52)) : 0ull;
    const int sh = min(ex - 1075 + 128, 191 - 53 - 1);   // X = m << sh (sh < 0: m >> -sh)
#pragma unroll
    for (int c = 0; c < FXCH; ++c) {
        const int d = 32 * c - sh;   // chunk c holds bits [32c, 32c + 32) of X = bits [d, d + 32) of m
        unsigned long long x;
        if (d >= 0) x = d < 64 ? (m >> d) : 0ull;
        else x = -d < 32 ? (m << (-d)) : 0ull;
        ch[c] = (unsigned)(x & 0xffffffffull);
    }
    if (bits >> 63) {   // two's complement over 192 bits: invert, add 1 with carry
        unsigned long long carry = 1ull;
#pragma unroll
        for (int c = 0; c < FXCH; ++c) {
            const unsigned long long t = (unsigned long long)(~ch[c]) + carry;
            ch[c] = (unsigned)(t & 0xffffffffull);
            carry = t >> 32;
        }
    }
}
// chunk sums S_c (each < 2^64) -> sum_c S_c 2^(32c) mod 2^192 -> double (value X 2^-128)
__device__ __forceinline__ double fx192_to_double(const unsigned long long (&S)[FXCH]) {
    unsigned long long w[3] = {0ull, 0ull, 0ull};   // 192-bit accumulator, little-endian 64-bit words
#pragma unroll
    for (int c = 0; c < FXCH; ++c) {
        // add S_c << 32c
        const int wi = c / 2, off = 32 * (c % 2);
        unsigned __int128 add = (unsigned __int128)S[c] << off;   // < 2^96
        unsigned long long lo = (unsigned long long)add, hi = (unsigned long long)(add >> 64);
        unsigned long long carry = 0ull;
        for (int k = wi; k < 3; ++k) {
            const unsigned long long a = k == wi ? lo : (k == wi + 1 ? hi : 0ull);
            const unsigned __int128 t = (unsigned __int128)w[k] + a + carry;
            w[k] = (unsigned long long)t;
            carry = (unsigned long long)(t >> 64);
        }
    }
    const bool neg = (w[2] >> 63) != 0;
    if (neg) {   // magnitude of the two's-complement value
        unsigned long long carry = 1ull;
        for (int k = 0; k < 3; ++k) {
            const unsigned __int128 t = (unsigned __int128)(~w[k]) + carry;
            w[k] = (unsigned long long)t;
            carry = (unsigned long long)(t >> 64);
        }
    }
    const double mag = (double)w[2] + (double)w[1] * 5.421010862427522e-20 + (double)w[0] * 2.938735877055719e-39;
    return neg ? -mag : mag;
}
// Used by the per-phase loop kernel (k_scg_loop4: G3 266 vs 258 proj/s); the common-kappa loop kernel
// keeps grid_sum below (C2 490 vs 487, C4 168 vs 167 with this form; profiles/r02_grid_sum_fx_ab.txt).
__device__ void grid_sum_fx(const double (&acc)[NSLOT], double* part, unsigned* gbar, unsigned epoch,
                            double (&tot)[NSLOT]) {
    __shared__ double sred[32][NSLOT];
    __shared__ double stot[NSLOT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int G = gridDim.x;
    unsigned long long* sets = reinterpret_cast<unsigned long long*>(part);
    unsigned long long* cur = sets + (size_t)(epoch % 3) * FXA;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
        const double v = warp_sum(acc[k]);
        if (lane == 0) sred[warp][k] = v;
    }
    __syncthreads();
    FL_TMARK(epoch, 0)
    if (threadIdx.x < NSLOT) {   // this CTA's sum k -> exact chunks
        const int k = threadIdx.x;
        double v = 0.0;
        for (int w = 0; w < nw; ++w) v += sred[w][k];
        if (isfinite(v)) {
            unsigned ch[FXCH];
            fx192_chunks(v, ch);
#pragma unroll
            for (int c = 0; c < FXCH; ++c)
                if (ch[c]) red_add_u64(cur + k * FXCH + c, (unsigned long long)ch[c]);
        } else {
            red_add_u64(cur + NSLOT * FXCH, 1ull);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // release-reduction: this CTA's phase output and its chunk adds (ordered before it by the
        // barrier above, cumulativity) become visible to any CTA that acquires the count
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
        FL_TMARK(epoch, 1)
        const unsigned target = (epoch + 1) * (unsigned)G;
        unsigned spins = 0;
        const unsigned long long tstart = now_ns();
        while (ld_acquire_u32(gbar) < target) {
            // a lost CTA: fail loudly (after 10 s; a phase takes < 1 ms) instead of hanging the device
            if ((++spins & 1023u) == 0 && now_ns() - tstart > 10000000000ull) __trap();
        }
        FL_TMARK(epoch, 2)
        if (blockIdx.x == 0) {
            unsigned long long* nxt = sets + (size_t)((epoch + 2) % 3) * FXA;
            for (int i = 0; i < FXA; ++i) nxt[i] = 0ull;
        }
    }
    __syncthreads();
    if (threadIdx.x < NSLOT) {
        const int k = threadIdx.x;
        unsigned long long S[FXCH];
#pragma unroll
        for (int c = 0; c < FXCH; ++c) S[c] = ld_relaxed_u64(cur + k * FXCH + c);
        const bool bad = ld_relaxed_u64(cur + NSLOT * FXCH) != 0ull;
        stot[k] = bad ? __longlong_as_double(0x7ff8000000000000ll) : fx192_to_double(S);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) tot[k] = stot[k];
    FL_TMARK(epoch, 3)
    // the next phase reads other CTAs' generic-proxy stores through the bulk-copy (async) proxy
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// grid-wide sum of acc over all threads of all CTAs in a fixed order; result in tot (all threads)
__device__ void grid_sum(const double (&acc)[NSLOT], double* part, unsigned* gbar, unsigned epoch,
                         double (&tot)[NSLOT]) {
    __shared__ double sred[32][NSLOT];
    __shared__ double stot[NSLOT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int G = gridDim.x;
    double* slot = part + (size_t)(epoch & 1) * NSLOT * G;   // double-buffered by phase parity
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
        const double v = warp_sum(acc[k]);
        if (lane == 0) sred[warp][k] = v;
    }
    __syncthreads();
    FL_TMARK(epoch, 0)
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) {
            double v = 0.0;
            for (int w = 0; w < nw; ++w) v += sred[w][k];
            slot[(size_t)k * G + blockIdx.x] = v;
        }
        // release-reduction: this CTA's phase output (ordered before it by the barrier above,
        // cumulativity) and its slots become visible to any CTA that acquires the count
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
        FL_TMARK(epoch, 1)
        const unsigned target = (epoch + 1) * (unsigned)G;
        unsigned spins = 0;
        const unsigned long long tstart = now_ns();
        while (ld_acquire_u32(gbar) < target) {
            // a lost CTA: fail loudly (after 10 s; a phase takes < 1 ms) instead of hanging the device
            if ((++spins & 1023u) == 0 && now_ns() - tstart > 10000000000ull) __trap();
        }
        FL_TMARK(epoch, 2)
    }
    __syncthreads();
    // every CTA: slot j of CTA j by thread j, fixed shuffle tree, fixed cross-warp order
    double loc[NSLOT];
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) loc[k] = 0.0;
    for (int j = threadIdx.x; j < G; j += blockDim.x) {
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) loc[k] += ld_relaxed_gpu(slot + (size_t)k * G + j);
    }
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
        const double v = warp_sum(loc[k]);
        if (lane == 0) sred[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < NSLOT) {
        double v = 0.0;
        for (int w = 0; w < nw; ++w) v += sred[w][threadIdx.x];
        stot[threadIdx.x] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) tot[k] = stot[k];
    FL_TMARK(epoch, 3)
    // the next phase reads other CTAs' generic-proxy stores through the bulk-copy (async) proxy
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// det mode: the grid barrier of grid_sum with exact fixed-point CTA slots (FXW words each)
template <int WPB>
__device__ void grid_sum_det(FxCta<WPB>& fc, double* part, unsigned* gbar, unsigned epoch,
                             double (&tot)[NSLOT]) {
    const int G = gridDim.x;
    __int128* slot = reinterpret_cast<__int128*>(part) + (size_t)(epoch & 1) * FXW * G;
    __syncthreads();
    fx_cta_reduce(fc);
    __syncthreads();
    if (threadIdx.x < FXW) slot[(size_t)blockIdx.x * FXW + threadIdx.x] = fx_cta(fc, threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
        const unsigned target = (epoch + 1) * (unsigned)G;
        unsigned spins = 0;
        const unsigned long long tstart = now_ns();
        while (ld_acquire_u32(gbar) < target)
            if ((++spins & 1023u) == 0 && now_ns() - tstart > 10000000000ull) __trap();
    }
    __syncthreads();
    fx_sum_slots(slot, G, tot);
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// det mode: total -> the SCG sums (scale of the affine correction, the whole image's offsets)
template <int WHICH>
__device__ __forceinline__ void affine_det(const StencilParams& sp, double (&t)[NSLOT]) {
    const double* aff = WHICH == 0 ? sp.aff_vg : sp.aff_uc;
    const double* off = WHICH == 0 ? sp.det_off_vg : sp.det_off_uc;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) t[k] = t[k] * aff[k] + off[k];
}

template <int WHICH>
__device__ __forceinline__ void affine(const StencilParams& sp, double (&t)[NSLOT]) {
    const double* aff = WHICH == 0 ? sp.aff_vg : sp.aff_uc;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) t[k] = t[k] * aff[k] + aff[NSLOT + k];
}

}  // namespace
}  // namespace flmisr
