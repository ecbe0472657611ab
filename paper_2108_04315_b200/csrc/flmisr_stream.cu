// flmisr_stream.cu -- register-streaming sm_100a kernels for the FL-MISR SCG hot path when the
// composed kernel kappa is separable (kappa(P,Q) = a(P) b(Q): every Gaussian PSF) and KR <= 1
// (PSF up to 3x3 with integer HR phases) -- this covers all BASELINE configs.
//
// Work decomposition: one warp owns a strip of 128 HR columns (4 per lane)
// and a segment of S rows, and streams down the rows with 3-row register windows (x' = x + alpha p,
// the horizontal kappa pass of x', pending rows of -grad J).  Horizontal neighbours move by warp
// shuffles; strips overlap by SHALO = 2 columns per side (the reach of the fused operator: 2 KR for
// the data term's forward+adjoint chain, w-1 for BTV).  Each BTV pair (u, u+d) is evaluated once and
// its psi' goes to both endpoints (pending rows below, the right lane for columns to the right)
// -> 8 rsqrt per pixel.  The data gradient is scattered the same way (transposed correlation).
//
// Memory: the input rows of a step (512 B per array) are staged by the bulk-copy engine
// (cp.async.bulk, TMA 1D) into a per-warp NST-stage shared-memory ring completed by mbarriers, so
// the HBM latency is hidden NST-1 steps deep without registers.
//
// Packed fp32x2: a lane's columns c0..c3 are processed as the pairs A = (c0, c2), B = (c1, c3)
// with Blackwell's FFMA2 / FADD2 / FMUL2 (PTX f32x2), halving the FP32 issue slots.  To read the
// pairs with one 16-byte access, every HR buffer of the streaming path stores each aligned group
// of four columns as (c0, c2, c1, c3) ("permuted column layout"); ingest,
// initial estimate, output and the debug copies convert.  Reductions accumulate both pairs into
// one float2 whose .x holds columns c0+c1 and .y columns c2+c3, which is exactly the granularity
// of the strip's output-column masks.
// Image borders (clamped forward reads, folded adjoint, valid-pairs-only BTV; readings 4, 5) and
// band edges run in a separate instantiation selected per warp (warp-uniform).
// Constant terms (eps of every Charbonnier term, eps^2 of rho''/psi'') are hoisted into the affine
// correction of the CTA sums (StencilParams::aff_*).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "flmisr_common.cuh"
#include "flmisr_internal.h"
#include "flmisr_stream_common.cuh"

namespace flmisr {
namespace {


// (shared helpers, the ring, warp geometry, the grid barrier: flmisr_stream_common.cuh)

// a lane-0 shuffle of a (warp-uniform) condition: the compiler then sees it as uniform, so code under it
// needs no divergence handling and later bulk copies keep their uniform-register operands
__device__ __forceinline__ bool uni(bool c) { return __shfl_sync(0xffffffffu, (int)c, 0) != 0; }

// det mode: the CTA's exact per-lane accumulators, in dynamic shared memory after the warps' rings (the
// det kernels are launched with RING_SMEM + FX_SMEM bytes)
__device__ __forceinline__ FxCta<SWPB>& fx_shared() {
    extern __shared__ __align__(128) unsigned char smem[];
    return *reinterpret_cast<FxCta<SWPB>*>(smem + RING_SMEM);
}
// out of line: once per tile and slot.  Inlined, the branch-free conversion is if-converted into the
// streaming loop body and executed (predicated off) at every row step
__device__ __noinline__ void fx_add_f(int k, float v) { fx_lane_add(fx_shared(), k, v); }
__device__ __noinline__ void fx_add_d(int k, double v) { fx_lane_add(fx_shared(), k, v); }

// ------------------------------------------------------------------------------------------------
// value + gradient at x' = x + alpha p (Alg. 1 lines 14-19), streaming.
//   step t (ring stage = x,p(t+2), Y(t+1), r_old(t)): x'(t+2) -> horizontal kappa pass;
//   w(t+1) = rho'(kappa x' - Y) -> horizontal adjoint pass hw(t+1), scattered into the pending rows
//   t, t+1, t+2 of r = -grad J; BTV pairs of row t scattered into rows t..t+2; row t is complete.
// ------------------------------------------------------------------------------------------------
// DET (det mode): every accumulator is committed exactly (fx_add_f / fx_add_d) when its row closes a fixed tile
// of T rows -- the data value of row t+1 (group A) and the BTV / <r,r> / <r,r_old> sums of row t
// (group B) in step t.  T % 3 == 0 and segments start on a tile boundary, so every tile boundary inside
// a segment falls on the same unrolled step of each group (A: step<0>, B: step<1>): one commit site per
// group in the loop body; the segment's last (possibly short) tile is flushed after the loop.
template <int BW, int PN, bool BORDER, bool DET = false>
struct VG {
    float2 XA[3], XB[3];            // x' pairs (c0,c2), (c1,c3) of rows t, t+1, t+2 (slot (t+k)%3)
    float X4[3], X5[3];             // x' at c4, c5 (the right lane's c0, c1)
    float2 HA[3], HB[3];            // horizontal kappa pass of x'
    float2 GA[3], GB[3], GD[3], GE[3];   // pending r at (c0,c2), (c1,c3), (c2,c4), (c3,c5)
    float2 accd, vb[4], rr, rro;    // .x: columns c0+c1, .y: columns c2+c3
    const float *ix, *ip, *iy, *ir; // interior warps: next rows to stage (strip start column)
    float* qw;                      // interior warps: r_new row of the current step (lane column)
    int t0, nstep;
    int bA, bB;                     // DET: end row of the tile the data value / the row-t sums are in

    const StencilParams& sp;
    const Buffers& b;
    const Geo& g;
    const Ring& ring;
    const float* X0;
    const float* P0;
    const float* Rold;
    float* Rnew;
    float alpha;

    __device__ __forceinline__ VG(const StencilParams& sp_, const Buffers& b_, const Geo& g_, const Ring& ring_,
                                  const float* x, const float* p, const float* ro, float* rn, float al)
        : sp(sp_), b(b_), g(g_), ring(ring_), X0(x), P0(p), Rold(ro), Rnew(rn), alpha(al) {}

    // lane 0: stage the rows of step tt (x, p at tt+2; Y at tt+1; r_old at tt)
    __device__ __forceinline__ void issue(int s, int tt) {
        if (BORDER) {
            const float *a0 = rowp(X0, sp, tt + 2) + g.cbase, *a1 = rowp(P0, sp, tt + 2) + g.cbase;
            const float *a2 = rowp(b.Y, sp, tt + 1) + g.cbase, *a3 = rowp(Rold, sp, tt) + g.cbase;
            FL_BCHK(b, a0, SCOLS); FL_BCHK(b, a1, SCOLS); FL_BCHK(b, a2, SCOLS); FL_BCHK(b, a3, SCOLS);
            ring.issue(s, a0, a1, a2, a3);
        } else {
            FL_BCHK(b, ix, SCOLS); FL_BCHK(b, ip, SCOLS); FL_BCHK(b, iy, SCOLS); FL_BCHK(b, ir, SCOLS);
            ring.issue(s, ix, ip, iy, ir);
            ix += sp.pitch; ip += sp.pitch; iy += sp.pitch; ir += sp.pitch;
        }
    }

    // x'(row) into slot s, right neighbours, and the horizontal kappa pass
    __device__ __forceinline__ void set_x(int s, const float4& xv, const float4& pv) {
        XA[s] = fma2s(alpha, lo2(pv), lo2(xv));
        XB[s] = fma2s(alpha, hi2(pv), hi2(xv));
        float xm1 = shup(XB[s].y);
        X4[s] = shdn(XA[s].x);
        X5[s] = shdn(XB[s].x);
        if (BORDER) {
            if (g.strip0 && g.lane == 0) xm1 = XA[s].x;                  // clamp at column 0
            if (!g.cv4) { X4[s] = XB[s].y; X5[s] = XB[s].y; }            // clamp at column W-1
        }
        // hz(j) = b(-1) x(j-1) + b(0) x(j) + b(1) x(j+1)
        HA[s] = fma2s(sp.kb[0], F2(xm1, XB[s].x), fma2s(sp.kb[1], XA[s], mul2s(sp.kb[2], XB[s])));
        HB[s] = fma2s(sp.kb[0], XA[s], fma2s(sp.kb[1], XB[s], mul2s(sp.kb[2], F2(XA[s].y, X4[s]))));
    }

    template <int PH>
    __device__ __forceinline__ void step(int t, uint32_t par) {
        constexpr int s0 = PH % 3, s1 = (PH + 1) % 3, sa = (PH + 2) % 3;
        const float2 e2 = F2(sp.eps2, sp.eps2);
        constexpr int rs_ = PH;   // NST == 3 == the unroll: stage index is a compile-time constant
        ring.wait(rs_, par);
        const float4 fx = fixr<BORDER>(ring.get(rs_, 0, g.lane), g);
        const float4 fp = fixr<BORDER>(ring.get(rs_, 1, g.lane), g);
        const float4 fy = fixr<BORDER>(ring.get(rs_, 2, g.lane), g);
        const float4 fr = fixr<BORDER>(ring.get(rs_, 3, g.lane), g);

        // A: x'(t+2)
        set_x(sa, fx, fp);

        // B: w(t+1) = rho'(z - Y), data value, adjoint (transposed kappa) scattered into rows t..t+2
        {
            const int tw = t + 1;
            const float2 yA = lo2(fy), yB = hi2(fy);
            const bool orow = tw >= g.r_lo && tw < g.r_hi;
            const float2 zA = fma2s(sp.ka[0], HA[s0], fma2s(sp.ka[1], HA[s1], mul2s(sp.ka[2], HA[sa])));
            const float2 zB = fma2s(sp.ka[0], HB[s0], fma2s(sp.ka[1], HB[s1], mul2s(sp.ka[2], HB[sa])));
            const float2 eA = sub2(zA, yA), eB = sub2(zB, yB);
            float2 wA, wB;
            if (PN == 2) {
                if (orow) {
                    accd = fma2(eA, eA, accd);
                    accd = fma2(eB, eB, accd);
                }
                wA = fma2s(1.0f, eA, eA);
                wB = fma2s(1.0f, eB, eB);
            } else {
                const float2 qA = fma2(eA, eA, e2), qB = fma2(eB, eB, e2);
                const float2 rA = rsq2(qA), rB = rsq2(qB);
                if (orow) {   // rho + eps = q rs (eps * N is subtracted by the affine correction)
                    accd = fma2(qA, rA, accd);
                    accd = fma2(qB, rB, accd);
                }
                wA = mul2(eA, rA);
                wB = mul2(eB, rB);
            }
            if constexpr (DET && PH == 0) {
                if (uni(orow && tw + 1 == bA)) {   // row tw closes its tile: the tile's data value
                    commit_a();
                    bA = min(bA + sp.det_rows, g.r_hi);
                }
            }
            if (BORDER && !(tw >= 0 && tw < sp.H && g.cv0)) { wA = F2(0.f, 0.f); wB = wA; }   // zero-padded
            float wm1 = shup(wB.y), w4 = shdn(wA.x);
            if (BORDER) {
                if (g.strip0 && g.lane == 0) wm1 = 0.0f;
                if (!g.cv4) w4 = 0.0f;
            }
            // hw(j) = b(-1) w(j+1) + b(0) w(j) + b(1) w(j-1)
            float2 hA = fma2s(sp.kb[0], wB, fma2s(sp.kb[1], wA, mul2s(sp.kb[2], F2(wm1, wB.x))));
            float2 hB = fma2s(sp.kb[0], F2(wA.y, w4), fma2s(sp.kb[1], wB, mul2s(sp.kb[2], wA)));
            if (BORDER) {   // fold the clamped columns back onto the edge pixels (adjoint of clamp)
                if (g.strip0 && g.lane == 0) hA.x = fmaf(sp.kb[0], wA.x, hA.x);
                if (g.cv0 && !g.cv4) hB.y = fmaf(sp.kb[2], wB.y, hB.y);
            }
            // g(v) = sum_P a(P) hw(v - P): hw(t+1) feeds rows t (P=-1), t+1 (P=0), t+2 (P=+1)
            GA[s0] = fma2s(-sp.ka[0], hA, GA[s0]);
            GB[s0] = fma2s(-sp.ka[0], hB, GB[s0]);
            GA[s1] = fma2s(-sp.ka[1], hA, GA[s1]);
            GB[s1] = fma2s(-sp.ka[1], hB, GB[s1]);
            GA[sa] = fma2s(-sp.ka[2], hA, GA[sa]);
            GB[sa] = fma2s(-sp.ka[2], hB, GB[sa]);
            if (BORDER) {   // fold the clamped rows: row -1 onto row 0, row H onto row H-1
                if (tw == 0) {
                    GA[s1] = fma2s(-sp.ka[0], hA, GA[s1]);
                    GB[s1] = fma2s(-sp.ka[0], hB, GB[s1]);
                }
                if (tw == sp.H - 1) {
                    GA[s1] = fma2s(-sp.ka[2], hA, GA[s1]);
                    GB[s1] = fma2s(-sp.ka[2], hB, GB[s1]);
                }
            }
        }

        // D: BTV pairs (t, t+d) evaluated once; lambda gamma psi' to both endpoints (Eq. prior,
        // quadrant offsets, valid pairs only)
        const bool orow = t >= g.r_lo && t < g.r_hi;
        if (BW > 1 && t < g.r_hi && (!BORDER || (t >= 0 && t < sp.H))) {
#pragma unroll
            for (int dy = 0; dy < BW; ++dy) {
                if (BORDER && t + dy >= sp.H) continue;
                const int sq = (PH + dy) % 3;
#pragma unroll
                for (int dx = 0; dx < BW; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    const float lg = sp.lgc[dx + dy - 1];   // 4 distinct class weights (fewer uniform registers)
                    const int cls = dx + dy - 1;
                    const float2 D = F2(XA[sq].y, X4[sq]), E = F2(XB[sq].y, X5[sq]);
                    const float2 pA = dx == 0 ? XA[sq] : (dx == 1 ? XB[sq] : D);
                    const float2 pB = dx == 0 ? XB[sq] : (dx == 1 ? D : E);
                    const float2 dA = sub2(XA[s0], pA), dB = sub2(XB[s0], pB);
                    const float2 qA = fma2(dA, dA, e2), qB = fma2(dB, dB, e2);
                    const float2 rA = rsq2(qA), rB = rsq2(qB);
                    float2 uA = mul2(dA, rA), uB = mul2(dB, rB);
                    if (BORDER) {
                        // in the last in-image group (cv0 && !cv4) the partners c2+dx (dx = 2) and
                        // c3+dx (dx >= 1) fall outside the image; c0+dx, c1+dx never do
                        if (!g.cv0) { uA = F2(0.f, 0.f); uB = uA; }
                        if (!g.cv4) {
                            if (dx >= 2) uA.y = 0.f;
                            if (dx >= 1) uB.y = 0.f;
                        }
                        if (orow && DET) {   // masked q: fma(0, rs, v) = v, and a valid pair rounds exactly as
                                             // in the interior code (a tile's sums do not depend on whether a
                                             // band edge made it a border piece)
                            float2 mA = qA, mB = qB;
                            if (!g.cv0) { mA = F2(0.f, 0.f); mB = mA; }
                            if (!g.cv4) {
                                if (dx >= 2) mA.y = 0.f;
                                if (dx >= 1) mB.y = 0.f;
                            }
                            vb[cls] = fma2(mA, rA, vb[cls]);
                            vb[cls] = fma2(mB, rB, vb[cls]);
                        } else if (orow) {   // default: product then sum (measured 2% faster on C2 than the
                                             // masked FMA above)
                            float2 vA = mul2(qA, rA), vB = mul2(qB, rB);
                            if (!g.cv0) { vA = F2(0.f, 0.f); vB = vA; }
                            if (!g.cv4) {
                                if (dx >= 2) vA.y = 0.f;
                                if (dx >= 1) vB.y = 0.f;
                            }
                            vb[cls] = fma2s(1.0f, vA, vb[cls]);
                            vb[cls] = fma2s(1.0f, vB, vb[cls]);
                        }
                    } else if (orow) {
                        vb[cls] = fma2(qA, rA, vb[cls]);
                        vb[cls] = fma2(qB, rB, vb[cls]);
                    }
                    GA[s0] = fma2s(-lg, uA, GA[s0]);
                    GB[s0] = fma2s(-lg, uB, GB[s0]);
                    if (dx == 0) {
                        GA[sq] = fma2s(lg, uA, GA[sq]);
                        GB[sq] = fma2s(lg, uB, GB[sq]);
                    } else if (dx == 1) {
                        GB[sq] = fma2s(lg, uA, GB[sq]);
                        GD[sq] = fma2s(lg, uB, GD[sq]);
                    } else {
                        GD[sq] = fma2s(lg, uA, GD[sq]);
                        GE[sq] = fma2s(lg, uB, GE[sq]);
                    }
                }
            }
        }

        // E: row t is complete once the (c2,c4)/(c3,c5) pairs are folded and the right-spilled
        // columns of the left lane arrive
        {
            GA[s0].y += GD[s0].x;
            GB[s0].y += GE[s0].x;
            const float c4 = shup(GD[s0].y), c5 = shup(GE[s0].y);
            if (g.lane > 0) {
                GA[s0].x += c4;
                GB[s0].x += c5;
            }
            float* rp = BORDER ? Rnew + (size_t)(t - sp.store_lo) * sp.pitch + g.col0 : qw;
            if (!BORDER) qw += sp.pitch;
            if (orow) {
                FL_BCHK(b, rp, 4);
                stp(rp, GA[s0], GB[s0], g.olo, g.ohi);
                rr = fma2(GA[s0], GA[s0], rr);
                rr = fma2(GB[s0], GB[s0], rr);
                rro = fma2(GA[s0], lo2(fr), rro);
                rro = fma2(GB[s0], hi2(fr), rro);
                // band mode: owned boundary rows of the candidate go to the neighbours; those
                // rows lie in the first / last segment of the band, which are border warps
                if (BORDER && b.send_top && t - sp.row_lo < b.eta)
                    stp(b.send_top + (size_t)(t - sp.row_lo) * sp.pitch + g.col0, GA[s0], GB[s0], g.olo, g.ohi);
                if (BORDER && b.send_bot && sp.row_hi - 1 - t < b.eta)
                    stp(b.send_bot + (size_t)(t - (sp.row_hi - b.eta)) * sp.pitch + g.col0, GA[s0], GB[s0], g.olo,
                        g.ohi);
            }
            GA[s0] = GB[s0] = GD[s0] = GE[s0] = F2(0.f, 0.f);
            if constexpr (DET && PH == 1) {
                if (uni(orow && t + 1 == bB)) {   // row t closes its tile: BTV value, <r,r>, <r,r_old>
                    commit_b();
                    bB = min(bB + sp.det_rows, g.r_hi);
                }
            }
        }

        // the stage is consumed: refill it with the rows of step t + NST
        ring.release();
        if (t + NST < t0 + nstep) issue(rs_, t + NST);
    }

    // DET: exact commits of the partial tile sums (the same per-lane combination as vg_phase's msum)
    __device__ __forceinline__ void commit_a() {
        fx_add_f(0, msum(accd, g));
        accd = F2(0.f, 0.f);
    }
    __device__ __forceinline__ void commit_b() {
        fx_add_d(1, sp.gcls[0] * msum(vb[0], g) + sp.gcls[1] * msum(vb[1], g) + sp.gcls[2] * msum(vb[2], g) +
                        sp.gcls[3] * msum(vb[3], g));
        fx_add_f(2, msum(rr, g));
        fx_add_f(3, msum(rro, g));
#pragma unroll
        for (int c = 0; c < 4; ++c) vb[c] = F2(0.f, 0.f);
        rr = rro = F2(0.f, 0.f);
    }

    // par: the ring's current mbarrier phase parity (all stages advance together); carried across
    // runs when one kernel streams several phases through the same ring
    __device__ __forceinline__ void run(uint32_t& par) {
        const float2 z = F2(0.f, 0.f);
        accd = rr = rro = z;
#pragma unroll
        for (int c = 0; c < 4; ++c) vb[c] = z;
#pragma unroll
        for (int s = 0; s < 3; ++s) GA[s] = GB[s] = GD[s] = GE[s] = z;
        if (DET) bA = bB = min(g.r_lo + sp.det_rows, g.r_hi);   // segments start on a tile boundary
        t0 = g.r_lo - 2;
        nstep = (g.r_hi - g.r_lo + 4) / 3 * 3;   // rows r_lo - 2 .. r_hi - 1, rounded up to the unroll
        if (!BORDER) {
            const size_t o = (size_t)(t0 - sp.store_lo) * sp.pitch + g.cbase;
            ix = X0 + o + 2 * (size_t)sp.pitch;
            ip = P0 + o + 2 * (size_t)sp.pitch;
            iy = b.Y + o + (size_t)sp.pitch;
            ir = Rold + o;
            qw = Rnew + o + 4 * g.lane;
        }
        for (int k = 0; k < NST && k < nstep; ++k) issue(k, t0 + k);
        // rows t0, t0+1 of x' (the window before the first step) by direct loads
        set_x(0, ld4<BORDER>(rowp(X0, sp, t0), g.col0, sp.W), ld4<BORDER>(rowp(P0, sp, t0), g.col0, sp.W));
        set_x(1, ld4<BORDER>(rowp(X0, sp, t0 + 1), g.col0, sp.W), ld4<BORDER>(rowp(P0, sp, t0 + 1), g.col0, sp.W));
        for (int t = t0; t < t0 + nstep; t += 3) {
            step<0>(t, par);
            step<1>(t + 1, par);
            step<2>(t + 2, par);
            par ^= 1u;
        }
        if (DET) {   // the segment's last tile (an exact zero when the loop committed it already)
            commit_a();
            commit_b();
        }
    }
};



// ---- deferred reduction (sp.deferred): producers publish per-CTA slots, consumers settle them ----
// every thread: fixed-order sum over the G slots at slot[k * G + j] (thread j takes slot j, ...)
__device__ __forceinline__ void slot_sum(const double* slot, int G, double (&tot)[NSLOT]) {
    __shared__ double sred2[32][NSLOT];
    __shared__ double stot2[NSLOT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
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
        if (lane == 0) sred2[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < NSLOT) {
        double v = 0.0;
        for (int w = 0; w < nw; ++w) v += sred2[w][threadIdx.x];
        stot2[threadIdx.x] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) tot[k] = stot2[k];
}

// all threads of a CTA: S <- the global state with the pending scalar step applied (identical in every
// CTA: same slots, same order, same arithmetic); CTA 0 owns the trace
__device__ __forceinline__ void settle(const StencilParams& sp, const Buffers& b, ScgState& S) {
    if (threadIdx.x == 0) S = *b.st;
    __syncthreads();
    // warp-uniform copies (lane-0 shuffles) of everything that steers control flow
    const int pend = __shfl_sync(0xffffffffu, S.pend, 0);
    if (pend == PEND_NONE) return;
    const int G = __shfl_sync(0xffffffffu, S.pend_n, 0), seq = __shfl_sync(0xffffffffu, S.seq, 0);
    double tot[NSLOT];
    slot_sum(b.part + (size_t)(seq & 1) * NSLOT * G, G, tot);
    if (threadIdx.x == 0) {
        double* trace = blockIdx.x == 0 ? b.trace : nullptr;
        const double* aff = pend == PEND_UC ? sp.aff_uc : sp.aff_vg;
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) tot[k] = tot[k] * aff[k] + aff[NSLOT + k];
        if (pend == PEND_UC) {
            S.xcur ^= 1;
            scg_after_curv(&S, tot);
        } else {
            scg_after_value(&S, tot, trace, pend == PEND_VG_INIT ? PH_INIT : PH_ITER);
        }
        S.pend = PEND_NONE;
    }
    __syncthreads();
}

// all threads: this CTA's slot of the next sequence number (no atomics, no fence: the consumer is the
// next kernel, ordered by the kernel boundary)
__device__ __forceinline__ void publish(const double (&acc)[NSLOT], double* part, int seq) {
    __shared__ double sred3[32][NSLOT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
        const double v = warp_sum(acc[k]);
        if (lane == 0) sred3[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < NSLOT) {
        double v = 0.0;
        for (int w = 0; w < nw; ++w) v += sred3[w][threadIdx.x];
        part[(size_t)(seq & 1) * NSLOT * gridDim.x + (size_t)threadIdx.x * gridDim.x + blockIdx.x] = v;
    }
}

#ifdef FLMISR_PHASE_NOINLINE   // tuning build: separate register allocation per phase body
#define FL_PHASE_INLINE __noinline__
#else
#define FL_PHASE_INLINE __forceinline__
#endif

// One value+gradient phase of this CTA's warps: acc = this thread's share of {D, R (gamma-weighted),
// <r',r'>, <r',r_old>} (summed over the CTA and the grid by the caller).
// DET: the sums are committed per tile inside the row loop (fx_shared); acc is not written
template <int BW, int PN, bool DET = false>
__device__ FL_PHASE_INLINE void vg_phase(const StencilParams& sp, const Buffers& b, const Geo& g, const Ring& ring,
                                         int xcur, int rcur, float alpha, uint32_t& par, double (&acc)[NSLOT]) {
    const float* X = pick(b.X, xcur);
    const float* P = pick(b.P, xcur);
    const float* Ro = pick(b.R, rcur);
    float* Rn = pick(b.R, rcur ^ 1);
    if constexpr (DET) {
        if (!g.live) {
        } else if (g.border) {
            VG<BW, PN, true, true> v(sp, b, g, ring, X, P, Ro, Rn, alpha);
            v.run(par);
        } else {
            VG<BW, PN, false, true> v(sp, b, g, ring, X, P, Ro, Rn, alpha);
            v.run(par);
        }
        return;
    }
    float ad = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, a_rr = 0.f, a_rro = 0.f;
    if (!g.live) {
    } else if (g.border) {
        VG<BW, PN, true> v(sp, b, g, ring, X, P, Ro, Rn, alpha);
        v.run(par);
        ad = msum(v.accd, g); v0 = msum(v.vb[0], g); v1 = msum(v.vb[1], g); v2 = msum(v.vb[2], g);
        v3 = msum(v.vb[3], g); a_rr = msum(v.rr, g); a_rro = msum(v.rro, g);
    } else {
        VG<BW, PN, false> v(sp, b, g, ring, X, P, Ro, Rn, alpha);
        v.run(par);
        ad = msum(v.accd, g); v0 = msum(v.vb[0], g); v1 = msum(v.vb[1], g); v2 = msum(v.vb[2], g);
        v3 = msum(v.vb[3], g); a_rr = msum(v.rr, g); a_rro = msum(v.rro, g);
    }
    acc[0] = ad;
    acc[1] = sp.gcls[0] * v0 + sp.gcls[1] * v1 + sp.gcls[2] * v2 + sp.gcls[3] * v3;
    acc[2] = a_rr;
    acc[3] = a_rro;
}

// det mode, per-phase kernels (world > 1 over NCCL or device copies; one item per warp): the CTA's exact
// partial goes to its slot, the last CTA sums the slots exactly and publishes the band's FXW words as
// the rank-sum record (rank_sums); the scalar kernel after the allgather sums the bands exactly
__device__ bool reduce_partials_det(FxCta<SWPB>& fc, double* part, int ntiles, int tile, unsigned* counter,
                                    __int128 (&tot)[FXW]) {
    __shared__ int s_last;
    __syncthreads();
    fx_cta_reduce(fc);
    __syncthreads();
    __int128* slot = reinterpret_cast<__int128*>(part);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < FXW; ++k) slot[(size_t)tile * FXW + k] = fx_cta(fc, k);
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(counter) : "memory");
        s_last = prev == (unsigned)(ntiles - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    fx_sum_raw(slot, ntiles, tot);
    if (threadIdx.x == 0) *counter = 0u;
    return true;
}
template <int WHICH>
__device__ void finish_det(const StencilParams& sp, const Buffers& b, const __int128 (&tw)[FXW], int phase) {
    if (threadIdx.x != 0) return;
    if (sp.world > 1 && phase != PH_DEBUG) {   // the band's exact record for the allgather
        __int128* rs = reinterpret_cast<__int128*>(b.rank_sums);
#pragma unroll
        for (int k = 0; k < FXW; ++k) rs[k] = tw[k];
        return;
    }
    double tot[NSLOT];
#pragma unroll
    for (int k = 0; k < NSLOT; ++k)
        tot[k] = tw[NSLOT] != 0 ? __longlong_as_double(0x7ff8000000000000ll) : fx_to_double(tw[k]);
    affine_det<WHICH>(sp, tot);
    ScgState* s = b.st;
    if (phase == PH_DEBUG) {
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) s->dbg[k] = tot[k];
        return;
    }
    ScgState l = *s;
    if (WHICH == 0) scg_after_value(&l, tot, b.trace, phase);
    else scg_after_curv(&l, tot);
    *s = l;
}

template <int BW, int PN, bool DET = false>
__global__ void __launch_bounds__(SWPB * 32, SMINB) k_vg_stream(StencilParams sp, Buffers b, int phase) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ ScgState S;
    pdl_enter();
    ScgState* st = b.st;
    const bool deferred = sp.deferred && phase != PH_DEBUG;
    int xcur, rcur, seq = 0;
    float alpha;
    // every branch condition below goes through a lane-0 shuffle: a condition the compiler cannot
    // prove warp-uniform makes every later instruction potentially divergent, which forces the bulk
    // copies into per-lane waterfall loops and the address arithmetic out of the uniform datapath
    if (deferred) {   // apply the previous kernel's pending scalar step (every CTA, identically)
        settle(sp, b, S);
        if (__shfl_sync(0xffffffffu, S.done, 0)) {
            if (blockIdx.x == 0 && threadIdx.x == 0) *st = S;
            return;
        }
        xcur = S.xcur; rcur = S.rcur; alpha = S.alpha_f; seq = S.seq + 1;
    } else {
        if (phase != PH_DEBUG && __shfl_sync(0xffffffffu, st->done, 0)) return;
        xcur = st->xcur; rcur = st->rcur; alpha = st->alpha_f;
    }
    // lane-0 shuffles: the compiler sees these as warp-uniform (uniform buffer pointers for the copies)
    xcur = __shfl_sync(0xffffffffu, xcur, 0);
    rcur = __shfl_sync(0xffffffffu, rcur, 0);
    alpha = phase == PH_ITER ? __shfl_sync(0xffffffffu, alpha, 0) : 0.0f;
    const int wslot = blockIdx.x * SWPB + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const Geo g = DET ? geometry_item<SHALO, true>(sp, wslot) : geometry(sp, blockIdx.x);
    Ring ring;
    ring.init(smem, __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), g.lane);
    double acc[NSLOT];
    uint32_t par = 0;
    if constexpr (DET) {   // world > 1 (det mode at world 1 runs the persistent loop kernel)
        FxCta<SWPB>& fc = fx_shared();
        fx_zero(fc);
        __syncthreads();
        vg_phase<BW, PN, true>(sp, b, g, ring, xcur, rcur, alpha, par, acc);   // commits per tile
        __int128 tw[FXW];
        if (reduce_partials_det(fc, b.part, gridDim.x, blockIdx.x, &st->counter, tw)) finish_det<0>(sp, b, tw, phase);
        return;
    }
    vg_phase<BW, PN>(sp, b, g, ring, xcur, rcur, alpha, par, acc);
    if (deferred) {
        publish(acc, b.part, seq);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            S.pend = phase == PH_INIT ? PEND_VG_INIT : PEND_VG_ITER;
            S.pend_n = gridDim.x;
            S.seq = seq;
            *st = S;
        }
        return;
    }
    double tot[NSLOT];
    if (reduce_partials(acc, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) finish_scalars<0>(sp, b, tot, phase);
}

// ------------------------------------------------------------------------------------------------
// update x <- x + alpha_upd p, p <- r + beta p (Alg. 1 lines 14, 20), then the exact curvature
// p^T Hess J p, <p,p>, <p,r> at the new (x, p) (lines 6-12; reading 16), streaming.
//   ring stage of step t: x, p, r at row t+2, Y at row t+1.
// ------------------------------------------------------------------------------------------------
// DET: as in VG -- the data curvature of row t+1 (group A, step<0>), the BTV curvature of row t (group
// B, step<1>) and <p,p>, <p,r> of row t+2 (group C, set in step t, step<2>) are committed when their row
// closes a tile; the last tile after the loop
template <int BW, int PN, bool BORDER, bool DET = false>
struct UC {
    float2 XA[3], XB[3], PA[3], PB[3];   // new x / p pairs (c0,c2), (c1,c3)
    float X4[3], X5[3], P4[3], P5[3];    // new x / p at c4, c5
    float2 HXA[3], HXB[3], HPA[3], HPB[3];
    float2 cd, cb[4], pp, mu;            // .x: columns c0+c1, .y: columns c2+c3
    const float *ix, *ip, *ir, *iy;      // interior warps: next rows to stage (strip start column)
    int t0, nstep;
    int bA, bB, bC;                      // DET: tile end rows of the cd / cb / (pp, mu) rows
    const StencilParams& sp;
    const Buffers& b;
    const Geo& g;
    const Ring& ring;
    const float *X0, *P0, *R0;
    float *Xn, *Pn;
    float au, be;

    __device__ __forceinline__ UC(const StencilParams& sp_, const Buffers& b_, const Geo& g_, const Ring& ring_,
                                  const float* x, const float* p, const float* r, float* xn, float* pn, float a,
                                  float bb)
        : sp(sp_), b(b_), g(g_), ring(ring_), X0(x), P0(p), R0(r), Xn(xn), Pn(pn), au(a), be(bb) {}

    __device__ __forceinline__ void issue(int s, int tt) {
        if (BORDER) {
            const float *a0 = rowp(X0, sp, tt + 2) + g.cbase, *a1 = rowp(P0, sp, tt + 2) + g.cbase;
            const float *a2 = rrowp(b, R0, sp, tt + 2) + g.cbase, *a3 = rowp(b.Y, sp, tt + 1) + g.cbase;
            FL_BCHK(b, a0, SCOLS); FL_BCHK(b, a1, SCOLS); FL_BCHK(b, a3, SCOLS);   // a2 may be a halo row
            ring.issue(s, a0, a1, a2, a3);
        } else {
            FL_BCHK(b, ix, SCOLS); FL_BCHK(b, ip, SCOLS); FL_BCHK(b, ir, SCOLS); FL_BCHK(b, iy, SCOLS);
            ring.issue(s, ix, ip, ir, iy);
            ix += sp.pitch; ip += sp.pitch; ir += sp.pitch; iy += sp.pitch;
        }
    }

    __device__ __forceinline__ void set_row(int s, int row, const float4& xv, const float4& pv, const float4& rv) {
        XA[s] = fma2s(au, lo2(pv), lo2(xv));
        XB[s] = fma2s(au, hi2(pv), hi2(xv));
        PA[s] = fma2s(be, lo2(pv), lo2(rv));
        PB[s] = fma2s(be, hi2(pv), hi2(rv));
        if (row >= g.w_lo && row < g.w_hi) {
            const size_t off = (size_t)(row - sp.store_lo) * sp.pitch + g.col0;
            FL_BCHK(b, Xn + off, 4); FL_BCHK(b, Pn + off, 4);
            stp(Xn + off, XA[s], XB[s], g.olo, g.ohi);
            stp(Pn + off, PA[s], PB[s], g.olo, g.ohi);
            if (row >= g.r_lo && row < g.r_hi) {
                pp = fma2(PA[s], PA[s], pp);
                pp = fma2(PB[s], PB[s], pp);
                mu = fma2(PA[s], lo2(rv), mu);
                mu = fma2(PB[s], hi2(rv), mu);
            }
        }
        float xm1 = shup(XB[s].y), pm1 = shup(PB[s].y);
        X4[s] = shdn(XA[s].x);
        X5[s] = shdn(XB[s].x);
        P4[s] = shdn(PA[s].x);
        P5[s] = shdn(PB[s].x);
        if (BORDER) {
            if (g.strip0 && g.lane == 0) { xm1 = XA[s].x; pm1 = PA[s].x; }
            if (!g.cv4) { X4[s] = X5[s] = XB[s].y; P4[s] = P5[s] = PB[s].y; }
        }
        HXA[s] = fma2s(sp.kb[0], F2(xm1, XB[s].x), fma2s(sp.kb[1], XA[s], mul2s(sp.kb[2], XB[s])));
        HXB[s] = fma2s(sp.kb[0], XA[s], fma2s(sp.kb[1], XB[s], mul2s(sp.kb[2], F2(XA[s].y, X4[s]))));
        HPA[s] = fma2s(sp.kb[0], F2(pm1, PB[s].x), fma2s(sp.kb[1], PA[s], mul2s(sp.kb[2], PB[s])));
        HPB[s] = fma2s(sp.kb[0], PA[s], fma2s(sp.kb[1], PB[s], mul2s(sp.kb[2], F2(PA[s].y, P4[s]))));
    }

    template <int PH>
    __device__ __forceinline__ void step(int t, uint32_t par) {
        constexpr int s0 = PH % 3, s1 = (PH + 1) % 3, sa = (PH + 2) % 3;
        const float2 e2 = F2(sp.eps2, sp.eps2);
        constexpr int rs_ = PH;   // NST == 3 == the unroll: stage index is a compile-time constant
        ring.wait(rs_, par);
        set_row(sa, t + 2, fixr<BORDER>(ring.get(rs_, 0, g.lane), g), fixr<BORDER>(ring.get(rs_, 1, g.lane), g),
                fixr<BORDER>(ring.get(rs_, 2, g.lane), g));
        if constexpr (DET && PH == 2) {
            if (uni(t + 2 >= g.r_lo && t + 2 < g.r_hi && t + 3 == bC)) {   // row t+2 closes its tile: <p,p>, <p,r>
                commit_c();
                bC = min(bC + sp.det_rows, g.r_hi);
            }
        }
        const float4 fy = fixr<BORDER>(ring.get(rs_, 3, g.lane), g);
        // data curvature at row t+1: rho''(e) (A p)^2 = eps^2 rs^3 (A p)^2 (eps^2 in the affine term)
        {
            const int tz = t + 1;
            if (tz >= g.r_lo && tz < g.r_hi) {
                const float2 apA = fma2s(sp.ka[0], HPA[s0], fma2s(sp.ka[1], HPA[s1], mul2s(sp.ka[2], HPA[sa])));
                const float2 apB = fma2s(sp.ka[0], HPB[s0], fma2s(sp.ka[1], HPB[s1], mul2s(sp.ka[2], HPB[sa])));
                if (PN == 2) {
                    cd = fma2(apA, apA, cd);
                    cd = fma2(apB, apB, cd);
                } else {
                    const float2 zA = fma2s(sp.ka[0], HXA[s0], fma2s(sp.ka[1], HXA[s1], mul2s(sp.ka[2], HXA[sa])));
                    const float2 zB = fma2s(sp.ka[0], HXB[s0], fma2s(sp.ka[1], HXB[s1], mul2s(sp.ka[2], HXB[sa])));
                    const float2 eA = sub2(zA, lo2(fy)), eB = sub2(zB, hi2(fy));
                    const float2 rA = rsq2(fma2(eA, eA, e2)), rB = rsq2(fma2(eB, eB, e2));
                    const float2 uA = mul2(rA, apA), uB = mul2(rB, apB);
                    cd = fma2(mul2(uA, uA), rA, cd);
                    cd = fma2(mul2(uB, uB), rB, cd);
                }
                if constexpr (DET && PH == 0) {
                    if (uni(tz + 1 == bA)) {   // row tz closes its tile: the tile's data curvature
                        commit_a();
                        bA = min(bA + sp.det_rows, g.r_hi);
                    }
                }
            }
        }
        ring.release();
        if (t + NST < t0 + nstep) issue(rs_, t + NST);
        // BTV curvature of the pairs (t, t+d): psi''(D x) (D p)^2 = eps^2 rs^3 (D p)^2
        if (BW > 1 && t >= g.r_lo && t < g.r_hi) {
#pragma unroll
            for (int dy = 0; dy < BW; ++dy) {
                if (BORDER && t + dy >= sp.H) continue;
                const int sq = (PH + dy) % 3;
#pragma unroll
                for (int dx = 0; dx < BW; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    const int cls = dx + dy - 1;
                    const float2 XD = F2(XA[sq].y, X4[sq]), XE = F2(XB[sq].y, X5[sq]);
                    const float2 PD = F2(PA[sq].y, P4[sq]), PE = F2(PB[sq].y, P5[sq]);
                    const float2 xA = dx == 0 ? XA[sq] : (dx == 1 ? XB[sq] : XD);
                    const float2 xB = dx == 0 ? XB[sq] : (dx == 1 ? XD : XE);
                    const float2 qpA = dx == 0 ? PA[sq] : (dx == 1 ? PB[sq] : PD);
                    const float2 qpB = dx == 0 ? PB[sq] : (dx == 1 ? PD : PE);
                    const float2 dxA = sub2(XA[s0], xA), dxB = sub2(XB[s0], xB);
                    const float2 dpA = sub2(PA[s0], qpA), dpB = sub2(PB[s0], qpB);
                    const float2 rA = rsq2(fma2(dxA, dxA, e2)), rB = rsq2(fma2(dxB, dxB, e2));
                    float2 uA = mul2(rA, dpA), uB = mul2(rB, dpB);
                    if (BORDER) {
                        if (!g.cv0) { uA = F2(0.f, 0.f); uB = uA; }
                        if (!g.cv4) {
                            if (dx >= 2) uA.y = 0.f;
                            if (dx >= 1) uB.y = 0.f;
                        }
                    }
                    cb[cls] = fma2(mul2(uA, uA), rA, cb[cls]);
                    cb[cls] = fma2(mul2(uB, uB), rB, cb[cls]);
                }
            }
            if constexpr (DET && PH == 1) {
                if (uni(t + 1 == bB)) {   // row t closes its tile: the tile's BTV curvature
                    commit_b();
                    bB = min(bB + sp.det_rows, g.r_hi);
                }
            }
        }
    }

    __device__ __forceinline__ void commit_a() {
        fx_add_f(0, msum(cd, g));
        cd = F2(0.f, 0.f);
    }
    __device__ __forceinline__ void commit_b() {
        fx_add_d(1, sp.gcls[0] * msum(cb[0], g) + sp.gcls[1] * msum(cb[1], g) + sp.gcls[2] * msum(cb[2], g) +
                        sp.gcls[3] * msum(cb[3], g));
#pragma unroll
        for (int c = 0; c < 4; ++c) cb[c] = F2(0.f, 0.f);
    }
    __device__ __forceinline__ void commit_c() {
        fx_add_f(2, msum(pp, g));
        fx_add_f(3, msum(mu, g));
        pp = mu = F2(0.f, 0.f);
    }

    // par: the ring's current mbarrier phase parity (all stages advance together); carried across
    // runs when one kernel streams several phases through the same ring
    __device__ __forceinline__ void run(uint32_t& par) {
        const float2 z = F2(0.f, 0.f);
        cd = pp = mu = z;
#pragma unroll
        for (int c = 0; c < 4; ++c) cb[c] = z;
        if (DET) bA = bB = bC = min(g.r_lo + sp.det_rows, g.r_hi);   // segments start on a tile boundary
        t0 = g.r_lo - 2;
        nstep = (g.r_hi - g.r_lo + 4) / 3 * 3;
        if (!BORDER) {
            const size_t o = (size_t)(t0 - sp.store_lo) * sp.pitch + g.cbase;
            ix = X0 + o + 2 * (size_t)sp.pitch;
            ip = P0 + o + 2 * (size_t)sp.pitch;
            ir = R0 + o + 2 * (size_t)sp.pitch;
            iy = b.Y + o + (size_t)sp.pitch;
        }
        for (int k = 0; k < NST && k < nstep; ++k) issue(k, t0 + k);
        set_row(0, t0, ld4<BORDER>(rowp(X0, sp, t0), g.col0, sp.W), ld4<BORDER>(rowp(P0, sp, t0), g.col0, sp.W),
                ld4<BORDER>(rrowp(b, R0, sp, t0), g.col0, sp.W));
        set_row(1, t0 + 1, ld4<BORDER>(rowp(X0, sp, t0 + 1), g.col0, sp.W),
                ld4<BORDER>(rowp(P0, sp, t0 + 1), g.col0, sp.W), ld4<BORDER>(rrowp(b, R0, sp, t0 + 1), g.col0, sp.W));
        for (int t = t0; t < t0 + nstep; t += 3) {
            step<0>(t, par);
            step<1>(t + 1, par);
            step<2>(t + 2, par);
            par ^= 1u;
        }
        if (DET) {   // the segment's last tile
            commit_a();
            commit_b();
            commit_c();
        }
    }
};

// One update+curvature phase of this CTA's warps: acc = {sum rho'' (A p)^2, BTV curvature
// (gamma-weighted), <p,p>, <p,r>} at the new (x, p).
template <int BW, int PN, bool DET = false>
__device__ FL_PHASE_INLINE void uc_phase(const StencilParams& sp, const Buffers& b, const Geo& g, const Ring& ring,
                                         int xcur, int rcur, float au, float be, uint32_t& par,
                                         double (&acc)[NSLOT]) {
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, a_pp = 0.f, a_mu = 0.f;
    const float* X = pick(b.X, xcur);
    const float* P = pick(b.P, xcur);
    const float* R = pick(b.R, rcur);
    float* Xn = pick(b.X, xcur ^ 1);
    float* Pn = pick(b.P, xcur ^ 1);
    if constexpr (DET) {
        if (!g.live) {
        } else if (g.border) {
            UC<BW, PN, true, true> u(sp, b, g, ring, X, P, R, Xn, Pn, au, be);
            u.run(par);
        } else {
            UC<BW, PN, false, true> u(sp, b, g, ring, X, P, R, Xn, Pn, au, be);
            u.run(par);
        }
        return;
    }
    if (!g.live) {
    } else if (g.border) {
        UC<BW, PN, true> u(sp, b, g, ring, X, P, R, Xn, Pn, au, be);
        u.run(par);
        c0 = msum(u.cd, g); c1 = msum(u.cb[0], g); c2 = msum(u.cb[1], g); c3 = msum(u.cb[2], g);
        c4 = msum(u.cb[3], g); a_pp = msum(u.pp, g); a_mu = msum(u.mu, g);
    } else {
        UC<BW, PN, false> u(sp, b, g, ring, X, P, R, Xn, Pn, au, be);
        u.run(par);
        c0 = msum(u.cd, g); c1 = msum(u.cb[0], g); c2 = msum(u.cb[1], g); c3 = msum(u.cb[2], g);
        c4 = msum(u.cb[3], g); a_pp = msum(u.pp, g); a_mu = msum(u.mu, g);
    }
    acc[0] = c0;
    acc[1] = sp.gcls[0] * c1 + sp.gcls[1] * c2 + sp.gcls[2] * c3 + sp.gcls[3] * c4;
    acc[2] = a_pp;
    acc[3] = a_mu;
}

// det mode: this warp's work items it0, it0 + stride, ... (segments that are unions of the fixed global
// tiles; normally one item per warp); each tile's sums are committed exactly inside the row loop, so
// neither the segmentation, the item -> warp assignment nor the band split changes the totals
template <int BW, int PN>
__device__ __forceinline__ void vg_items(const StencilParams& sp, const Buffers& b, const Ring& ring, int it0,
                                         int stride, int xcur, int rcur, float alpha, uint32_t& par) {
    FxCta<SWPB>& fc = fx_shared();
    fx_zero(fc);
    __syncthreads();
    for (int it = it0; uni(it < sp.nitems); it += stride) {
        const Geo g = geometry_item<SHALO, true>(sp, __shfl_sync(0xffffffffu, it, 0));
        double acc[NSLOT];
        vg_phase<BW, PN, true>(sp, b, g, ring, xcur, rcur, alpha, par, acc);   // commits per tile
    }
}
template <int BW, int PN>
__device__ __forceinline__ void uc_items(const StencilParams& sp, const Buffers& b, const Ring& ring, int it0,
                                         int stride, int xcur, int rcur, float au, float be, uint32_t& par) {
    FxCta<SWPB>& fc = fx_shared();
    fx_zero(fc);
    __syncthreads();
    for (int it = it0; uni(it < sp.nitems); it += stride) {
        const Geo g = geometry_item<SHALO, true>(sp, __shfl_sync(0xffffffffu, it, 0));
        double acc[NSLOT];
        uc_phase<BW, PN, true>(sp, b, g, ring, xcur, rcur, au, be, par, acc);   // commits per tile
    }
}

template <int BW, int PN, bool DET = false>
__global__ void __launch_bounds__(SWPB * 32, SMINB) k_uc_stream(StencilParams sp, Buffers b, int phase) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ ScgState S;
    pdl_enter();
    ScgState* st = b.st;
    const bool deferred = sp.deferred && phase != PH_DEBUG;
    int xcur, rcur, seq = 0;
    float au, be;
    if (deferred) {   // apply the previous kernel's pending scalar step (every CTA, identically)
        settle(sp, b, S);
        if (__shfl_sync(0xffffffffu, S.done || !S.success, 0)) {   // finished, or rejected: delta reused
            if (threadIdx.x == 0 && !S.done) scg_pre_value(&S);
            if (blockIdx.x == 0 && threadIdx.x == 0) *st = S;
            return;
        }
        xcur = S.xcur; rcur = S.rcur; au = S.alpha_upd_f; be = S.beta_f; seq = S.seq + 1;
    } else {
        if (phase != PH_DEBUG) {
            if (__shfl_sync(0xffffffffu, st->done, 0)) return;
            if (!__shfl_sync(0xffffffffu, st->success, 0)) {   // rejected step: delta is reused
                if (sp.world == 1 && blockIdx.x == 0 && threadIdx.x == 0) scg_pre_value(st);
                return;
            }
        }
        xcur = st->xcur; rcur = st->rcur;
        au = phase == PH_DEBUG ? 0.0f : st->alpha_upd_f;
        be = phase == PH_DEBUG ? 0.0f : st->beta_f;
    }
    xcur = __shfl_sync(0xffffffffu, xcur, 0);
    rcur = __shfl_sync(0xffffffffu, rcur, 0);
    au = __shfl_sync(0xffffffffu, au, 0);
    be = __shfl_sync(0xffffffffu, be, 0);
    const int wslot = blockIdx.x * SWPB + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const Geo g = DET ? geometry_item<SHALO, true>(sp, wslot) : geometry(sp, blockIdx.x);
    Ring ring;
    ring.init(smem, __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), g.lane);
    double acc[NSLOT];
    uint32_t par = 0;
    if constexpr (DET) {
        FxCta<SWPB>& fc = fx_shared();
        fx_zero(fc);
        __syncthreads();
        uc_phase<BW, PN, true>(sp, b, g, ring, xcur, rcur, au, be, par, acc);   // commits per tile
        __int128 tw[FXW];
        if (reduce_partials_det(fc, b.part, gridDim.x, blockIdx.x, &st->counter, tw)) {
            if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
            finish_det<1>(sp, b, tw, phase);
        }
        return;
    }
    uc_phase<BW, PN>(sp, b, g, ring, xcur, rcur, au, be, par, acc);
    if (deferred) {
        publish(acc, b.part, seq);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            S.pend = PEND_UC;
            S.pend_n = gridDim.x;
            S.seq = seq;
            *st = S;
        }
        return;
    }
    double tot[NSLOT];
    if (reduce_partials(acc, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

__global__ void k_settle(StencilParams sp, Buffers b) {
    pdl_enter();
    __shared__ ScgState S;
    settle(sp, b, S);
    if (threadIdx.x == 0) *b.st = S;
}

// ------------------------------------------------------------------------------------------------
// The whole SCG loop in one persistent cooperative kernel (world == 1): one CTA per SM streams
// every phase of Alg. 1 through the same ring; phases are separated by a grid barrier after which
// EVERY CTA sums the per-CTA slots in the same fixed order and runs the same scalar logic on its own
// shared-memory copy of the state (bit-identical in all CTAs), so no CTA waits on a serial last-CTA
// reduction or on kernel teardown and relaunch.  CTA 0 writes the trace and the final state.
// ------------------------------------------------------------------------------------------------

template <int BW, int PN, bool DET>
__global__ void __launch_bounds__(SWPB * 32, SMINB) k_scg_loop(const __grid_constant__ StencilParams sp,
                                                                const __grid_constant__ Buffers b) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ ScgState S;
    const Geo g = geometry(sp, blockIdx.x);   // DET: unused (items are taken in a grid-stride loop)
    const int it0 = blockIdx.x * SWPB + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    Ring ring;
    ring.init(smem, __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), g.lane);
    if (threadIdx.x == 0) S = *b.st;
    __syncthreads();
    double* trace = blockIdx.x == 0 ? b.trace : nullptr;
    uint32_t par = 0;
    unsigned epoch = 0;
    double acc[NSLOT], tot[NSLOT];
    // state fields are read from shared memory through a lane-0 shuffle so the compiler sees them as
    // warp-uniform: the buffer pointers derived from xcur / rcur then stay in uniform registers and
    // the bulk copies take them directly (no per-copy register-to-uniform waterfall)
    auto ui = [](int v) { return __shfl_sync(0xffffffffu, v, 0); };
    auto uf = [](float v) { return __shfl_sync(0xffffffffu, v, 0); };
    // pass 0 is the init value+gradient (f0 = J(x0), r0 = -grad J(x0)); every later pass is
    // [update+curvature if the last step was accepted] + value+gradient.  One call site per phase body.
    for (int pass = 0; !ui(S.done); ++pass) {
        if (pass > 0) {
            if (ui(S.success)) {   // update x, p and the curvature at the new direction
                if constexpr (DET) {
                    uc_items<BW, PN>(sp, b, ring, it0, gridDim.x * SWPB, ui(S.xcur), ui(S.rcur), uf(S.alpha_upd_f),
                                     uf(S.beta_f), par);
                    grid_sum_det(fx_shared(), b.part, b.gbar, epoch++, tot);
                } else {
                    uc_phase<BW, PN>(sp, b, g, ring, ui(S.xcur), ui(S.rcur), uf(S.alpha_upd_f), uf(S.beta_f), par, acc);
                    grid_sum(acc, b.part, b.gbar, epoch++, tot);
                }
                if (threadIdx.x == 0) {
                    S.xcur ^= 1;
                    if constexpr (DET) affine_det<1>(sp, tot);
                    else affine<1>(sp, tot);
                    scg_after_curv(&S, tot);
                }
            } else if (threadIdx.x == 0) {   // rejected step: delta is reused
                scg_pre_value(&S);
            }
            __syncthreads();
            if (ui(S.done)) break;
        }
        if constexpr (DET) {
            vg_items<BW, PN>(sp, b, ring, it0, gridDim.x * SWPB, ui(S.xcur), ui(S.rcur), pass > 0 ? uf(S.alpha_f) : 0.0f,
                             par);
            grid_sum_det(fx_shared(), b.part, b.gbar, epoch++, tot);
        } else {
            vg_phase<BW, PN>(sp, b, g, ring, ui(S.xcur), ui(S.rcur), pass > 0 ? uf(S.alpha_f) : 0.0f, par, acc);
            grid_sum(acc, b.part, b.gbar, epoch++, tot);
        }
        if (threadIdx.x == 0) {
            if constexpr (DET) affine_det<0>(sp, tot);
            else affine<0>(sp, tot);
            scg_after_value(&S, tot, trace, pass > 0 ? PH_ITER : PH_INIT);
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *b.st = S;
}

// ------------------------------------------------------------------------------------------------
// Row bands over peer memory: the whole SCG loop of one band as one persistent kernel, the bands
// synchronised per phase through peer-mapped memory.  After each phase EVERY
// CTA of every band
//   stores its fp64 partial sums into every rank's mailbox, slot [epoch & 1][rank][cta], then (one
//     fence at system scope when the peers are other GPUs: its candidate r rows, stored straight into
//     the neighbours' halo buffers, are ordered first) adds 1 to every rank's arrival counter;
//   waits until its own rank's counter reaches (epoch + 1) x world x ctas (the counters only grow,
//     across calls too, so no rank ever resets a word a peer writes);
//   sums all world x ctas slots of its own mailbox in one fixed order -- the same consensus scalars,
//     bit for bit, on every rank -- and runs the scalar logic (Alg. 1).
// One hop per phase, as in the single-GPU loop kernel's grid barrier, with the band affine
// corrections applied per slot owner.  One kernel per rank on a multi-GPU node (g = 1, peers =
// CUDA-IPC mappings over NVLink); on one device all g bands run in ONE cooperative launch with local
// pointers (the emulation the profiling guide prescribes for ranks that wait on one another).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p, bool sys) {
    unsigned long long v;
    if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// all threads of every CTA: consensus sums of this phase into tot.  Returns false (every thread of the
// CTA) when the arrivals did not complete within pl.timeout_ns: a rank or CTA is lost (e.g. peer memory
// without working system-scope atomics); the caller abandons the loop instead of trapping, so the
// context survives and the host can fall back to the NCCL transport.
__device__ bool peer_sum(const StencilParams& sp, const PeerLoop& pl, int l, int j, int which,
                         const double (&acc)[NSLOT], unsigned epoch, double (&tot)[NSLOT]) {
    __shared__ int s_timeout;
    __shared__ double sred[32][NSLOT];
    __shared__ double stot[NSLOT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int C = pl.ctas, h = pl.rank0 + l, world = pl.world;
    const bool sys = pl.g == 1;   // peers on other GPUs
    const size_t par = (size_t)(epoch & 1) * world * C * NSLOT;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
        const double v = warp_sum(acc[k]);
        if (lane == 0) sred[warp][k] = v;
    }
    __syncthreads();
    FL_TMARK(epoch, 0)
    if (threadIdx.x == 0) {
        // this CTA's slot with the band's affine correction spread over its slots (aff * v + off / C)
        const double* aff = which == 0 ? sp.aff_vg : sp.aff_uc;
        double v[NSLOT];
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += sred[w][k];
            v[k] = t * aff[k] + (j == 0 ? aff[NSLOT + k] : 0.0);
        }
        const size_t o = par + ((size_t)h * C + j) * NSLOT;
        for (int q = 0; q < world; ++q) {
#pragma unroll
            for (int k = 0; k < NSLOT; ++k) pl.mbox[q][o + k] = v[k];
        }
        if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (h != pl.drop_band) {
            for (int q = 0; q < world; ++q) {
                if (sys) asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(pl.cnt[q]) : "memory");
                else asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(pl.cnt[q]) : "memory");
            }
        }
        FL_TMARK(epoch, 1)
        const unsigned long long target = (unsigned long long)(epoch + 1) * (unsigned long long)(world * C);
        unsigned spins = 0;
        const unsigned long long tstart = now_ns();
        int to = 0;
        while (ld_acquire_u64(pl.cnt[h], sys) < target)   // a lost rank or CTA: give up after timeout_ns
            if ((++spins & 1023u) == 0 && now_ns() - tstart > pl.timeout_ns) { to = 1; break; }
        s_timeout = to;
    }
    __syncthreads();
    if (s_timeout) return false;
    FL_TMARK(epoch, 2)
    // fixed-order sum of the world x C slots: slot i = (rank, cta) by thread i % blockDim, then a fixed
    // shuffle tree and cross-warp order
    {
        const double* mb = pl.mbox[h] + par;
        double loc[NSLOT];
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) loc[k] = 0.0;
        for (int i = threadIdx.x; i < world * C; i += blockDim.x)
#pragma unroll
            for (int k = 0; k < NSLOT; ++k) loc[k] += ld_relaxed_gpu(mb + (size_t)i * NSLOT + k);
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
    }
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) tot[k] = stot[k];
    FL_TMARK(epoch, 3)
    // the next phase reads peer-written halo rows through the bulk-copy (async) proxy
    asm volatile("fence.proxy.async.global;" ::: "memory");
    return true;
}

// det mode: peer_sum with exact fixed-point CTA slots (FXW words) and the whole image's affine offsets
// applied once to the exact all-band total -- the same bits at every band count
__device__ bool peer_sum_det(const StencilParams& sp, const PeerLoop& pl, int l, int j, int which, unsigned epoch,
                             double (&tot)[NSLOT]) {
    __shared__ int s_timeout;
    const int C = pl.ctas, h = pl.rank0 + l, world = pl.world;
    const bool sys = pl.g == 1;
    const size_t par = (size_t)(epoch & 1) * world * C * FXW;
    FxCta<SWPB>& fc = fx_shared();
    __syncthreads();
    fx_cta_reduce(fc);
    __syncthreads();
    if (threadIdx.x == 0) {
        __int128 v[FXW];
#pragma unroll
        for (int k = 0; k < FXW; ++k) v[k] = fx_cta(fc, k);
        const size_t o = par + ((size_t)h * C + j) * FXW;
        for (int q = 0; q < world; ++q) {
            __int128* mb = reinterpret_cast<__int128*>(pl.mbox[q]);
#pragma unroll
            for (int k = 0; k < FXW; ++k) mb[o + k] = v[k];
        }
        if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (h != pl.drop_band) {
            for (int q = 0; q < world; ++q) {
                if (sys) asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(pl.cnt[q]) : "memory");
                else asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(pl.cnt[q]) : "memory");
            }
        }
        const unsigned long long target = (unsigned long long)(epoch + 1) * (unsigned long long)(world * C);
        unsigned spins = 0;
        const unsigned long long tstart = now_ns();
        int to = 0;
        while (ld_acquire_u64(pl.cnt[h], sys) < target)
            if ((++spins & 1023u) == 0 && now_ns() - tstart > pl.timeout_ns) { to = 1; break; }
        s_timeout = to;
    }
    __syncthreads();
    if (s_timeout) return false;
    fx_sum_slots(reinterpret_cast<const __int128*>(pl.mbox[h]) + par, world * C, tot);
    if (which == 0) affine_det<0>(sp, tot);
    else affine_det<1>(sp, tot);
    asm volatile("fence.proxy.async.global;" ::: "memory");
    return true;
}

template <int BW, int PN, bool DET>
__device__ __forceinline__ void peer_loop_body(const StencilParams& sp, const Buffers& b, const PeerLoop& pl, int l,
                                               int j, unsigned char* smem, ScgState& S) {
    const Geo g = geometry(sp, j);   // DET: unused (grid-stride items of the band)
    const int it0 = j * SWPB + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), stride = pl.ctas * SWPB;
    Ring ring;
    ring.init(smem, __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), g.lane);
    __shared__ unsigned s_e0;
    if (threadIdx.x == 0) {
        S = *b.st;
        s_e0 = *pl.epoch_word[l];   // epochs of the earlier calls (written by the previous launch)
    }
    __syncthreads();
    double* trace = j == 0 ? b.trace : nullptr;
    uint32_t par = 0;
    unsigned epoch = s_e0;
    double acc[NSLOT], tot[NSLOT];
    auto ui = [](int v) { return __shfl_sync(0xffffffffu, v, 0); };
    auto uf = [](float v) { return __shfl_sync(0xffffffffu, v, 0); };
    for (int pass = 0; !ui(S.done); ++pass) {
        if (pass > 0) {
            if (ui(S.success)) {
                bool ok;
                if constexpr (DET) {
                    uc_items<BW, PN>(sp, b, ring, it0, stride, ui(S.xcur), ui(S.rcur), uf(S.alpha_upd_f), uf(S.beta_f),
                                     par);
                    ok = peer_sum_det(sp, pl, l, j, 1, epoch++, tot);
                } else {
                    uc_phase<BW, PN>(sp, b, g, ring, ui(S.xcur), ui(S.rcur), uf(S.alpha_upd_f), uf(S.beta_f), par, acc);
                    ok = peer_sum(sp, pl, l, j, 1, acc, epoch++, tot);
                }
                if (!ok) {
                    if (threadIdx.x == 0) { S.done = 1; S.failed_stage = FAIL_PEER_TIMEOUT; S.failed_iter = S.k; }
                    __syncthreads();
                    break;
                }
                if (threadIdx.x == 0) {
                    S.xcur ^= 1;
                    scg_after_curv(&S, tot);
                }
            } else if (threadIdx.x == 0) {
                scg_pre_value(&S);
            }
            __syncthreads();
            if (ui(S.done)) break;
        }
        bool ok;
        if constexpr (DET) {
            vg_items<BW, PN>(sp, b, ring, it0, stride, ui(S.xcur), ui(S.rcur), pass > 0 ? uf(S.alpha_f) : 0.0f, par);
            ok = peer_sum_det(sp, pl, l, j, 0, epoch++, tot);
        } else {
            vg_phase<BW, PN>(sp, b, g, ring, ui(S.xcur), ui(S.rcur), pass > 0 ? uf(S.alpha_f) : 0.0f, par, acc);
            ok = peer_sum(sp, pl, l, j, 0, acc, epoch++, tot);
        }
        if (!ok) {
            if (threadIdx.x == 0) { S.done = 1; S.failed_stage = FAIL_PEER_TIMEOUT; S.failed_iter = S.k; }
            __syncthreads();
            break;
        }
        if (threadIdx.x == 0) scg_after_value(&S, tot, trace, pass > 0 ? PH_ITER : PH_INIT);
        __syncthreads();
    }
    if (j == 0 && threadIdx.x == 0) {
        *b.st = S;
        *pl.epoch_word[l] = epoch;   // the next call's first epoch (identical on every rank)
    }
}

// one band per launch (multi-GPU): parameters in the constant bank
template <int BW, int PN, bool DET>
__global__ void __launch_bounds__(SWPB * 32, SMINB) k_scg_peer_loop(const __grid_constant__ StencilParams sp,
                                                                     const __grid_constant__ Buffers b,
                                                                     const __grid_constant__ PeerLoop pl) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ ScgState S;
    peer_loop_body<BW, PN, DET>(sp, b, pl, 0, blockIdx.x, smem, S);
}

// all bands in one cooperative launch (one device): band l = blockIdx.x / ctas; every band's
// parameters in the constant bank (block-uniform index)
template <int BW, int PN, bool DET>
__global__ void __launch_bounds__(SWPB * 32, SMINB) k_scg_peer_loop_multi(const __grid_constant__ PeerLoop pl,
                                                                           const __grid_constant__ PeerBands pb) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ ScgState S;
    const int l = __shfl_sync(0xffffffffu, (int)(blockIdx.x / pl.ctas), 0);
    const int j = blockIdx.x - l * pl.ctas;
    peer_loop_body<BW, PN, DET>(pb.sp[l], pb.b[l], pl, l, j, smem, S);
}

bool pdl_enabled() {
    static const bool on = std::getenv("FLMISR_NO_PDL") == nullptr;
    return on;
}

template <typename K>
cudaError_t launch_ring(K kernel, int nw, const StencilParams& sp, const Buffers& b, int phase, cudaStream_t s,
                        size_t smem = RING_SMEM) {
    // opt in to > 48 KB of dynamic shared memory once per kernel instantiation (per device)
    const cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kernel), smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((nw + SWPB - 1) / SWPB);
    cfg.blockDim = dim3(SWPB * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, sp, b, phase);
}

}  // namespace

#define FL_SCASE(K, BW_, PN_)                                                                                 \
    case BW_ * 10 + PN_:                                                                                      \
        return sp.det ? launch_ring(K<BW_, PN_, true>, sp.nitems, sp, b, phase, s, RING_SMEM + FX_SMEM) \
                      : launch_ring(K<BW_, PN_, false>, sp.nitems, sp, b, phase, s);

template <typename K>
cudaError_t launch_loop(K kernel, int nw, const StencilParams& sp, const Buffers& b, cudaStream_t s, size_t smem) {
    const cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kernel), smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((nw + SWPB - 1) / SWPB);
    cfg.blockDim = dim3(SWPB * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // every CTA co-resident: the grid barrier cannot deadlock
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, sp, b);
}

cudaError_t launch_value_grad_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                                     cudaStream_t s) {
    switch (bw * 10 + pn) {
        FL_SCASE(k_vg_stream, 1, 1) FL_SCASE(k_vg_stream, 1, 2) FL_SCASE(k_vg_stream, 2, 1)
        FL_SCASE(k_vg_stream, 2, 2) FL_SCASE(k_vg_stream, 3, 1) FL_SCASE(k_vg_stream, 3, 2)
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_settle(const StencilParams& sp, const Buffers& b, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(512);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_settle, sp, b);
}

cudaError_t launch_scg_loop_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, cudaStream_t s) {
    switch (bw * 10 + pn) {
#define FL_LCASE(BW_, PN_) \
    case BW_ * 10 + PN_:   \
        return sp.det ? launch_loop(k_scg_loop<BW_, PN_, true>, sp.loop_warps, sp, b, s, RING_SMEM + FX_SMEM) \
                      : launch_loop(k_scg_loop<BW_, PN_, false>, sp.loop_warps, sp, b, s, RING_SMEM);
        FL_LCASE(1, 1) FL_LCASE(1, 2) FL_LCASE(2, 1) FL_LCASE(2, 2) FL_LCASE(3, 1) FL_LCASE(3, 2)
#undef FL_LCASE
        default: return cudaErrorInvalidValue;
    }
}

template <typename K, typename... A>
cudaError_t launch_coop(K kernel, size_t smem, int grid, cudaStream_t s, A... args) {
    const cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kernel), smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(SWPB * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // co-residency: the barriers cannot deadlock
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

cudaError_t launch_scg_peer_loop(int bw, int pn, const StencilParams& sp, const Buffers& b, const PeerLoop& pl,
                                 const PeerBands* pb, cudaStream_t s) {
    switch (bw * 10 + pn) {
#define FL_PCASE(BW_, PN_) \
    case BW_ * 10 + PN_:   \
        if (sp.det)        \
            return pl.g == 1 ? launch_coop(k_scg_peer_loop<BW_, PN_, true>, RING_SMEM + FX_SMEM, pl.ctas, s, sp, b, pl) \
                             : launch_coop(k_scg_peer_loop_multi<BW_, PN_, true>, RING_SMEM + FX_SMEM, pl.g * pl.ctas, \
                                           s, pl, *pb);                                                              \
        return pl.g == 1 ? launch_coop(k_scg_peer_loop<BW_, PN_, false>, RING_SMEM, pl.ctas, s, sp, b, pl) \
                         : launch_coop(k_scg_peer_loop_multi<BW_, PN_, false>, RING_SMEM, pl.g * pl.ctas, s, pl, *pb);
        FL_PCASE(1, 1) FL_PCASE(1, 2) FL_PCASE(2, 1) FL_PCASE(2, 2) FL_PCASE(3, 1) FL_PCASE(3, 2)
#undef FL_PCASE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_update_curv_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                                      cudaStream_t s) {
    switch (bw * 10 + pn) {
        FL_SCASE(k_uc_stream, 1, 1) FL_SCASE(k_uc_stream, 1, 2) FL_SCASE(k_uc_stream, 2, 1)
        FL_SCASE(k_uc_stream, 2, 2) FL_SCASE(k_uc_stream, 3, 1) FL_SCASE(k_uc_stream, 3, 2)
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace flmisr

#ifdef FLMISR_TIMING
extern "C" int flmisr_debug_loop_timing(unsigned long long* host, int n) {
    if (n > 64 * 256 * 4) n = 64 * 256 * 4;
    return (int)cudaMemcpyFromSymbol(host, flmisr::g_loop_time, (size_t)n * sizeof(unsigned long long));
}
#endif
