// flmisr_stream4.cu -- register-streaming sm_100a kernels for polyphase-complete stacks whose frames
// carry DIFFERENT composed kernels (the "per-phase" path, fast_path 4): K = mag^2 = 4 frames whose
// integer HR phases s_i tile [0,2)^2 but whose sub-pixel remainders phi_i differ, so frame i has its
// own kappa_i = h (*) bilinear(phi_i) (reading 19) -- e.g. G3's quarter-LR-pixel detector positions
// at x2, or any real acquisition whose shifts are only approximately half pixels.  Eq. sisr
// with arbitrary translations.
//
// Because the integer phases are complete, every HR pixel u still holds exactly one LR sample (the
// polyphase Y of the common-kappa path) and the data term is an HR-grid stencil whose 4x4 kernel
// depends on the pixel's phase class c(u) = (u_y mod 2, u_x mod 2):
//     z(u) = sum_{P,Q in [-1,2]} kappa_{c(u)}(P,Q) x~(u + (P,Q)),   r(v) = -sum_u kappa_{c(u)}(v-u) rho'(z(u)-Y(u)) - lambda grad R
// (clamped reads, folded adjoint at the image border; readings 4, 5).  The work decomposition is the
// common-kappa streaming kernels' (flmisr_stream.cu): one warp per (128-column strip, row segment),
// 4 columns per lane held as the fp32x2 pairs A = (c0, c2) and B = (c1, c3) -- both members of a pair
// share a column class, so every tap is a warp-uniform scalar broadcast into FFMA2 -- rows staged by
// the bulk-copy engine into a per-warp ring.  Differences: a 4-row x' window and 4 pending rows
// (kappa offsets -1..2), 4 ring stages (the row loop is unrolled by 4, so the row class of every step
// is a compile-time constant: segments start on even rows), strips overlap by 4 columns per side
// (forward + adjoint reach 3), the adjoint is gathered from shuffled residual pairs, and the residual
// is formed as y - z so that the pending rows accumulate r = -grad J directly.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "flmisr_common.cuh"
#include "flmisr_internal.h"
#include "flmisr_stream_common.cuh"

namespace flmisr {
namespace {

constexpr int NS4 = 4;   // ring stages == row-loop unroll == x' window rows == pending rows
constexpr int H4 = 4;    // strip column overlap per side
using Ring4 = RingT<NS4>;
constexpr size_t RING4_SMEM = RingDims<NS4, PC_WPB>::SMEM;
static_assert(SCOLS - 2 * H4 == PC_SSTEP, "per-phase strip step");

// tap of phase class cls = 2 rho + gamma at offset (P, Q), P, Q in [-1, 2] (compile-time indices:
// a constant-bank operand)
#define TK(cls, P, Q) T.k[(cls)][((P) + 1) * 4 + ((Q) + 1)]

// acc += k (a, b) for a pair whose members live in different registers ((c-1, c1), (c2, c4), (c3, c5)):
// two scalar FFMAs instead of materialising the pair -- the compiler otherwise re-forms such pairs with
// MOVs at every use (~17 per pixel measured)
__device__ __forceinline__ float2 fmam(float k, float a, float b, float2 acc) {
    return F2(fmaf(k, a, acc.x), fmaf(k, b, acc.y));
}

// ------------------------------------------------------------------------------------------------
// value + gradient at x' = x + alpha p, streaming.  Step t (ring stage = x, p(t+3), Y(t+1), r_old(t)):
// x'(t+3) into the window; w(t+1) = -rho'(z(t+1) - Y(t+1)) from window rows t..t+3, gathered into the
// pending rows t..t+3; BTV pairs of row t scattered into rows t..t+2; row t is complete.
// Segment start r_lo is even, t0 = r_lo - 3 is odd: row t0 + PH has parity (1 + PH) & 1.
// ------------------------------------------------------------------------------------------------
template <int BW, int PN, bool BORDER>
struct VG4 {
    // x' of the window rows (slot = (row - t0) & 3): the pairs A = (c0, c2), B = (c1, c3) and the
    // neighbours c-1 (left lane's c3), c4, c5 (right lane's c0, c1); the kappa offsets Q = -1 of A and
    // Q = 1, 2 of B read the mixed pairs (c-1, c1), (c2, c4), (c3, c5) through fmam
    float2 XA[4], XB[4];
    float XM[4], X4[4], X5[4];
    float2 GA[4], GB[4], GD[4], GE[4];   // pending r at (c0,c2), (c1,c3), (c2,c4), (c3,c5)
    float2 accd, vb[4], rr, rro;    // .x: columns c0+c1, .y: columns c2+c3
    const float *ix, *ip, *iy, *ir; // interior warps: next rows to stage (strip start column)
    float* qw;                      // interior warps: r_new row of the current step (lane column)
    int t0, nstep;

    const StencilParams& sp;
    const Buffers& b;
    const PcTaps& T;
    const Geo& g;
    const Ring4& ring;
    const float* X0;
    const float* P0;
    const float* Rold;
    float* Rnew;
    float alpha;

    __device__ __forceinline__ VG4(const StencilParams& sp_, const Buffers& b_, const PcTaps& T_, const Geo& g_,
                                   const Ring4& ring_, const float* x, const float* p, const float* ro, float* rn,
                                   float al)
        : sp(sp_), b(b_), T(T_), g(g_), ring(ring_), X0(x), P0(p), Rold(ro), Rnew(rn), alpha(al) {}

    __device__ __forceinline__ void issue(int s, int tt) {
        if (BORDER) {
            const float *a0 = rowp(X0, sp, tt + 3) + g.cbase, *a1 = rowp(P0, sp, tt + 3) + g.cbase;
            const float *a2 = rowp(b.Y, sp, tt + 1) + g.cbase, *a3 = rowp(Rold, sp, tt) + g.cbase;
            FL_BCHK(b, a0, SCOLS); FL_BCHK(b, a1, SCOLS); FL_BCHK(b, a2, SCOLS); FL_BCHK(b, a3, SCOLS);
            ring.issue(s, a0, a1, a2, a3);
        } else {
            FL_BCHK(b, ix, SCOLS); FL_BCHK(b, ip, SCOLS); FL_BCHK(b, iy, SCOLS); FL_BCHK(b, ir, SCOLS);
            ring.issue(s, ix, ip, iy, ir);
            ix += sp.pitch; ip += sp.pitch; iy += sp.pitch; ir += sp.pitch;
        }
    }

    __device__ __forceinline__ void set_x(int s, const float4& xv, const float4& pv) {
        XA[s] = fma2s(alpha, lo2(pv), lo2(xv));
        XB[s] = fma2s(alpha, hi2(pv), hi2(xv));
        float xm1 = shup(XB[s].y), x4 = shdn(XA[s].x), x5 = shdn(XB[s].x);
        if (BORDER) {
            if (g.strip0 && g.lane == 0) xm1 = XA[s].x;                  // clamp at column 0
            if (!g.cv4) { x4 = XB[s].y; x5 = XB[s].y; }                  // clamp at column W-1
        }
        XM[s] = xm1;
        X4[s] = x4;
        X5[s] = x5;
    }

    template <int PH>
    __device__ __forceinline__ void step(int t, uint32_t par) {
        constexpr int s0 = PH, s1 = (PH + 1) & 3, s2 = (PH + 2) & 3, s3 = (PH + 3) & 3;
        constexpr int rho = PH & 1;                  // parity of row t + 1 (t0 odd)
        constexpr int cA = 2 * rho, cB = 2 * rho + 1;   // classes of the pairs A (even cols), B (odd cols)
        const float2 e2 = F2(sp.eps2, sp.eps2);
        ring.wait(PH, par);
        const float4 fx = fixr<BORDER>(ring.get(PH, 0, g.lane), g);
        const float4 fp = fixr<BORDER>(ring.get(PH, 1, g.lane), g);
        const float4 fy = fixr<BORDER>(ring.get(PH, 2, g.lane), g);
        const float4 fr = fixr<BORDER>(ring.get(PH, 3, g.lane), g);

        // A: x'(t+3)
        set_x(s3, fx, fp);

        // B: w(t+1) = -rho'(z - Y) (as rho'(Y - z)), data value, gathered adjoint into rows t..t+3
        {
            const int tw = t + 1;
            float2 zA = F2(0.f, 0.f), zB = zA;
            const int sl[4] = {s0, s1, s2, s3};
#pragma unroll
            for (int j = 0; j < 4; ++j) {   // window row j = offset P = j - 1
                const int q = sl[j];
                zA = fmam(TK(cA, j - 1, -1), XM[q], XB[q].x, zA);
                zA = fma2s(TK(cA, j - 1, 0), XA[q], zA);
                zA = fma2s(TK(cA, j - 1, 1), XB[q], zA);
                zA = fmam(TK(cA, j - 1, 2), XA[q].y, X4[q], zA);
                zB = fma2s(TK(cB, j - 1, -1), XA[q], zB);
                zB = fma2s(TK(cB, j - 1, 0), XB[q], zB);
                zB = fmam(TK(cB, j - 1, 1), XA[q].y, X4[q], zB);
                zB = fmam(TK(cB, j - 1, 2), XB[q].y, X5[q], zB);
            }
            const bool orow = tw >= g.r_lo && tw < g.r_hi;
            const float2 eA = sub2(lo2(fy), zA), eB = sub2(hi2(fy), zB);   // Y - z = -e
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
            if (BORDER && !(tw >= 0 && tw < sp.H && g.cv0)) { wA = F2(0.f, 0.f); wB = wA; }   // zero-padded
            float wm1 = shup(wB.y), wm2 = shup(wA.y), w4 = shdn(wA.x);
            if (BORDER) {
                if (g.strip0 && g.lane == 0) { wm1 = 0.0f; wm2 = 0.0f; }
                if (!g.cv4) w4 = 0.0f;
            }
            // mixed residual pairs (c-1, c1) = (wm1, wB.x), (c-2, c0) = (wm2, wA.x), (c2, c4) = (wA.y, w4)
            // target row t+1+P gets sum_Q kappa_{c(u)}(P,Q) w(u), u = v - (P,Q):
            //   v in A: Q=-1 u=(c1,c3) class B, Q=0 A, Q=1 (c-1,c1) class B, Q=2 (c-2,c0) class A
            //   v in B: Q=-1 u=(c2,c4) class A, Q=0 B, Q=1 A, Q=2 (c-1,c1) class B
            if (!BORDER) {
                // interior: straight into the pending rows t..t+3
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int q = sl[j];
                    GA[q] = fma2s(TK(cB, j - 1, -1), wB, GA[q]);
                    GA[q] = fma2s(TK(cA, j - 1, 0), wA, GA[q]);
                    GA[q] = fmam(TK(cB, j - 1, 1), wm1, wB.x, GA[q]);
                    GA[q] = fmam(TK(cA, j - 1, 2), wm2, wA.x, GA[q]);
                    GB[q] = fmam(TK(cA, j - 1, -1), wA.y, w4, GB[q]);
                    GB[q] = fma2s(TK(cB, j - 1, 0), wB, GB[q]);
                    GB[q] = fma2s(TK(cA, j - 1, 1), wA, GB[q]);
                    GB[q] = fmam(TK(cB, j - 1, 2), wm1, wB.x, GB[q]);
                }
            } else {
                float2 cAa[4], cBa[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float2 a = mul2s(TK(cB, j - 1, -1), wB);
                    a = fma2s(TK(cA, j - 1, 0), wA, a);
                    a = fmam(TK(cB, j - 1, 1), wm1, wB.x, a);
                    cAa[j] = fmam(TK(cA, j - 1, 2), wm2, wA.x, a);
                    float2 c = F2(TK(cA, j - 1, -1) * wA.y, TK(cA, j - 1, -1) * w4);
                    c = fma2s(TK(cB, j - 1, 0), wB, c);
                    c = fma2s(TK(cA, j - 1, 1), wA, c);
                    cBa[j] = fmam(TK(cB, j - 1, 2), wm1, wB.x, c);
                }
                // columns: the clamped forward reads fold back onto the edge pixels (adjoint of clamp):
                // v = 0 also takes u = 0 at Q = -1; v = W-1 (c3 of the last in-image group) takes
                // u = W-1 at Q = 1, 2 and u = W-2 at Q = 2
                if (g.strip0 && g.lane == 0) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) cAa[j].x = fmaf(TK(cA, j - 1, -1), wA.x, cAa[j].x);
                }
                if (g.cv0 && !g.cv4) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        cBa[j].y = fmaf(TK(cB, j - 1, 1) + TK(cB, j - 1, 2), wB.y, fmaf(TK(cA, j - 1, 2), wA.y, cBa[j].y));
                }
                // rows: row -1 folds onto row 0, rows H and H+1 onto row H-1
                if (tw == 0) {
                    cAa[1] = add2(cAa[1], cAa[0]); cBa[1] = add2(cBa[1], cBa[0]);
                    cAa[0] = cBa[0] = F2(0.f, 0.f);
                }
                if (tw == sp.H - 1) {
                    cAa[1] = add2(cAa[1], add2(cAa[2], cAa[3])); cBa[1] = add2(cBa[1], add2(cBa[2], cBa[3]));
                    cAa[2] = cBa[2] = cAa[3] = cBa[3] = F2(0.f, 0.f);
                } else if (tw == sp.H - 2) {
                    cAa[2] = add2(cAa[2], cAa[3]); cBa[2] = add2(cBa[2], cBa[3]);
                    cAa[3] = cBa[3] = F2(0.f, 0.f);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    GA[sl[j]] = add2(GA[sl[j]], cAa[j]);
                    GB[sl[j]] = add2(GB[sl[j]], cBa[j]);
                }
            }
        }

        // D: BTV pairs (t, t+d) evaluated once; lambda gamma psi' to both endpoints (Eq. prior,
        // quadrant offsets, valid pairs only) -- as in flmisr_stream.cu
        const bool orow = t >= g.r_lo && t < g.r_hi;
        if (BW > 1 && t < g.r_hi && (!BORDER || (t >= 0 && t < sp.H))) {
#pragma unroll
            for (int dy = 0; dy < BW; ++dy) {
                if (BORDER && t + dy >= sp.H) continue;
                const int sq = (PH + dy) & 3;
#pragma unroll
                for (int dx = 0; dx < BW; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    const float lg = sp.lgc[dx + dy - 1];
                    const int cls = dx + dy - 1;
                    // partners: dx = 0: A, B; dx = 1: B, (c2, c4); dx = 2: (c2, c4), (c3, c5) of row t + dy
                    const float2 dA = dx == 0 ? sub2(XA[s0], XA[sq])
                                    : dx == 1 ? sub2(XA[s0], XB[sq])
                                              : F2(XA[s0].x - XA[sq].y, XA[s0].y - X4[sq]);
                    const float2 dB = dx == 0 ? sub2(XB[s0], XB[sq])
                                    : dx == 1 ? F2(XB[s0].x - XA[sq].y, XB[s0].y - X4[sq])
                                              : F2(XB[s0].x - XB[sq].y, XB[s0].y - X5[sq]);
                    const float2 qA = fma2(dA, dA, e2), qB = fma2(dB, dB, e2);
                    const float2 rA = rsq2(qA), rB = rsq2(qB);
                    float2 uA = mul2(dA, rA), uB = mul2(dB, rB);
                    if (BORDER) {
                        if (!g.cv0) { uA = F2(0.f, 0.f); uB = uA; }
                        if (!g.cv4) {
                            if (dx >= 2) uA.y = 0.f;
                            if (dx >= 1) uB.y = 0.f;
                        }
                        if (orow) {
                            float2 vA = mul2(qA, rA), vB = mul2(qB, rB);
                            if (!g.cv0) { vA = F2(0.f, 0.f); vB = vA; }
                            if (!g.cv4) {
                                if (dx >= 2) vA.y = 0.f;
                                if (dx >= 1) vB.y = 0.f;
                            }
                            vb[cls] = add2(vb[cls], add2(vA, vB));
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

        // E: row t is complete once the BTV spills of the (c2,c4)/(c3,c5) pairs are folded
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
            }
            GA[s0] = GB[s0] = GD[s0] = GE[s0] = F2(0.f, 0.f);
        }

        ring.release();
        if (t + NS4 < t0 + nstep) issue(PH, t + NS4);
    }

    __device__ __forceinline__ void run(uint32_t& par) {
        const float2 z = F2(0.f, 0.f);
        accd = rr = rro = z;
#pragma unroll
        for (int c = 0; c < 4; ++c) vb[c] = z;
#pragma unroll
        for (int s = 0; s < 4; ++s) GA[s] = GB[s] = GD[s] = GE[s] = z;
        t0 = g.r_lo - 3;
        nstep = (g.r_hi - g.r_lo + 3 + 3) / 4 * 4;   // rows r_lo - 3 .. r_hi - 1, rounded up to the unroll
        if (!BORDER) {
            const size_t o = (size_t)(t0 - sp.store_lo) * sp.pitch + g.cbase;
            ix = X0 + o + 3 * (size_t)sp.pitch;
            ip = P0 + o + 3 * (size_t)sp.pitch;
            iy = b.Y + o + (size_t)sp.pitch;
            ir = Rold + o;
            qw = Rnew + o + 4 * g.lane;
        }
        for (int k = 0; k < NS4 && k < nstep; ++k) issue(k, t0 + k);
        // rows t0 .. t0 + 2 of x' (the window before the first step) by direct loads
#pragma unroll
        for (int k = 0; k < 3; ++k)
            set_x(k, ld4<BORDER>(rowp(X0, sp, t0 + k), g.col0, sp.W), ld4<BORDER>(rowp(P0, sp, t0 + k), g.col0, sp.W));
        for (int t = t0; t < t0 + nstep; t += 4) {
            step<0>(t, par);
            step<1>(t + 1, par);
            step<2>(t + 2, par);
            step<3>(t + 3, par);
            par ^= 1u;
        }
    }
};

template <int BW, int PN>
__device__ __forceinline__ void vg4_phase(const StencilParams& sp, const Buffers& b, const PcTaps& T, const Geo& g,
                                          const Ring4& ring, int xcur, int rcur, float alpha, uint32_t& par,
                                          double (&acc)[NSLOT]) {
    const float* X = pick(b.X, xcur);
    const float* P = pick(b.P, xcur);
    const float* Ro = pick(b.R, rcur);
    float* Rn = pick(b.R, rcur ^ 1);
    float ad = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, a_rr = 0.f, a_rro = 0.f;
    if (!g.live) {
    } else if (g.border) {
        VG4<BW, PN, true> v(sp, b, T, g, ring, X, P, Ro, Rn, alpha);
        v.run(par);
        ad = msum(v.accd, g); v0 = msum(v.vb[0], g); v1 = msum(v.vb[1], g); v2 = msum(v.vb[2], g);
        v3 = msum(v.vb[3], g); a_rr = msum(v.rr, g); a_rro = msum(v.rro, g);
    } else {
        VG4<BW, PN, false> v(sp, b, T, g, ring, X, P, Ro, Rn, alpha);
        v.run(par);
        ad = msum(v.accd, g); v0 = msum(v.vb[0], g); v1 = msum(v.vb[1], g); v2 = msum(v.vb[2], g);
        v3 = msum(v.vb[3], g); a_rr = msum(v.rr, g); a_rro = msum(v.rro, g);
    }
    acc[0] = ad;
    acc[1] = sp.gcls[0] * v0 + sp.gcls[1] * v1 + sp.gcls[2] * v2 + sp.gcls[3] * v3;
    acc[2] = a_rr;
    acc[3] = a_rro;
}

// ------------------------------------------------------------------------------------------------
// update x <- x + alpha_upd p, p <- r + beta p, then the exact curvature p^T Hess J p, <p,p>, <p,r>
// at the new (x, p), streaming.  Step t (ring stage = x, p, r(t+3), Y(t+1)): new x/p row t+3 into
// the window (written out if owned); data curvature rho''(z(t+1) - Y) (kappa p)(t+1)^2; BTV curvature
// of the pairs of row t.  t0 = r_lo - 1 is odd.
// ------------------------------------------------------------------------------------------------
template <int BW, int PN, bool BORDER>
struct UC4 {
    float2 XA[4], XB[4], PA[4], PB[4];
    float XM[4], X4[4], X5[4], PM[4], P4[4], P5[4];
    float2 cd, cb[4], pp, mu;
    const float *ix, *ip, *ir, *iy;
    int t0, nstep;
    const StencilParams& sp;
    const Buffers& b;
    const PcTaps& T;
    const Geo& g;
    const Ring4& ring;
    const float *X0, *P0, *R0;
    float *Xn, *Pn;
    float au, be;

    __device__ __forceinline__ UC4(const StencilParams& sp_, const Buffers& b_, const PcTaps& T_, const Geo& g_,
                                   const Ring4& ring_, const float* x, const float* p, const float* r, float* xn,
                                   float* pn, float a, float bb)
        : sp(sp_), b(b_), T(T_), g(g_), ring(ring_), X0(x), P0(p), R0(r), Xn(xn), Pn(pn), au(a), be(bb) {}

    __device__ __forceinline__ void issue(int s, int tt) {
        if (BORDER) {
            const float *a0 = rowp(X0, sp, tt + 3) + g.cbase, *a1 = rowp(P0, sp, tt + 3) + g.cbase;
            const float *a2 = rowp(R0, sp, tt + 3) + g.cbase, *a3 = rowp(b.Y, sp, tt + 1) + g.cbase;
            FL_BCHK(b, a0, SCOLS); FL_BCHK(b, a1, SCOLS); FL_BCHK(b, a2, SCOLS); FL_BCHK(b, a3, SCOLS);
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
        XM[s] = shup(XB[s].y);
        PM[s] = shup(PB[s].y);
        X4[s] = shdn(XA[s].x);
        X5[s] = shdn(XB[s].x);
        P4[s] = shdn(PA[s].x);
        P5[s] = shdn(PB[s].x);
        if (BORDER) {
            if (g.strip0 && g.lane == 0) { XM[s] = XA[s].x; PM[s] = PA[s].x; }
            if (!g.cv4) { X4[s] = X5[s] = XB[s].y; P4[s] = P5[s] = PB[s].y; }
        }
    }

    template <int PH>
    __device__ __forceinline__ void step(int t, uint32_t par) {
        constexpr int s0 = PH, s1 = (PH + 1) & 3, s2 = (PH + 2) & 3, s3 = (PH + 3) & 3;
        constexpr int rho = PH & 1;                     // parity of row t + 1 (t0 odd)
        constexpr int cA = 2 * rho, cB = 2 * rho + 1;
        const float2 e2 = F2(sp.eps2, sp.eps2);
        ring.wait(PH, par);
        set_row(s3, t + 3, fixr<BORDER>(ring.get(PH, 0, g.lane), g), fixr<BORDER>(ring.get(PH, 1, g.lane), g),
                fixr<BORDER>(ring.get(PH, 2, g.lane), g));
        const float4 fy = fixr<BORDER>(ring.get(PH, 3, g.lane), g);
        // data curvature at row t+1: rho''(e) (A p)^2 = eps^2 rs^3 (A p)^2 (eps^2 in the affine term)
        {
            const int tz = t + 1;
            if (tz >= g.r_lo && tz < g.r_hi) {
                float2 zA = F2(0.f, 0.f), zB = zA, aA = zA, aB = zA;
                const int sl[4] = {s0, s1, s2, s3};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int s = sl[j];
                    aA = fmam(TK(cA, j - 1, -1), PM[s], PB[s].x, aA);
                    aA = fma2s(TK(cA, j - 1, 0), PA[s], aA);
                    aA = fma2s(TK(cA, j - 1, 1), PB[s], aA);
                    aA = fmam(TK(cA, j - 1, 2), PA[s].y, P4[s], aA);
                    aB = fma2s(TK(cB, j - 1, -1), PA[s], aB);
                    aB = fma2s(TK(cB, j - 1, 0), PB[s], aB);
                    aB = fmam(TK(cB, j - 1, 1), PA[s].y, P4[s], aB);
                    aB = fmam(TK(cB, j - 1, 2), PB[s].y, P5[s], aB);
                    if (PN != 2) {
                        zA = fmam(TK(cA, j - 1, -1), XM[s], XB[s].x, zA);
                        zA = fma2s(TK(cA, j - 1, 0), XA[s], zA);
                        zA = fma2s(TK(cA, j - 1, 1), XB[s], zA);
                        zA = fmam(TK(cA, j - 1, 2), XA[s].y, X4[s], zA);
                        zB = fma2s(TK(cB, j - 1, -1), XA[s], zB);
                        zB = fma2s(TK(cB, j - 1, 0), XB[s], zB);
                        zB = fmam(TK(cB, j - 1, 1), XA[s].y, X4[s], zB);
                        zB = fmam(TK(cB, j - 1, 2), XB[s].y, X5[s], zB);
                    }
                }
                if (PN == 2) {
                    cd = fma2(aA, aA, cd);
                    cd = fma2(aB, aB, cd);
                } else {
                    const float2 eA = sub2(zA, lo2(fy)), eB = sub2(zB, hi2(fy));
                    const float2 rA = rsq2(fma2(eA, eA, e2)), rB = rsq2(fma2(eB, eB, e2));
                    const float2 uA = mul2(rA, aA), uB = mul2(rB, aB);
                    cd = fma2(mul2(uA, uA), rA, cd);
                    cd = fma2(mul2(uB, uB), rB, cd);
                }
            }
        }
        ring.release();
        if (t + NS4 < t0 + nstep) issue(PH, t + NS4);
        // BTV curvature of the pairs (t, t+d): psi''(D x) (D p)^2 = eps^2 rs^3 (D p)^2
        if (BW > 1 && t >= g.r_lo && t < g.r_hi) {
#pragma unroll
            for (int dy = 0; dy < BW; ++dy) {
                if (BORDER && t + dy >= sp.H) continue;
                const int sq = (PH + dy) & 3;
#pragma unroll
                for (int dx = 0; dx < BW; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    const int cls = dx + dy - 1;
                    const float2 dxA = dx == 0 ? sub2(XA[s0], XA[sq])
                                     : dx == 1 ? sub2(XA[s0], XB[sq])
                                               : F2(XA[s0].x - XA[sq].y, XA[s0].y - X4[sq]);
                    const float2 dxB = dx == 0 ? sub2(XB[s0], XB[sq])
                                     : dx == 1 ? F2(XB[s0].x - XA[sq].y, XB[s0].y - X4[sq])
                                               : F2(XB[s0].x - XB[sq].y, XB[s0].y - X5[sq]);
                    const float2 dpA = dx == 0 ? sub2(PA[s0], PA[sq])
                                     : dx == 1 ? sub2(PA[s0], PB[sq])
                                               : F2(PA[s0].x - PA[sq].y, PA[s0].y - P4[sq]);
                    const float2 dpB = dx == 0 ? sub2(PB[s0], PB[sq])
                                     : dx == 1 ? F2(PB[s0].x - PA[sq].y, PB[s0].y - P4[sq])
                                               : F2(PB[s0].x - PB[sq].y, PB[s0].y - P5[sq]);
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
        }
    }

    __device__ __forceinline__ void run(uint32_t& par) {
        const float2 z = F2(0.f, 0.f);
        cd = pp = mu = z;
#pragma unroll
        for (int c = 0; c < 4; ++c) cb[c] = z;
        t0 = g.r_lo - 1;
        nstep = (g.r_hi - g.r_lo + 1 + 3) / 4 * 4;   // rows r_lo - 1 .. r_hi - 1, rounded up to the unroll
        if (!BORDER) {
            const size_t o = (size_t)(t0 - sp.store_lo) * sp.pitch + g.cbase;
            ix = X0 + o + 3 * (size_t)sp.pitch;
            ip = P0 + o + 3 * (size_t)sp.pitch;
            ir = R0 + o + 3 * (size_t)sp.pitch;
            iy = b.Y + o + (size_t)sp.pitch;
        }
        for (int k = 0; k < NS4 && k < nstep; ++k) issue(k, t0 + k);
#pragma unroll
        for (int k = 0; k < 3; ++k)
            set_row(k, t0 + k, ld4<BORDER>(rowp(X0, sp, t0 + k), g.col0, sp.W),
                    ld4<BORDER>(rowp(P0, sp, t0 + k), g.col0, sp.W), ld4<BORDER>(rowp(R0, sp, t0 + k), g.col0, sp.W));
        for (int t = t0; t < t0 + nstep; t += 4) {
            step<0>(t, par);
            step<1>(t + 1, par);
            step<2>(t + 2, par);
            step<3>(t + 3, par);
            par ^= 1u;
        }
    }
};

template <int BW, int PN>
__device__ __forceinline__ void uc4_phase(const StencilParams& sp, const Buffers& b, const PcTaps& T, const Geo& g,
                                          const Ring4& ring, int xcur, int rcur, float au, float be, uint32_t& par,
                                          double (&acc)[NSLOT]) {
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, a_pp = 0.f, a_mu = 0.f;
    const float* X = pick(b.X, xcur);
    const float* P = pick(b.P, xcur);
    const float* R = pick(b.R, rcur);
    float* Xn = pick(b.X, xcur ^ 1);
    float* Pn = pick(b.P, xcur ^ 1);
    if (!g.live) {
    } else if (g.border) {
        UC4<BW, PN, true> u(sp, b, T, g, ring, X, P, R, Xn, Pn, au, be);
        u.run(par);
        c0 = msum(u.cd, g); c1 = msum(u.cb[0], g); c2 = msum(u.cb[1], g); c3 = msum(u.cb[2], g);
        c4 = msum(u.cb[3], g); a_pp = msum(u.pp, g); a_mu = msum(u.mu, g);
    } else {
        UC4<BW, PN, false> u(sp, b, T, g, ring, X, P, R, Xn, Pn, au, be);
        u.run(par);
        c0 = msum(u.cd, g); c1 = msum(u.cb[0], g); c2 = msum(u.cb[1], g); c3 = msum(u.cb[2], g);
        c4 = msum(u.cb[3], g); a_pp = msum(u.pp, g); a_mu = msum(u.mu, g);
    }
    acc[0] = c0;
    acc[1] = sp.gcls[0] * c1 + sp.gcls[1] * c2 + sp.gcls[2] * c3 + sp.gcls[3] * c4;
    acc[2] = a_pp;
    acc[3] = a_mu;
}

// ---- per-phase kernels (debug entries and the non-persistent fallback; last-CTA reduction) ----
template <int BW, int PN>
__global__ void __launch_bounds__(PC_WPB * 32, 1) k_vg4(const __grid_constant__ StencilParams sp,
                                                           const __grid_constant__ Buffers b,
                                                           const __grid_constant__ PcTaps T, int phase) {
    extern __shared__ __align__(128) unsigned char smem[];
    ScgState* st = b.st;
    if (phase != PH_DEBUG && __shfl_sync(0xffffffffu, st->done, 0)) return;
    const int xcur = __shfl_sync(0xffffffffu, st->xcur, 0);
    const int rcur = __shfl_sync(0xffffffffu, st->rcur, 0);
    const float alpha = phase == PH_ITER ? __shfl_sync(0xffffffffu, st->alpha_f, 0) : 0.0f;
    const Geo g = geometry<H4, PC_WPB>(sp, blockIdx.x);
    Ring4 ring;
    ring.init(smem, __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), g.lane);
    double acc[NSLOT], tot[NSLOT];
    uint32_t par = 0;
    vg4_phase<BW, PN>(sp, b, T, g, ring, xcur, rcur, alpha, par, acc);
    if (reduce_partials(acc, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) finish_scalars<0>(sp, b, tot, phase);
}

template <int BW, int PN>
__global__ void __launch_bounds__(PC_WPB * 32, 1) k_uc4(const __grid_constant__ StencilParams sp,
                                                           const __grid_constant__ Buffers b,
                                                           const __grid_constant__ PcTaps T, int phase) {
    extern __shared__ __align__(128) unsigned char smem[];
    ScgState* st = b.st;
    if (phase != PH_DEBUG) {
        if (__shfl_sync(0xffffffffu, st->done, 0)) return;
        if (!__shfl_sync(0xffffffffu, st->success, 0)) {   // rejected step: delta is reused
            if (blockIdx.x == 0 && threadIdx.x == 0) scg_pre_value(st);
            return;
        }
    }
    const int xcur = __shfl_sync(0xffffffffu, st->xcur, 0);
    const int rcur = __shfl_sync(0xffffffffu, st->rcur, 0);
    const float au = phase == PH_DEBUG ? 0.0f : __shfl_sync(0xffffffffu, st->alpha_upd_f, 0);
    const float be = phase == PH_DEBUG ? 0.0f : __shfl_sync(0xffffffffu, st->beta_f, 0);
    const Geo g = geometry<H4, PC_WPB>(sp, blockIdx.x);
    Ring4 ring;
    ring.init(smem, __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), g.lane);
    double acc[NSLOT], tot[NSLOT];
    uint32_t par = 0;
    uc4_phase<BW, PN>(sp, b, T, g, ring, xcur, rcur, au, be, par, acc);
    if (reduce_partials(acc, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

// ---- the whole SCG loop as one persistent cooperative kernel (as k_scg_loop, flmisr_stream.cu) ----
template <int BW, int PN>
__global__ void __launch_bounds__(PC_WPB * 32, 1) k_scg_loop4(const __grid_constant__ StencilParams sp,
                                                                 const __grid_constant__ Buffers b,
                                                                 const __grid_constant__ PcTaps T) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ ScgState S;
    const Geo g = geometry<H4, PC_WPB>(sp, blockIdx.x);
    Ring4 ring;
    ring.init(smem, __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), g.lane);
    if (threadIdx.x == 0) S = *b.st;
    __syncthreads();
    double* trace = blockIdx.x == 0 ? b.trace : nullptr;
    uint32_t par = 0;
    unsigned epoch = 0;
    double acc[NSLOT], tot[NSLOT];
    auto ui = [](int v) { return __shfl_sync(0xffffffffu, v, 0); };
    auto uf = [](float v) { return __shfl_sync(0xffffffffu, v, 0); };
    for (int pass = 0; !ui(S.done); ++pass) {
        if (pass > 0) {
            if (ui(S.success)) {
                uc4_phase<BW, PN>(sp, b, T, g, ring, ui(S.xcur), ui(S.rcur), uf(S.alpha_upd_f), uf(S.beta_f), par, acc);
                grid_sum_fx(acc, b.part, b.gbar, epoch++, tot);
                if (threadIdx.x == 0) {
                    S.xcur ^= 1;
                    affine<1>(sp, tot);
                    scg_after_curv(&S, tot);
                }
            } else if (threadIdx.x == 0) {   // rejected step: delta is reused
                scg_pre_value(&S);
            }
            __syncthreads();
            if (ui(S.done)) break;
        }
        vg4_phase<BW, PN>(sp, b, T, g, ring, ui(S.xcur), ui(S.rcur), pass > 0 ? uf(S.alpha_f) : 0.0f, par, acc);
        grid_sum_fx(acc, b.part, b.gbar, epoch++, tot);
        if (threadIdx.x == 0) {
            affine<0>(sp, tot);
            scg_after_value(&S, tot, trace, pass > 0 ? PH_ITER : PH_INIT);
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *b.st = S;
}

// ---- debug operators (natural layout, per pixel; FORWARD / ADJOINT parity entries) ----
__device__ __forceinline__ int pc_cls(int u, int v) { return 2 * (u & 1) + (v & 1); }

// z(u) = sum_PQ kappa_{c(u)}(P,Q) x~(u + (P,Q)), clamped reads (reading 4)
__global__ void k_pc_forward(StencilParams sp, PcTaps T, const float* __restrict__ x, float* __restrict__ z) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)sp.H * sp.W) return;
    const int u = (int)(i / sp.W), v = (int)(i - (long long)u * sp.W);
    const int c = pc_cls(u, v);
    float acc = 0.0f;
    for (int P = -1; P <= 2; ++P)
        for (int Q = -1; Q <= 2; ++Q)
            acc = fmaf(T.k[c][(P + 1) * 4 + (Q + 1)],
                       x[(size_t)clampi(u + P, 0, sp.H - 1) * sp.pitch + clampi(v + Q, 0, sp.W - 1)], acc);
    z[(size_t)u * sp.pitch + v] = acc;
}

// g(v) = sum over the virtual positions v' that clamp to v, sum_PQ kappa_{c(u)}(P,Q) w(u), u = v' - (P,Q)
__global__ void k_pc_adjoint(StencilParams sp, PcTaps T, const float* __restrict__ w, float* __restrict__ g) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)sp.H * sp.W) return;
    const int vy = (int)(i / sp.W), vx = (int)(i - (long long)vy * sp.W);
    const int ylo = vy == 0 ? -1 : vy, yhi = vy == sp.H - 1 ? sp.H + 1 : vy;
    const int xlo = vx == 0 ? -1 : vx, xhi = vx == sp.W - 1 ? sp.W + 1 : vx;
    float acc = 0.0f;
    for (int yy = ylo; yy <= yhi; ++yy)
        for (int xx = xlo; xx <= xhi; ++xx)
            for (int P = -1; P <= 2; ++P)
                for (int Q = -1; Q <= 2; ++Q) {
                    const int uy = yy - P, ux = xx - Q;
                    if (uy < 0 || uy >= sp.H || ux < 0 || ux >= sp.W) continue;
                    acc = fmaf(T.k[pc_cls(uy, ux)][(P + 1) * 4 + (Q + 1)], w[(size_t)uy * sp.pitch + ux], acc);
                }
    g[(size_t)vy * sp.pitch + vx] = acc;
}

template <typename K>
cudaError_t set_smem(K kernel) {
    return ensure_dyn_smem(reinterpret_cast<const void*>(kernel), RING4_SMEM);
}

template <typename K, typename... A>
cudaError_t launch4(K kernel, bool coop, int nw, cudaStream_t s, A... args) {
    cudaError_t e = set_smem(kernel);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((nw + PC_WPB - 1) / PC_WPB);
    cfg.blockDim = dim3(PC_WPB * 32);
    cfg.dynamicSmemBytes = RING4_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // the loop kernel's grid barrier: every CTA co-resident
    attr[0].val.cooperative = coop ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

#define FL_PC_CASES(MACRO) MACRO(1, 1) MACRO(1, 2) MACRO(2, 1) MACRO(2, 2) MACRO(3, 1) MACRO(3, 2)

cudaError_t launch_pc_vg(int bw, int pn, const StencilParams& sp, const Buffers& b, const PcTaps& T, int phase,
                         cudaStream_t s) {
    switch (bw * 10 + pn) {
#define FL_C(BW_, PN_) \
    case BW_ * 10 + PN_: return launch4(k_vg4<BW_, PN_>, false, sp.nitems, s, sp, b, T, phase);
        FL_PC_CASES(FL_C)
#undef FL_C
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_pc_uc(int bw, int pn, const StencilParams& sp, const Buffers& b, const PcTaps& T, int phase,
                         cudaStream_t s) {
    switch (bw * 10 + pn) {
#define FL_C(BW_, PN_) \
    case BW_ * 10 + PN_: return launch4(k_uc4<BW_, PN_>, false, sp.nitems, s, sp, b, T, phase);
        FL_PC_CASES(FL_C)
#undef FL_C
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_pc_loop(int bw, int pn, const StencilParams& sp, const Buffers& b, const PcTaps& T,
                           cudaStream_t s) {
    switch (bw * 10 + pn) {
#define FL_C(BW_, PN_) \
    case BW_ * 10 + PN_: return launch4(k_scg_loop4<BW_, PN_>, true, sp.nitems, s, sp, b, T);
        FL_PC_CASES(FL_C)
#undef FL_C
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_pc_forward_debug(const StencilParams& sp, const PcTaps& T, const float* x, float* z, cudaStream_t s) {
    const long long n = (long long)sp.H * sp.W;
    k_pc_forward<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sp, T, x, z);
    return cudaGetLastError();
}

cudaError_t launch_pc_adjoint_debug(const StencilParams& sp, const PcTaps& T, const float* w, float* g, cudaStream_t s) {
    const long long n = (long long)sp.H * sp.W;
    k_pc_adjoint<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sp, T, w, g);
    return cudaGetLastError();
}

}  // namespace flmisr
