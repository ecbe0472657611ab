// flmisr_stream.cu -- register-streaming sm_100a kernels for the FL-MISR SCG hot path when the
// composed kernel kappa is separable (kappa(P,Q) = a(P) b(Q): every Gaussian PSF) and KR <= 1
// (PSF up to 3x3 with integer HR phases) -- this covers all BASELINE configs.
//
// Work decomposition: one warp owns a strip of 128 HR columns (4 per lane,
// float4 I/O) and a segment of S rows, and streams down the rows with 3-row register windows
// (x' = x + alpha p, the horizontal kappa pass of x', pending rows of -grad J).  Horizontal
// neighbours move by warp shuffles; strips overlap by SHALO = 2 columns per side (the reach of the
// fused operator: 2 KR for the data term's forward+adjoint chain, w-1 for BTV), so no shared
// memory is needed.  Each BTV pair (u, u+d) is evaluated once and its psi' goes to both endpoints
// (pending rows below, the right lane for columns to the right) -> 8 rsqrt per pixel.  The data
// gradient is scattered the same way (adjoint = transposed correlation, P:251 A^T).
// Image borders (clamped forward reads, folded adjoint, valid-pairs-only BTV; readings 4, 5) run in
// a separate instantiation selected per warp (warp-uniform), so interior warps carry no masks.
// Constant terms (eps of every Charbonnier term, eps^2 of rho''/psi'') are hoisted into the affine
// correction of the CTA sums (StencilParams::aff_*).
#include <cstdint>
#include <cuda_runtime.h>

#include "flmisr_common.cuh"
#include "flmisr_internal.h"

namespace flmisr {
namespace {

constexpr int SWPB = 8;   // warps per CTA

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

template <bool BORDER>
__device__ __forceinline__ float4 ld4(const float* rp, int col, int W) {
    if (!BORDER || col + 3 < W) return __ldg(reinterpret_cast<const float4*>(rp + col));
    // right image border (W % 4 == 0): a chunk is either inside or wholly outside -> replicate col W-1
    float v = __ldg(rp + (W - 1));
    return make_float4(v, v, v, v);
}

__device__ __forceinline__ void st4(float* rp, int col, float a, float b, float c, float d, bool full,
                                    const bool (&m)[4]) {
    if (full) {
        *reinterpret_cast<float4*>(rp + col) = make_float4(a, b, c, d);
    } else {
        if (m[0]) rp[col] = a;
        if (m[1]) rp[col + 1] = b;
        if (m[2]) rp[col + 2] = c;
        if (m[3]) rp[col + 3] = d;
    }
}

struct Geo {
    int lane, col0, r_lo, r_hi, w_lo, w_hi;
    bool strip0, live, full, border;
    bool outc[4];   // this lane's column j is an output column of the strip
    bool cv[6];     // column col0 + j (j = 0..5) lies inside the image
};

__device__ __forceinline__ Geo geometry(const StencilParams& sp) {
    Geo g;
    const int warp = threadIdx.x >> 5;
    g.lane = threadIdx.x & 31;
    const int gw = blockIdx.x * SWPB + warp;
    g.live = gw < sp.nstrips * sp.nsegs;
    const int strip = g.live ? gw % sp.nstrips : 0, seg = g.live ? gw / sp.nstrips : 0;
    const int cbase = strip * SSTEP;
    g.col0 = cbase + 4 * g.lane;
    g.strip0 = strip == 0;
    const int oc_lo = g.strip0 ? 0 : cbase + SHALO;
    const int oc_hi = (strip == sp.nstrips - 1) ? sp.W : min(cbase + SCOLS - SHALO, sp.W);
    g.full = true;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        g.outc[j] = g.live && g.col0 + j >= oc_lo && g.col0 + j < oc_hi;
        g.full = g.full && g.outc[j];
    }
#pragma unroll
    for (int j = 0; j < 6; ++j) g.cv[j] = g.col0 + j < sp.W;
    g.r_lo = sp.row_lo + seg * sp.seg_rows;
    g.r_hi = min(g.r_lo + sp.seg_rows, sp.row_hi);
    if (!g.live) g.r_hi = g.r_lo;
    // rows whose new x/p this segment writes: owned rows, plus the band's halo rows for the first /
    // last segment of a band with a neighbour on that side (bit-identical to the neighbour's owned
    // rows: same inputs, same fp32 operations)
    g.w_lo = g.r_lo;
    g.w_hi = g.r_hi;
    if (g.live && seg == 0 && sp.row_lo > 0) g.w_lo = sp.store_lo;
    if (g.live && seg == sp.nsegs - 1 && sp.row_hi < sp.H) g.w_hi = sp.store_hi;
    g.border = g.strip0 || cbase + SCOLS > sp.W || g.r_lo < 3 || g.r_hi > sp.H - 3;
    return g;
}

__device__ __forceinline__ float shup(float v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ float shdn(float v) { return __shfl_down_sync(0xffffffffu, v, 1); }

// ------------------------------------------------------------------------------------------------
// value + gradient at x' = x + alpha p (Alg. 1 lines 14-19), streaming.
//   step t: x'(t+2) -> HZ(t+2); w(t+1) = rho'(kappa x' - Y) -> horizontal adjoint pass hw(t+1),
//   scattered into the pending rows t, t+1, t+2 of r = -grad J; BTV pairs of row t scattered into
//   rows t..t+2; row t is then complete and stored.
// ------------------------------------------------------------------------------------------------
template <int BW, int PN, bool BORDER>
struct VG {
    float X[3][6];    // x' at columns 0 .. 5 relative to col0 (rows t, t+1, t+2 in slots (t+k)%3)
    float HZ[3][4];   // horizontal kappa pass of x'
    float G[3][6];    // pending r = -grad J of rows t, t+1, t+2 at columns 0 .. 5
    float4 fx, fp, fy, fr;   // prefetched rows: x/p (t+2), Y (t+1), r_old (t)
    float acc_d, vb[4], rr, rro;

    const StencilParams& sp;
    const Buffers& b;
    const Geo& g;
    const float* X0;
    const float* P0;
    const float* Rold;
    float* Rnew;
    float alpha;

    __device__ __forceinline__ VG(const StencilParams& sp_, const Buffers& b_, const Geo& g_, const float* x,
                                  const float* p, const float* ro, float* rn, float al)
        : sp(sp_), b(b_), g(g_), X0(x), P0(p), Rold(ro), Rnew(rn), alpha(al) {}

    __device__ __forceinline__ void load_xp(int row, float4& xv, float4& pv) {
        xv = ld4<BORDER>(rowp(X0, sp, row), g.col0, sp.W);
        pv = ld4<BORDER>(rowp(P0, sp, row), g.col0, sp.W);
    }

    // x'(row) into slot s, right neighbours, and the horizontal kappa pass
    __device__ __forceinline__ void set_x(int s, const float4& xv, const float4& pv) {
        X[s][0] = fmaf(alpha, pv.x, xv.x);
        X[s][1] = fmaf(alpha, pv.y, xv.y);
        X[s][2] = fmaf(alpha, pv.z, xv.z);
        X[s][3] = fmaf(alpha, pv.w, xv.w);
        float xm1 = shup(X[s][3]);
        X[s][4] = shdn(X[s][0]);
        X[s][5] = shdn(X[s][1]);
        if (BORDER) {
            if (g.strip0 && g.lane == 0) xm1 = X[s][0];                  // clamp at column 0
            if (!g.cv[4]) { X[s][4] = X[s][3]; X[s][5] = X[s][3]; }      // clamp at column W-1
        }
        HZ[s][0] = fmaf(sp.kb[0], xm1, fmaf(sp.kb[1], X[s][0], sp.kb[2] * X[s][1]));
#pragma unroll
        for (int j = 1; j < 4; ++j)
            HZ[s][j] = fmaf(sp.kb[0], X[s][j - 1], fmaf(sp.kb[1], X[s][j], sp.kb[2] * X[s][j + 1]));
    }

    template <int PH>
    __device__ __forceinline__ void step(int t) {
        constexpr int s0 = PH % 3, s1 = (PH + 1) % 3, sa = (PH + 2) % 3;
        const float eps2 = sp.eps2;
        // A: x'(t+2) from the prefetch, then prefetch x/p(t+3)
        set_x(sa, fx, fp);
        load_xp(t + 3, fx, fp);

        // B: w(t+1) = rho'(z - Y), data value, adjoint (transposed kappa) scattered into rows t..t+2
        {
            const int tw = t + 1;
            float w[4];
            const float yv[4] = {fy.x, fy.y, fy.z, fy.w};
            fy = ld4<BORDER>(rowp(b.Y, sp, t + 2), g.col0, sp.W);
            const bool orow = tw >= g.r_lo && tw < g.r_hi;
            const bool vrow = !BORDER || (tw >= 0 && tw < sp.H);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float z = fmaf(sp.ka[0], HZ[s0][j], fmaf(sp.ka[1], HZ[s1][j], sp.ka[2] * HZ[sa][j]));
                float e = z - yv[j];
                float vr, wj;
                if (PN == 2) {
                    vr = e * e;
                    wj = 2.0f * e;
                } else {
                    float q = fmaf(e, e, eps2);
                    float rs = rsqrtf(q);
                    vr = q * rs;          // rho + eps (eps * N is subtracted by the affine correction)
                    wj = e * rs;
                }
                if (orow && g.outc[j]) acc_d += vr;
                if (BORDER && !(vrow && g.cv[j])) wj = 0.0f;   // zero-padded adjoint outside the image
                w[j] = wj;
            }
            float wm1 = shup(w[3]), w4 = shdn(w[0]);
            if (BORDER) {
                if (g.strip0 && g.lane == 0) wm1 = 0.0f;
                if (!g.cv[4]) w4 = 0.0f;
            }
            float hw[4];
            hw[0] = fmaf(sp.kb[0], w[1], fmaf(sp.kb[1], w[0], sp.kb[2] * wm1));
            hw[1] = fmaf(sp.kb[0], w[2], fmaf(sp.kb[1], w[1], sp.kb[2] * w[0]));
            hw[2] = fmaf(sp.kb[0], w[3], fmaf(sp.kb[1], w[2], sp.kb[2] * w[1]));
            hw[3] = fmaf(sp.kb[0], w4, fmaf(sp.kb[1], w[3], sp.kb[2] * w[2]));
            if (BORDER) {   // fold the clamped columns back onto the edge pixels (adjoint of clamp)
                if (g.strip0 && g.lane == 0) hw[0] = fmaf(sp.kb[0], w[0], hw[0]);
                if (g.cv[3] && !g.cv[4]) hw[3] = fmaf(sp.kb[2], w[3], hw[3]);
            }
            // g(v) = sum_P a(P) hw(v - P): hw(t+1) feeds rows t (P=-1), t+1 (P=0), t+2 (P=+1)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                G[s0][j] = fmaf(-sp.ka[0], hw[j], G[s0][j]);
                G[s1][j] = fmaf(-sp.ka[1], hw[j], G[s1][j]);
                G[sa][j] = fmaf(-sp.ka[2], hw[j], G[sa][j]);
            }
            if (BORDER) {   // fold the clamped rows: row -1 onto row 0, row H onto row H-1
                if (tw == 0)
#pragma unroll
                    for (int j = 0; j < 4; ++j) G[s1][j] = fmaf(-sp.ka[0], hw[j], G[s1][j]);
                if (tw == sp.H - 1)
#pragma unroll
                    for (int j = 0; j < 4; ++j) G[s1][j] = fmaf(-sp.ka[2], hw[j], G[s1][j]);
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
                    const float lg = sp.lam * sp.gam[dy * MAXBW + dx];
                    const int cls = dx + dy - 1;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float d = X[s0][j] - X[sq][j + dx];
                        float q = fmaf(d, d, eps2);
                        float rs = rsqrtf(q);
                        float u = d * rs;
                        if (BORDER && !g.cv[j + dx]) u = 0.0f;
                        if (orow && g.outc[j] && (!BORDER || g.cv[j + dx])) vb[cls] = fmaf(q, rs, vb[cls]);
                        G[s0][j] = fmaf(-lg, u, G[s0][j]);
                        G[sq][j + dx] = fmaf(lg, u, G[sq][j + dx]);
                    }
                }
            }
        }

        // E: row t is complete once the right-spilled columns of the left lane arrive
        {
            float c4 = shup(G[s0][4]), c5 = shup(G[s0][5]);
            if (g.lane > 0) {
                G[s0][0] += c4;
                G[s0][1] += c5;
            }
            const float ro[4] = {fr.x, fr.y, fr.z, fr.w};
            fr = ld4<BORDER>(rowp(Rold, sp, t + 1), g.col0, sp.W);
            if (orow) {
                float* rp = Rnew + (size_t)(t - sp.store_lo) * sp.pitch;
                st4(rp, g.col0, G[s0][0], G[s0][1], G[s0][2], G[s0][3], g.full, g.outc);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (g.outc[j]) {
                        rr = fmaf(G[s0][j], G[s0][j], rr);
                        rro = fmaf(G[s0][j], ro[j], rro);
                    }
                }
                // band mode: owned boundary rows of the candidate go to the neighbours
                if (b.send_top && t - sp.row_lo < b.eta)
                    st4(b.send_top + (size_t)(t - sp.row_lo) * sp.pitch, g.col0, G[s0][0], G[s0][1], G[s0][2],
                        G[s0][3], g.full, g.outc);
                if (b.send_bot && sp.row_hi - 1 - t < b.eta)
                    st4(b.send_bot + (size_t)(t - (sp.row_hi - b.eta)) * sp.pitch, g.col0, G[s0][0], G[s0][1],
                        G[s0][2], G[s0][3], g.full, g.outc);
            }
#pragma unroll
            for (int j = 0; j < 6; ++j) G[s0][j] = 0.0f;
        }
    }

    __device__ __forceinline__ void run() {
        acc_d = 0.f; rr = 0.f; rro = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) vb[c] = 0.f;
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int j = 0; j < 6; ++j) G[s][j] = 0.f;
        const int t0 = g.r_lo - 2;
        float4 xv, pv;
        load_xp(t0, xv, pv);
        set_x(0, xv, pv);
        load_xp(t0 + 1, xv, pv);
        set_x(1, xv, pv);
        load_xp(t0 + 2, fx, fp);
        fy = ld4<BORDER>(rowp(b.Y, sp, t0 + 1), g.col0, sp.W);
        fr = ld4<BORDER>(rowp(Rold, sp, t0), g.col0, sp.W);
        const int nstep = sp.seg_rows + 2;   // multiple of 3 (seg_rows = 1 mod 3)
        for (int t = t0; t < t0 + nstep; t += 3) {
            step<0>(t);
            step<1>(t + 1);
            step<2>(t + 2);
        }
    }
};

template <int BW, int PN>
__global__ void __launch_bounds__(SWPB * 32, 2) k_vg_stream(StencilParams sp, Buffers b, int phase) {
    ScgState* st = b.st;
    if (phase != PH_DEBUG && st->done) return;
    const int xcur = st->xcur, rcur = st->rcur;
    const float alpha = (phase == PH_ITER) ? st->alpha_f : 0.0f;
    const Geo g = geometry(sp);
    double acc[NSLOT];
    {
        const float* X = pick(b.X, xcur);
        const float* P = pick(b.P, xcur);
        const float* Ro = pick(b.R, rcur);
        float* Rn = pick(b.R, rcur ^ 1);
        float ad = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, a_rr = 0.f, a_rro = 0.f;
        if (!g.live) {
        } else if (g.border) {
            VG<BW, PN, true> v(sp, b, g, X, P, Ro, Rn, alpha);
            v.run();
            ad = v.acc_d; v0 = v.vb[0]; v1 = v.vb[1]; v2 = v.vb[2]; v3 = v.vb[3]; a_rr = v.rr; a_rro = v.rro;
        } else {
            VG<BW, PN, false> v(sp, b, g, X, P, Ro, Rn, alpha);
            v.run();
            ad = v.acc_d; v0 = v.vb[0]; v1 = v.vb[1]; v2 = v.vb[2]; v3 = v.vb[3]; a_rr = v.rr; a_rro = v.rro;
        }
        acc[0] = ad;
        acc[1] = sp.gcls[0] * v0 + sp.gcls[1] * v1 + sp.gcls[2] * v2 + sp.gcls[3] * v3;
        acc[2] = a_rr;
        acc[3] = a_rro;
    }
    double tot[NSLOT];
    if (reduce_partials(acc, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) finish_scalars<0>(sp, b, tot, phase);
}

// ------------------------------------------------------------------------------------------------
// update x <- x + alpha_upd p, p <- r + beta p (Alg. 1 lines 14, 20), then the exact curvature
// p^T Hess J p, <p,p>, <p,r> at the new (x, p) (lines 6-12; reading 16), streaming.
// ------------------------------------------------------------------------------------------------
template <int BW, int PN, bool BORDER>
struct UC {
    float XN[3][6], PN_[3][6];
    float HX[3][4], HP[3][4];
    float4 fx, fp, fr, fy;   // prefetched: x/p/r rows (t+2), Y (t+1)
    float cd, cb[4], pp, mu;
    const StencilParams& sp;
    const Buffers& b;
    const Geo& g;
    const float *X0, *P0, *R0;
    float *Xn, *Pn;
    float au, be;

    __device__ __forceinline__ UC(const StencilParams& sp_, const Buffers& b_, const Geo& g_, const float* x,
                                  const float* p, const float* r, float* xn, float* pn, float a, float bb)
        : sp(sp_), b(b_), g(g_), X0(x), P0(p), R0(r), Xn(xn), Pn(pn), au(a), be(bb) {}

    __device__ __forceinline__ void load(int row, float4& xv, float4& pv, float4& rv) {
        xv = ld4<BORDER>(rowp(X0, sp, row), g.col0, sp.W);
        pv = ld4<BORDER>(rowp(P0, sp, row), g.col0, sp.W);
        rv = ld4<BORDER>(rrowp(b, R0, sp, row), g.col0, sp.W);
    }

    __device__ __forceinline__ void set_row(int s, int row, const float4& xv, const float4& pv, const float4& rv) {
        const float xo[4] = {xv.x, xv.y, xv.z, xv.w}, po[4] = {pv.x, pv.y, pv.z, pv.w};
        const float ro[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            XN[s][j] = fmaf(au, po[j], xo[j]);
            PN_[s][j] = fmaf(be, po[j], ro[j]);
        }
        if (row >= g.w_lo && row < g.w_hi) {
            const size_t off = (size_t)(row - sp.store_lo) * sp.pitch;
            st4(Xn + off, g.col0, XN[s][0], XN[s][1], XN[s][2], XN[s][3], g.full, g.outc);
            st4(Pn + off, g.col0, PN_[s][0], PN_[s][1], PN_[s][2], PN_[s][3], g.full, g.outc);
            if (row >= g.r_lo && row < g.r_hi) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (g.outc[j]) {
                        pp = fmaf(PN_[s][j], PN_[s][j], pp);
                        mu = fmaf(PN_[s][j], ro[j], mu);
                    }
                }
            }
        }
        float xm1 = shup(XN[s][3]), pm1 = shup(PN_[s][3]);
        XN[s][4] = shdn(XN[s][0]);
        XN[s][5] = shdn(XN[s][1]);
        PN_[s][4] = shdn(PN_[s][0]);
        PN_[s][5] = shdn(PN_[s][1]);
        if (BORDER) {
            if (g.strip0 && g.lane == 0) { xm1 = XN[s][0]; pm1 = PN_[s][0]; }
            if (!g.cv[4]) { XN[s][4] = XN[s][5] = XN[s][3]; PN_[s][4] = PN_[s][5] = PN_[s][3]; }
        }
        HX[s][0] = fmaf(sp.kb[0], xm1, fmaf(sp.kb[1], XN[s][0], sp.kb[2] * XN[s][1]));
        HP[s][0] = fmaf(sp.kb[0], pm1, fmaf(sp.kb[1], PN_[s][0], sp.kb[2] * PN_[s][1]));
#pragma unroll
        for (int j = 1; j < 4; ++j) {
            HX[s][j] = fmaf(sp.kb[0], XN[s][j - 1], fmaf(sp.kb[1], XN[s][j], sp.kb[2] * XN[s][j + 1]));
            HP[s][j] = fmaf(sp.kb[0], PN_[s][j - 1], fmaf(sp.kb[1], PN_[s][j], sp.kb[2] * PN_[s][j + 1]));
        }
    }

    template <int PH>
    __device__ __forceinline__ void step(int t) {
        constexpr int s0 = PH % 3, s1 = (PH + 1) % 3, sa = (PH + 2) % 3;
        const float eps2 = sp.eps2;
        set_row(sa, t + 2, fx, fp, fr);
        load(t + 3, fx, fp, fr);
        // data curvature at row t+1: rho''(e) (A p)^2 = eps^2 rs^3 (A p)^2 (eps^2 in the affine term)
        {
            const int tz = t + 1;
            const float yv[4] = {fy.x, fy.y, fy.z, fy.w};
            fy = ld4<BORDER>(rowp(b.Y, sp, t + 2), g.col0, sp.W);
            if (tz >= g.r_lo && tz < g.r_hi) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float ap = fmaf(sp.ka[0], HP[s0][j], fmaf(sp.ka[1], HP[s1][j], sp.ka[2] * HP[sa][j]));
                    if (PN == 2) {
                        if (g.outc[j]) cd = fmaf(ap, ap, cd);
                    } else {
                        float z = fmaf(sp.ka[0], HX[s0][j], fmaf(sp.ka[1], HX[s1][j], sp.ka[2] * HX[sa][j]));
                        float e = z - yv[j];
                        float rs = rsqrtf(fmaf(e, e, eps2));
                        float u = rs * ap;
                        if (g.outc[j]) cd = fmaf(u * u, rs, cd);
                    }
                }
            }
        }
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
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float dxv = XN[s0][j] - XN[sq][j + dx];
                        float dpv = PN_[s0][j] - PN_[sq][j + dx];
                        float rs = rsqrtf(fmaf(dxv, dxv, eps2));
                        float u = rs * dpv;
                        if (g.outc[j] && (!BORDER || g.cv[j + dx])) cb[cls] = fmaf(u * u, rs, cb[cls]);
                    }
                }
            }
        }
    }

    __device__ __forceinline__ void run() {
        cd = 0.f; pp = 0.f; mu = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) cb[c] = 0.f;
        const int t0 = g.r_lo - 2;
        float4 xv, pv, rv;
        load(t0, xv, pv, rv);
        set_row(0, t0, xv, pv, rv);
        load(t0 + 1, xv, pv, rv);
        set_row(1, t0 + 1, xv, pv, rv);
        load(t0 + 2, fx, fp, fr);
        fy = ld4<BORDER>(rowp(b.Y, sp, t0 + 1), g.col0, sp.W);
        const int nstep = sp.seg_rows + 2;
        for (int t = t0; t < t0 + nstep; t += 3) {
            step<0>(t);
            step<1>(t + 1);
            step<2>(t + 2);
        }
    }
};

template <int BW, int PN>
__global__ void __launch_bounds__(SWPB * 32, 2) k_uc_stream(StencilParams sp, Buffers b, int phase) {
    ScgState* st = b.st;
    if (phase != PH_DEBUG) {
        if (st->done) return;
        if (!st->success) {   // rejected step: delta is reused, only the scalar pre-value step runs
            if (sp.world == 1 && blockIdx.x == 0 && threadIdx.x == 0) scg_pre_value(st);
            return;
        }
    }
    const int xcur = st->xcur, rcur = st->rcur;
    const float au = (phase == PH_DEBUG) ? 0.0f : st->alpha_upd_f;
    const float be = (phase == PH_DEBUG) ? 0.0f : st->beta_f;
    const Geo g = geometry(sp);
    double acc[NSLOT];
    {
        float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f, c4 = 0.f, a_pp = 0.f, a_mu = 0.f;
        if (!g.live) {
        } else if (g.border) {
            UC<BW, PN, true> u(sp, b, g, pick(b.X, xcur), pick(b.P, xcur), pick(b.R, rcur), pick(b.X, xcur ^ 1), pick(b.P, xcur ^ 1), au, be);
            u.run();
            c0 = u.cd; c1 = u.cb[0]; c2 = u.cb[1]; c3 = u.cb[2]; c4 = u.cb[3]; a_pp = u.pp; a_mu = u.mu;
        } else {
            UC<BW, PN, false> u(sp, b, g, pick(b.X, xcur), pick(b.P, xcur), pick(b.R, rcur), pick(b.X, xcur ^ 1), pick(b.P, xcur ^ 1), au, be);
            u.run();
            c0 = u.cd; c1 = u.cb[0]; c2 = u.cb[1]; c3 = u.cb[2]; c4 = u.cb[3]; a_pp = u.pp; a_mu = u.mu;
        }
        acc[0] = c0;
        acc[1] = sp.gcls[0] * c1 + sp.gcls[1] * c2 + sp.gcls[2] * c3 + sp.gcls[3] * c4;
        acc[2] = a_pp;
        acc[3] = a_mu;
    }
    double tot[NSLOT];
    if (reduce_partials(acc, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

}  // namespace

#define FL_SCASE(K, BW_, PN_) \
    case BW_ * 10 + PN_: K<BW_, PN_><<<grid, SWPB * 32, 0, s>>>(sp, b, phase); break;

cudaError_t launch_value_grad_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                                     cudaStream_t s) {
    const int nw = sp.nstrips * sp.nsegs;
    dim3 grid((nw + SWPB - 1) / SWPB);
    switch (bw * 10 + pn) {
        FL_SCASE(k_vg_stream, 1, 1) FL_SCASE(k_vg_stream, 1, 2) FL_SCASE(k_vg_stream, 2, 1)
        FL_SCASE(k_vg_stream, 2, 2) FL_SCASE(k_vg_stream, 3, 1) FL_SCASE(k_vg_stream, 3, 2)
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_update_curv_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                                      cudaStream_t s) {
    const int nw = sp.nstrips * sp.nsegs;
    dim3 grid((nw + SWPB - 1) / SWPB);
    switch (bw * 10 + pn) {
        FL_SCASE(k_uc_stream, 1, 1) FL_SCASE(k_uc_stream, 1, 2) FL_SCASE(k_uc_stream, 2, 1)
        FL_SCASE(k_uc_stream, 2, 2) FL_SCASE(k_uc_stream, 3, 1) FL_SCASE(k_uc_stream, 3, 2)
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace flmisr
