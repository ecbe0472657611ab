// flmisr_general3.cu -- fused tiled kernels of the general-geometry path, the
// hot loop whenever every frame's integer HR phase lies in [-(R+1), mag-1+R] on both axes
// (GenParams::fused; the kernels of flmisr_general.cu cover everything else).  One kernel per SCG
// phase, no rho' round trip through HBM:
//   k_gen3_vg: an HR tile of G3Y x G3X output pixels stages x' = x + alpha p over the tile and a
//     G3<R,MAG>::H-pixel halo (clamped reads, so the staged halo holds x~ at every virtual position
//     a forward sample of the tile's LR windows reads), then, G3FC frames at a time, evaluates
//     w = rho'(A_i x' - y_i) over the LR window of each frame whose clamped footprint reaches the tile
//     (zero outside the frame) into shared memory and gathers the exact transpose A_i^T w from it:
//     for mag | 4 a thread's pixels (one column, rows 4 apart) share one residue class per frame,
//     so the taps sit in registers and every window read is a compile-time offset; image-border
//     pixels walk their virtual positions (clamp folds).  BTV gradient and value from the staged
//     tile.  Reads x, p, r_old, y once (+ halo), writes r'.
//   k_gen3_uc: stages x_new = x + a p and p_new = r + b p over the tile + halo, writes the owned
//     pixels, and accumulates the BTV curvature, <p,p>, <p,r> and the data curvature
//     rho''(e) (A_i p)^2 of every LR pixel the tile owns (the tile holding its clamped anchor
//     (mag a + s_iy, mag b + s_ix): each LR pixel is counted exactly once).
// Operator definitions: eq:sisr, eq:prior, eq:objective;
// readings 4, 5, 19 of DESIGN.md section 3.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "flmisr_common.cuh"
#include "flmisr_internal.h"

namespace flmisr {
namespace {

constexpr int G3X = 64, G3Y = 32, G3T = 256, G3FC = 4;
// resident CTAs per SM the fused kernels are compiled for (measured on G3: value+gradient 0.67 ms at 3
// vs 0.72 at 4, and G3 53.8 proj/s at 3 vs 50.7 at 2 (profiles/r01_g3_minblocks_ab.txt); update+curvature
// 0.32 at 3 vs 0.30 at 4)
#ifndef FLMISR_G3MINB_VG
#define FLMISR_G3MINB_VG 3
#endif
#ifndef FLMISR_G3MINB_UC
#define FLMISR_G3MINB_UC 4
#endif
constexpr int G3MINB_VG = FLMISR_G3MINB_VG, G3MINB_UC = FLMISR_G3MINB_UC;   // tuning builds override
constexpr int G3PPT = G3X * G3Y / G3T;   // 8 output pixels per thread: column t % 64, rows t / 64 + 4 k

__device__ __forceinline__ int fdiv(int a, int m) { return a >= 0 ? a / m : -((-a + m - 1) / m); }
__device__ __forceinline__ int cdiv(int a, int m) { return -fdiv(-a, m); }
// floor / ceil division by the compile-time magnification: an arithmetic shift when MAG is a power of two
__host__ __device__ constexpr int ilog2c(int m) { return m <= 1 ? 0 : 1 + ilog2c(m / 2); }
template <int M>
__device__ __forceinline__ int fdivc(int a) {
    if constexpr ((M & (M - 1)) == 0) return a >> ilog2c(M);
    else return fdiv(a, M);
}
template <int M>
__device__ __forceinline__ int cdivc(int a) { return -fdivc<M>(-a); }
__device__ __forceinline__ int pmod(int a, int m) { return ((a % m) + m) % m; }

template <int R, int MAG>
struct G3 {
    static constexpr int KD = 2 * R + 2;                          // kappa offsets [-R, R+1]
    static constexpr int H = (2 * R + 1 > 2) ? 2 * R + 1 : 2;     // halo: forward + adjoint reach, BTV
    static constexpr int CL = (H + 3) / 4 * 4;                    // column halo rounded to 16 B (float4 staging)
    static constexpr int XR = G3Y + 2 * H, XC = G3X + 2 * CL;     // staged tile: rows ty0-H.., cols tx0-CL..
    static constexpr int WR = (G3Y + 2 * H + 2 * R) / MAG + 2;    // LR window bound (incl. border folds)
    static constexpr int WC = (G3X + 2 * H + 2 * R) / MAG + 2;
    static constexpr int NT = (KD + MAG - 1) / MAG;               // taps per axis in one residue class
    static constexpr size_t smem_vg(int k) {
        return ((size_t)XR * XC + (size_t)G3FC * WR * WC + (size_t)k * KD * KD) * sizeof(float);
    }
    static constexpr size_t smem_uc(int k) { return ((size_t)2 * XR * XC + (size_t)k * KD * KD) * sizeof(float); }
};

// stage fma(a, B, A) over rows ty0 - H .. ty0 + G3Y + H - 1 and the matching columns (clamped),
// every load of a thread issued before its first store
template <int R, int MAG>
__device__ __forceinline__ void g3_stage(const StencilParams& sp, const float* __restrict__ A,
                                         const float* __restrict__ B, float a, int ty0, int tx0, float* xs) {
    using T = G3<R, MAG>;
    const int w8 = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (tx0 - T::CL >= 0 && tx0 + G3X + T::CL <= sp.W) {
        // interior columns: 16-byte loads (pitch and tx0 - CL are multiples of 4 floats), rows clamped
        constexpr int C4 = T::XC / 4, N4 = T::XR * C4, J4 = (N4 + G3T - 1) / G3T;
        float4 v4[J4];
#pragma unroll
        for (int j = 0; j < J4; ++j) {
            const int e = threadIdx.x + j * G3T;
            const int r = e / C4, c = (e - r * C4) * 4;
            if (e < N4) {
                const size_t o = (size_t)(clampi(ty0 - T::H + r, 0, sp.H - 1) - sp.store_lo) * sp.pitch + tx0 - T::CL + c;
                const float4 xa = __ldg(reinterpret_cast<const float4*>(A + o));
                if (B) {
                    const float4 xb = __ldg(reinterpret_cast<const float4*>(B + o));
                    v4[j] = make_float4(fmaf(a, xb.x, xa.x), fmaf(a, xb.y, xa.y), fmaf(a, xb.z, xa.z), fmaf(a, xb.w, xa.w));
                } else {
                    v4[j] = xa;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < J4; ++j) {
            const int e = threadIdx.x + j * G3T;
            if (e < N4) reinterpret_cast<float4*>(xs)[e] = v4[j];   // XC % 4 == 0: row-major float4 index
        }
        return;
    }
    constexpr int RJ = (T::XR + 7) / 8, CQ = (T::XC + 31) / 32;
    float v[RJ][CQ];
#pragma unroll
    for (int j = 0; j < RJ; ++j) {
        const int r = w8 + 8 * j;
        const size_t ro = (size_t)(clampi(ty0 - T::H + r, 0, sp.H - 1) - sp.store_lo) * sp.pitch;
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
            const int c = lane + 32 * q;
            const size_t o = ro + clampi(tx0 - T::CL + c, 0, sp.W - 1);
            v[j][q] = (r < T::XR && c < T::XC) ? fmaf(a, __ldg(B + o), __ldg(A + o)) : 0.0f;
        }
    }
#pragma unroll
    for (int j = 0; j < RJ; ++j)
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
            const int r = w8 + 8 * j, c = lane + 32 * q;
            if (r < T::XR && c < T::XC) xs[r * T::XC + c] = v[j][q];
        }
}

// forward sample: sum_PQ kappa_i(P,Q) xs[r0 + P][c0 + Q] (taps in registers)
template <int R, int MAG>
__device__ __forceinline__ float g3_fwd(const float (&tk)[(2 * R + 2) * (2 * R + 2)], const float* xs, int r0, int c0) {
    using T = G3<R, MAG>;
    const float* xr = xs + r0 * T::XC + c0;
    float z = 0.0f;
#pragma unroll
    for (int P = 0; P < T::KD; ++P)
#pragma unroll
        for (int Q = 0; Q < T::KD; ++Q) z = fmaf(tk[P * T::KD + Q], xr[P * T::XC + Q], z);
    return z;
}
template <int KD>
__device__ __forceinline__ void load_taps(const float* ti, float (&tk)[KD * KD]) {
#pragma unroll
    for (int j = 0; j < KD * KD; ++j) tk[j] = ti[j];
}

// flat index e -> (row, col) of a w x ... grid (exact for e < 2^20: (e + 1/2) / w stays >= 1/(2w)
// away from every integer)
__device__ __forceinline__ void split(int e, int w, float inv_w, int& r, int& c) {
    r = (int)(((float)e + 0.5f) * inv_w);
    c = e - r * w;
}

// BTV gradient contribution and value at one pixel of the staged tile (valid pairs only; INNER:
// every pair is valid).  The value accumulates gamma q rs = gamma (psi + eps): the eps part is the
// plan's affine correction (aff_vg).
template <int BQ, bool INNER>
__device__ __forceinline__ void btv_grad(const StencilParams& sp, const GenParams& gp, const float* xs, int XC,
                                         int ly, int lx, int vy, int vx, float& gb, float& val) {
    const float xv = xs[ly * XC + lx];
    auto pair = [&](int dy, int dx, float gm) {
        if (INNER || (vy + dy < sp.H && vx + dx >= 0 && vx + dx < sp.W)) {   // pair (v, v + d)
            const float t = xv - xs[(ly + dy) * XC + lx + dx];
            const float q = fmaf(t, t, sp.eps2), rs = rsqrtf(q);
            val = fmaf(gm * q, rs, val);
            gb = fmaf(gm * t, rs, gb);
        }
        if (INNER || (vy - dy >= 0 && vx - dx >= 0 && vx - dx < sp.W)) {     // pair (v - d, v)
            const float t = xs[(ly - dy) * XC + lx - dx] - xv;
            gb = fmaf(-gm * t, rsqrtf(fmaf(t, t, sp.eps2)), gb);
        }
    };
    if (BQ > 0) {   // the quadrant of window BQ with compile-time offsets (list order: dy-major)
#pragma unroll
        for (int dy = 0; dy < BQ; ++dy)
#pragma unroll
            for (int dx = 0; dx < BQ; ++dx)
                if (dy || dx) pair(dy, dx, gp.ogam[dy * BQ + dx - 1]);
    } else {
        for (int o = 0; o < gp.noff; ++o) pair(gp.offy[o], gp.offx[o], gp.ogam[o]);
    }
}

// BTV curvature sum_d gamma_d psi''(D_d x)(D_d p)^2 / eps^2 of the pairs anchored at one pixel
// (psi'' = eps^2 rs^3: the eps^2 factor is the plan's affine correction, aff_uc)
template <int BQ, bool INNER>
__device__ __forceinline__ float btv_curv(const StencilParams& sp, const GenParams& gp, const float* xs,
                                          const float* ps, int XC, int ly, int lx, int uy, int ux) {
    const int j0 = ly * XC + lx;
    const float xn = xs[j0], pn = ps[j0];
    float c = 0.0f;
    auto pair = [&](int dy, int dx, float gm) {
        if (INNER || (uy + dy < sp.H && ux + dx >= 0 && ux + dx < sp.W)) {
            const int j = j0 + dy * XC + dx;
            const float tt = xn - xs[j], dp = pn - ps[j];
            const float rs = rsqrtf(fmaf(tt, tt, sp.eps2));
            const float u = rs * dp;
            c = fmaf(gm * u, u * rs, c);
        }
    };
    if (BQ > 0) {
#pragma unroll
        for (int dy = 0; dy < BQ; ++dy)
#pragma unroll
            for (int dx = 0; dx < BQ; ++dx)
                if (dy || dx) pair(dy, dx, gp.ogam[dy * BQ + dx - 1]);
    } else {
        for (int q = 0; q < gp.noff; ++q) pair(gp.offy[q], gp.offx[q], gp.ogam[q]);
    }
    return c;
}

// L2 prefetch (bulk-copy engine, no registers) of the row segment [c0, c1) of `rows` rows of A,
// spread over the CTA's threads: the next tile's operands are in L2 when its staging loads issue
__device__ __forceinline__ void l2_prefetch_rows(const float* A, size_t pitch, int r0, int nrows, int rlo, int rhi,
                                                 int c0, int c1, int first_thread) {
    const int t = (int)threadIdx.x - first_thread;
    if (t < 0 || t >= nrows) return;
    const int r = min(max(r0 + t, rlo), rhi);
    const uintptr_t a = reinterpret_cast<uintptr_t>(A + (size_t)r * pitch + c0) & ~(uintptr_t)15;
    const uintptr_t e = (reinterpret_cast<uintptr_t>(A + (size_t)r * pitch + c1) + 15) & ~(uintptr_t)15;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

template <int PN, int R, int MAG, int BQ>
__global__ void __launch_bounds__(G3T, G3MINB_VG) k_gen3_vg(StencilParams sp, GenParams gp, Buffers b, int phase) {
    using T = G3<R, MAG>;
    constexpr int KD = T::KD, HX = T::H, CL = T::CL, XC = T::XC, WC = T::WC, NT = T::NT;
    extern __shared__ __align__(16) float g3s[];
    float* xs = g3s;                                   // XR x XC staged x'
    float* ws = xs + T::XR * XC;                       // FC x WR x WC rho' windows
    float* ts = ws + G3FC * T::WR * WC;                // k x KD x KD taps
    ScgState* st = b.st;
    if (phase != PH_DEBUG && st->done) return;
    const float alpha = (phase == PH_ITER) ? st->alpha_f : 0.0f;
    const int xcur = st->xcur, rcur = st->rcur;
    const float* X = pick(b.X, xcur);
    const float* P = pick(b.P, xcur);
    const float* Ro = pick(b.R, rcur);
    float* Rn = pick(b.R, rcur ^ 1);
    const int tid = threadIdx.x;
    for (int e = tid; e < gp.k * KD * KD; e += G3T) ts[e] = __ldg(gp.taps + e);   // ordered by the tile barriers
    const int ntx = (sp.W + G3X - 1) / G3X, nty = (sp.H + G3Y - 1) / G3Y;
    const int cx = tid % G3X, ry = tid / G3X;
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // D, R, <r',r'>, <r',r_old>
    for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {
        const int ty0 = (t / ntx) * G3Y, tx0 = (t % ntx) * G3X;
        // virtual rows / cols that clamp into the tile (image-border tiles add the fold ranges)
        const int vylo = ty0 == 0 ? gp.fy_lo : ty0, vyhi = ty0 + G3Y >= sp.H ? gp.fy_hi : ty0 + G3Y - 1;
        const int vxlo = tx0 == 0 ? gp.fx_lo : tx0, vxhi = tx0 + G3X >= sp.W ? gp.fx_hi : tx0 + G3X - 1;
        const int vx = tx0 + cx, vy0 = ty0 + ry;
        // image-border pixels take their whole data gradient from the fold walk below
        const bool btile = ty0 == 0 || ty0 + G3Y >= sp.H || tx0 == 0 || tx0 + G3X >= sp.W;
        unsigned nb = 0;   // bit k: pixel k is not on the image border
#pragma unroll
        for (int k = 0; k < G3PPT; ++k) {
            const int vy = vy0 + 4 * k;
            if (!(vy == 0 || vy == sp.H - 1 || vx == 0 || vx == sp.W - 1)) nb |= 1u << k;
        }
        __syncthreads();   // the previous tile's x' and windows are consumed
        g3_stage<R, MAG>(sp, X, P, alpha, ty0, tx0, xs);
        {   // prefetch the next tile's x, p (tile + halo) and r_old rows into L2 while this one computes
            const int tn = t + gridDim.x;
            if (tn < ntx * nty) {
                const int ny0 = (tn / ntx) * G3Y, nx0 = (tn % ntx) * G3X;
                const int c0 = max(nx0 - HX, 0), c1 = min(nx0 + G3X + HX, sp.W);
                const float* Xb = X - (size_t)sp.store_lo * sp.pitch;
                const float* Pb = P - (size_t)sp.store_lo * sp.pitch;
                const float* Rb = Ro - (size_t)sp.store_lo * sp.pitch;
                l2_prefetch_rows(Xb, sp.pitch, ny0 - HX, T::XR, 0, sp.H - 1, c0, c1, 0);
                l2_prefetch_rows(Pb, sp.pitch, ny0 - HX, T::XR, 0, sp.H - 1, c0, c1, 64);
                l2_prefetch_rows(Rb, sp.pitch, ny0, G3Y, 0, sp.H - 1, nx0, min(nx0 + G3X, sp.W), 128);
            }
        }
        float g[G3PPT];
#pragma unroll
        for (int k = 0; k < G3PPT; ++k) g[k] = 0.0f;
        for (int i0 = 0; i0 < gp.k; i0 += G3FC) {
            __syncthreads();   // x' staged / the previous chunk's windows consumed
            // w = rho'(e) over each frame's window (unclipped: zero outside the frame)
#pragma unroll 1
            for (int f = 0; f < G3FC && i0 + f < gp.k; ++f) {
                const int i = i0 + f, sy = gp.sy[i], sx = gp.sx[i];
                const int alo = cdivc<MAG>(vylo - sy - R - 1), ahi = fdivc<MAG>(vyhi - sy + R);
                const int blo = cdivc<MAG>(vxlo - sx - R - 1), bhi = fdivc<MAG>(vxhi - sx + R);
                const int wr = ahi - alo + 1, wc = bhi - blo + 1;
                const float inv = 1.0f / (float)wc;
                float tk[KD * KD];
                load_taps<KD>(ts + i * KD * KD, tk);
                const float* yi = gp.lr + (size_t)i * gp.lr_h * gp.lr_w;
                float* wf = ws + f * T::WR * WC;
                // this thread's window samples of y, all loads issued before the first use (fixed trip
                // count: the window is at most WR x WC)
                constexpr int NE = (T::WR * WC + G3T - 1) / G3T;
                float yr[NE];
#pragma unroll
                for (int n = 0; n < NE; ++n) {
                    const int e = tid + n * G3T;
                    int ra, cb;
                    split(e, wc, inv, ra, cb);
                    const int a = alo + ra, bb = blo + cb;
                    yr[n] = (e < wr * wc && a >= 0 && a < gp.lr_h && bb >= 0 && bb < gp.lr_w)
                                ? __ldg(yi + (size_t)a * gp.lr_w + bb) : 0.0f;
                }
#pragma unroll
                for (int n = 0; n < NE; ++n) {
                    const int e = tid + n * G3T;
                    if (e >= wr * wc) break;
                    int ra, cb;
                    split(e, wc, inv, ra, cb);
                    const int a = alo + ra, bb = blo + cb;
                    float d1 = 0.0f;
                    if (a >= 0 && a < gp.lr_h && bb >= 0 && bb < gp.lr_w) {
                        const float yv = yr[n];
                        const float ev = g3_fwd<R, MAG>(tk, xs, MAG * a + sy - R - (ty0 - HX), MAG * bb + sx - R - (tx0 - CL)) - yv;
                        float v;
                        if (PN == 2) {
                            v = ev * ev;
                            d1 = 2.0f * ev;
                        } else {   // v = rho + eps (eps per LR pixel is the affine correction)
                            const float q = fmaf(ev, ev, sp.eps2), rs = rsqrtf(q);
                            v = q * rs;
                            d1 = ev * rs;
                        }
                        const int ay = clampi(MAG * a + sy, 0, sp.H - 1), ax = clampi(MAG * bb + sx, 0, sp.W - 1);
                        if (ay >= ty0 && ay < ty0 + G3Y && ax >= tx0 && ax < tx0 + G3X) acc[0] += v;   // owner counts
                    }
                    wf[ra * WC + cb] = d1;
                }
            }
            __syncthreads();
            // gather A_i^T w
#pragma unroll 1
            for (int f = 0; f < G3FC && i0 + f < gp.k; ++f) {
                const int i = i0 + f, sy = gp.sy[i], sx = gp.sx[i];
                const int alo = cdivc<MAG>(vylo - sy - R - 1), blo = cdivc<MAG>(vxlo - sx - R - 1);
                const float* ti = ts + i * KD * KD;
                const float* wf = ws + f * T::WR * WC;
                const int uy = vy0 - sy, ux = vx - sx;   // frame-relative HR coordinates
                if (4 % MAG == 0) {
                    // one residue class per thread: taps in registers, window offsets compile-time
                    const int p0 = pmod(uy + R, MAG), q0 = pmod(ux + R, MAG);   // first P + R / Q + R
                    const int a0 = (uy - (p0 - R)) / MAG - alo, b0 = (ux - (q0 - R)) / MAG - blo;   // exact
                    float tv[NT][NT];
#pragma unroll
                    for (int jp = 0; jp < NT; ++jp)
#pragma unroll
                        for (int jq = 0; jq < NT; ++jq) {
                            const int Pp = p0 + jp * MAG, Qq = q0 + jq * MAG;
                            tv[jp][jq] = (Pp < KD && Qq < KD) ? ti[Pp * KD + Qq] : 0.0f;
                        }
                    // taps outside kappa read an in-window neighbour (times 0); a class without taps
                    // (KD < MAG) reads the window origin
                    const bool anyt = p0 < KD && q0 < KD;
                    const int jpv = anyt ? (KD - 1 - p0) / MAG : 0, jqv = anyt ? (KD - 1 - q0) / MAG : 0;
                    const float* wb = anyt ? wf + a0 * WC + b0 : wf;
#pragma unroll
                    for (int k = 0; k < G3PPT; ++k) {
                        float ga = 0.0f;
#pragma unroll
                        for (int jp = 0; jp < NT; ++jp)
#pragma unroll
                            for (int jq = 0; jq < NT; ++jq)
                                ga = fmaf(tv[jp][jq], wb[(4 / MAG) * k * WC - min(jp, jpv) * WC - min(jq, jqv)], ga);
                        g[k] += ((nb >> k) & 1u) ? ga : 0.0f;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < G3PPT; ++k) {
                        const int vy = vy0 + 4 * k;
                        const int p0 = pmod(vy - sy + R, MAG), q0 = pmod(ux + R, MAG);
                        float ga = 0.0f;
#pragma unroll
                        for (int jp = 0; jp < NT; ++jp) {
                            const int Pp = p0 + jp * MAG;
                            if (Pp >= KD) break;
                            const int a = (vy - sy - (Pp - R)) / MAG;
#pragma unroll
                            for (int jq = 0; jq < NT; ++jq) {
                                const int Qq = q0 + jq * MAG;
                                if (Qq >= KD) break;
                                const int bb = (ux - (Qq - R)) / MAG;
                                ga = fmaf(ti[Pp * KD + Qq], wf[(a - alo) * WC + bb - blo], ga);
                            }
                        }
                        g[k] += ((nb >> k) & 1u) ? ga : 0.0f;
                    }
                }
            }
            // image-border pixels: the walk over the virtual positions v' with clamp(v') = v (the
            // exact transpose of the clamped forward reads; one row / column per side)
            if (btile) {
#pragma unroll 1
                for (int k = 0; k < G3PPT; ++k) {
                    const int vy = vy0 + 4 * k;
                    if (((nb >> k) & 1u) || vy >= sp.H || vx >= sp.W) continue;
                    float gk = 0.0f;
                    for (int f = 0; f < G3FC && i0 + f < gp.k; ++f) {
                        const int i = i0 + f, sy = gp.sy[i], sx = gp.sx[i];
                        const int alo = cdivc<MAG>(vylo - sy - R - 1), blo = cdivc<MAG>(vxlo - sx - R - 1);
                        const float* ti = ts + i * KD * KD;
                        const float* wf = ws + f * T::WR * WC;
                        const int ylo = vy == 0 ? gp.fy_lo : vy, yhi = vy == sp.H - 1 ? gp.fy_hi : vy;
                        const int xlo = vx == 0 ? gp.fx_lo : vx, xhi = vx == sp.W - 1 ? gp.fx_hi : vx;
                        float all = 0.0f;
                        for (int yy = ylo; yy <= yhi; ++yy)
                            for (int xx = xlo; xx <= xhi; ++xx)
                                for (int Pp = 0; Pp < KD; ++Pp) {
                                    const int ny = yy - sy - (Pp - R);
                                    if (pmod(ny, MAG)) continue;
                                    const int a = fdivc<MAG>(ny);
                                    for (int Qq = 0; Qq < KD; ++Qq) {
                                        const int nx = xx - sx - (Qq - R);
                                        if (pmod(nx, MAG)) continue;
                                        const int bb = fdivc<MAG>(nx);
                                        all = fmaf(ti[Pp * KD + Qq], wf[(a - alo) * WC + bb - blo], all);
                                    }
                                }
                        gk += all;
                    }
                    g[k] += gk;
                }
            }
        }
        // BTV (valid pairs only) and the output; r_old of the 8 pixels loaded first (in flight
        // during the BTV arithmetic)
        const bool inner = ty0 >= HX && ty0 + G3Y + HX <= sp.H && tx0 >= HX && tx0 + G3X + HX <= sp.W;
        float rold[G3PPT];
#pragma unroll
        for (int k = 0; k < G3PPT; ++k) {
            const int vy = vy0 + 4 * k;
            rold[k] = (vy < sp.H && vx < sp.W) ? __ldg(Ro + (size_t)(vy - sp.store_lo) * sp.pitch + vx) : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < G3PPT; ++k) {
            const int vy = vy0 + 4 * k;
            if (vy >= sp.H || vx >= sp.W) continue;
            float gb = 0.0f;
            if (inner) btv_grad<BQ, true>(sp, gp, xs, XC, ry + 4 * k + HX, cx + CL, vy, vx, gb, acc[1]);
            else btv_grad<BQ, false>(sp, gp, xs, XC, ry + 4 * k + HX, cx + CL, vy, vx, gb, acc[1]);
            const float rn = -fmaf(sp.lam, gb, g[k]);
            const size_t o = (size_t)(vy - sp.store_lo) * sp.pitch + vx;
            Rn[o] = rn;
            acc[2] = fmaf(rn, rn, acc[2]);
            acc[3] = fmaf(rn, rold[k], acc[3]);
        }
    }
    double accd[NSLOT] = {acc[0], acc[1], acc[2], acc[3]}, tot[NSLOT];
    if (reduce_partials(accd, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) finish_scalars<0>(sp, b, tot, phase);
}

template <int PN, int R, int MAG, int BQ>
__global__ void __launch_bounds__(G3T, G3MINB_UC) k_gen3_uc(StencilParams sp, GenParams gp, Buffers b, int phase) {
    using T = G3<R, MAG>;
    constexpr int KD = T::KD, HX = T::H, CL = T::CL, XC = T::XC;
    extern __shared__ __align__(16) float g3s[];
    float* xs = g3s;                 // new x on the tile + halo
    float* ps = xs + T::XR * XC;     // new p
    float* ts = ps + T::XR * XC;     // taps
    ScgState* st = b.st;
    if (phase != PH_DEBUG) {
        if (st->done) return;
        if (!st->success) {   // rejected step: delta is reused, only the scalar pre-value step runs
            if (blockIdx.x == 0 && threadIdx.x == 0) scg_pre_value(st);
            return;
        }
    }
    const int xcur = st->xcur, rcur = st->rcur;
    const float au = (phase == PH_DEBUG) ? 0.0f : st->alpha_upd_f;
    const float be = (phase == PH_DEBUG) ? 0.0f : st->beta_f;
    const float* X = pick(b.X, xcur);
    const float* Pc = pick(b.P, xcur);
    const float* Rc = pick(b.R, rcur);
    float* Xn = pick(b.X, xcur ^ 1);
    float* Pn = pick(b.P, xcur ^ 1);
    const int tid = threadIdx.x;
    for (int e = tid; e < gp.k * KD * KD; e += G3T) ts[e] = __ldg(gp.taps + e);
    const int ntx = (sp.W + G3X - 1) / G3X, nty = (sp.H + G3Y - 1) / G3Y;
    const int cx = tid % G3X, ry = tid / G3X;
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // data curvature, BTV curvature, <p,p>, <p,r>
    for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {
        const int ty0 = (t / ntx) * G3Y, tx0 = (t % ntx) * G3X;
        __syncthreads();
        g3_stage<R, MAG>(sp, X, Pc, au, ty0, tx0, xs);
        g3_stage<R, MAG>(sp, Rc, Pc, be, ty0, tx0, ps);
        {   // prefetch the next tile's x, p, r (tile + halo) into L2 while this one computes
            const int tn = t + gridDim.x;
            if (tn < ntx * nty) {
                const int ny0 = (tn / ntx) * G3Y, nx0 = (tn % ntx) * G3X;
                const int c0 = max(nx0 - HX, 0), c1 = min(nx0 + G3X + HX, sp.W);
                const size_t so = (size_t)sp.store_lo * sp.pitch;
                l2_prefetch_rows(X - so, sp.pitch, ny0 - HX, T::XR, 0, sp.H - 1, c0, c1, 0);
                l2_prefetch_rows(Pc - so, sp.pitch, ny0 - HX, T::XR, 0, sp.H - 1, c0, c1, 64);
                l2_prefetch_rows(Rc - so, sp.pitch, ny0 - HX, T::XR, 0, sp.H - 1, c0, c1, 128);
            }
        }
        __syncthreads();
        const bool inner = ty0 >= HX && ty0 + G3Y + HX <= sp.H && tx0 >= HX && tx0 + G3X + HX <= sp.W;
#pragma unroll
        for (int k = 0; k < G3PPT; ++k) {
            const int uy = ty0 + ry + 4 * k, ux = tx0 + cx;
            if (uy >= sp.H || ux >= sp.W) continue;
            const int ly = ry + 4 * k + HX, lx = cx + CL;
            const float xn = xs[ly * XC + lx], pn = ps[ly * XC + lx];
            const size_t o = (size_t)(uy - sp.store_lo) * sp.pitch + ux;
            Xn[o] = xn;
            Pn[o] = pn;
            acc[2] = fmaf(pn, pn, acc[2]);
            acc[3] = fmaf(pn, __ldg(Rc + o), acc[3]);
            acc[1] += inner ? btv_curv<BQ, true>(sp, gp, xs, ps, XC, ly, lx, uy, ux)
                            : btv_curv<BQ, false>(sp, gp, xs, ps, XC, ly, lx, uy, ux);
        }
        // data curvature of the LR pixels this tile owns (clamped anchor inside the tile)
#pragma unroll 1
        for (int i = 0; i < gp.k; ++i) {
            const int sy = gp.sy[i], sx = gp.sx[i];
            const int alo = ty0 == 0 ? 0 : max(0, cdivc<MAG>(ty0 - sy));
            const int ahi = ty0 + G3Y >= sp.H ? gp.lr_h - 1 : min(gp.lr_h - 1, fdivc<MAG>(ty0 + G3Y - 1 - sy));
            const int blo = tx0 == 0 ? 0 : max(0, cdivc<MAG>(tx0 - sx));
            const int bhi = tx0 + G3X >= sp.W ? gp.lr_w - 1 : min(gp.lr_w - 1, fdivc<MAG>(tx0 + G3X - 1 - sx));
            const int wr = ahi - alo + 1, wc = bhi - blo + 1;
            if (wr <= 0 || wc <= 0) continue;
            const float inv = 1.0f / (float)wc;
            float tk[KD * KD];
            load_taps<KD>(ts + i * KD * KD, tk);
            const float* yi = gp.lr + (size_t)i * gp.lr_h * gp.lr_w;
            for (int e = tid; e < wr * wc; e += G3T) {
                int ra, cb;
                split(e, wc, inv, ra, cb);
                const int a = alo + ra, bb = blo + cb;
                const float yv = __ldg(yi + (size_t)a * gp.lr_w + bb);
                const int r0 = MAG * a + sy - R - (ty0 - HX), c0 = MAG * bb + sx - R - (tx0 - CL);
                const float ev = g3_fwd<R, MAG>(tk, xs, r0, c0) - yv;
                const float ap = g3_fwd<R, MAG>(tk, ps, r0, c0);
                if (PN == 2) {   // rho'' = 2: the affine factor
                    acc[0] = fmaf(ap, ap, acc[0]);
                } else {         // rho'' = eps^2 rs^3: eps^2 is the affine factor
                    const float rs = rsqrtf(fmaf(ev, ev, sp.eps2));
                    const float u = rs * ap;
                    acc[0] = fmaf(u, u * rs, acc[0]);
                }
            }
        }
    }
    double accd[NSLOT] = {acc[0], acc[1], acc[2], acc[3]}, tot[NSLOT];
    if (reduce_partials(accd, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

template <typename K>
cudaError_t g3_launch(K kernel, size_t smem, const StencilParams& sp, const GenParams& gp, const Buffers& b, int phase,
                      cudaStream_t s) {
    // > 48 KB of dynamic shared memory needs the opt-in (raised only, thread-safe)
    cudaError_t e = raise_dyn_smem(reinterpret_cast<const void*>(kernel), smem);
    if (e != cudaSuccess) return e;
    kernel<<<gp.nblk3, G3T, smem, s>>>(sp, gp, b, phase);
    return cudaGetLastError();
}

template <int PN, int BQ, bool VG>
cudaError_t g3_dispatch(const StencilParams& sp, const GenParams& gp, const Buffers& b, int phase, cudaStream_t s) {
#define FL_G3(R_, M_)                                                                                     \
    case R_ * 8 + M_:                                                                                     \
        return VG ? g3_launch(k_gen3_vg<PN, R_, M_, BQ>, G3<R_, M_>::smem_vg(gp.k), sp, gp, b, phase, s) \
                  : g3_launch(k_gen3_uc<PN, R_, M_, BQ>, G3<R_, M_>::smem_uc(gp.k), sp, gp, b, phase, s);
    switch (gp.R * 8 + gp.mag) {
        FL_G3(0, 1) FL_G3(0, 2) FL_G3(0, 3) FL_G3(0, 4) FL_G3(1, 1) FL_G3(1, 2) FL_G3(1, 3) FL_G3(1, 4)
        FL_G3(2, 1) FL_G3(2, 2) FL_G3(2, 3) FL_G3(2, 4)
        default: return cudaErrorInvalidValue;
    }
#undef FL_G3
}

}  // namespace

unsigned gen3_blocks(int W, int H, int cap) {
    const long long n = (long long)((W + G3X - 1) / G3X) * ((H + G3Y - 1) / G3Y);
    return (unsigned)std::min<long long>(n, cap);
}

size_t gen3_smem(int R, int mag, int k) {
    switch (R * 8 + mag) {
#define FL_G3S(R_, M_) \
    case R_ * 8 + M_: return std::max(G3<R_, M_>::smem_vg(k), G3<R_, M_>::smem_uc(k));
        FL_G3S(0, 1) FL_G3S(0, 2) FL_G3S(0, 3) FL_G3S(0, 4) FL_G3S(1, 1) FL_G3S(1, 2) FL_G3S(1, 3) FL_G3S(1, 4)
        FL_G3S(2, 1) FL_G3S(2, 2) FL_G3S(2, 3) FL_G3S(2, 4)
#undef FL_G3S
        default: return (size_t)1 << 30;
    }
}

cudaError_t launch_gen3_vg(int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b, int phase,
                           cudaStream_t s) {
    if (gp.btvq == 3) return pn == 2 ? g3_dispatch<2, 3, true>(sp, gp, b, phase, s) : g3_dispatch<1, 3, true>(sp, gp, b, phase, s);
    return pn == 2 ? g3_dispatch<2, 0, true>(sp, gp, b, phase, s) : g3_dispatch<1, 0, true>(sp, gp, b, phase, s);
}

cudaError_t launch_gen3_uc(int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b, int phase,
                           cudaStream_t s) {
    if (gp.btvq == 3) return pn == 2 ? g3_dispatch<2, 3, false>(sp, gp, b, phase, s) : g3_dispatch<1, 3, false>(sp, gp, b, phase, s);
    return pn == 2 ? g3_dispatch<2, 0, false>(sp, gp, b, phase, s) : g3_dispatch<1, 0, false>(sp, gp, b, phase, s);
}

}  // namespace flmisr
