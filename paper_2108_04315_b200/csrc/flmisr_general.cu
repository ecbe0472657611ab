// flmisr_general.cu -- the general-geometry path: any number of frames K >= 1,
// arbitrary shifts (integer HR phases anywhere, fractional phases, repeated or missing phases) and a
// per-frame composed kernel kappa_i = PSF (*) bilinear(frac(mag * shift_i)) (reading 19).
//
// The data term is evaluated on the LR grid of every frame (no polyphase interleave):
//   residual pass (LR pixels)  e_i(a,b) = sum_PQ kappa_i(P,Q) x~(mag a + s_iy + P, mag b + s_ix + Q) - y_i(a,b)
//   gradient pass (HR pixels)  g(v) = sum over the virtual positions v' with clamp(v') = v of
//                              sum_i sum_PQ kappa_i(P,Q) w_i((v'_y - s_iy - P)/mag, (v'_x - s_ix - Q)/mag)
//                              (a gather: the exact transpose of the clamped strided correlation)
// and the curvature likewise (update pass on HR pixels with the BTV curvature, data-curvature pass
// on LR pixels).  Each pair of passes ends in one last-CTA reduction that feeds the same on-device
// SCG scalar logic as the fast paths.  Correctness first: one pixel per thread, taps from a small
// device table; the fast paths carry the performance.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "flmisr_common.cuh"
#include "flmisr_internal.h"

namespace flmisr {
namespace {

constexpr int GT = 256;

__device__ __forceinline__ float tapk(const GenParams& gp, int i, int P, int Q) {
    return __ldg(gp.taps + ((size_t)i * gp.kd + (P + gp.R)) * gp.kd + (Q + gp.R));
}

// plain fixed-order CTA sum of NSLOT fp32 partials into part[slot * nblk + blk] (no last-CTA logic)
__device__ void block_partials(const float (&acc)[NSLOT], double* part, int nblk, int blk) {
    __shared__ double sred[GT / 32][NSLOT];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
        double v = warp_sum((double)acc[k]);
        if (lane == 0) sred[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < NSLOT) {
        double v = 0.0;
        for (int w = 0; w < GT / 32; ++w) v += sred[w][threadIdx.x];
        part[(size_t)threadIdx.x * nblk + blk] = v;
    }
}

// last CTA: fixed-order sum of another kernel's partial array (slot-major, nblk CTAs)
__device__ double sum_slot(const double* part, int slot, int nblk) {
    __shared__ double sh[GT / 32];
    double v = 0.0;
    for (int i = threadIdx.x; i < nblk; i += GT) v += __ldcg(part + (size_t)slot * nblk + i);
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < GT / 32; ++w) t += sh[w];
    __syncthreads();
    return t;
}

__device__ __forceinline__ float xval(const StencilParams& sp, const float* X, const float* P, float a, int u, int v) {
    const size_t o = (size_t)(u - sp.store_lo) * sp.pitch + v;
    return fmaf(a, __ldg(P + o), __ldg(X + o));
}

// forward sample of frame i at LR (a, b) on x' = x + alpha p (clamp-extended, reading 4)
__device__ __forceinline__ float fwd_sample(const StencilParams& sp, const GenParams& gp, const float* X,
                                            const float* P, float alpha, int i, int a, int b) {
    const int by = gp.mag * a + gp.sy[i], bx = gp.mag * b + gp.sx[i];
    float z = 0.0f;
    for (int Pp = -gp.R; Pp <= gp.R + 1; ++Pp) {
        const int u = clampi(by + Pp, 0, sp.H - 1);
        for (int Qq = -gp.R; Qq <= gp.R + 1; ++Qq) {
            const float k = tapk(gp, i, Pp, Qq);
            if (k == 0.0f) continue;
            z = fmaf(k, xval(sp, X, P, alpha, u, clampi(bx + Qq, 0, sp.W - 1)), z);
        }
    }
    return z;
}

// transpose of the clamped strided correlation at HR pixel (vy, vx), from LR-layout weights w.
// Interior pixels: for frame i only the taps with P = vy - s_iy (mod mag) and Q = vx - s_ix (mod mag)
// reach v (ceil(kd/mag)^2 of the kd^2 taps).  Border pixels also collect the clamped virtual
// positions v' (clamp(v') = v) through the generic fold loop.
__device__ float adj_gather(const StencilParams& sp, const GenParams& gp, const float* __restrict__ w, int vy, int vx) {
    float g = 0.0f;
    const int mag = gp.mag;
    if (vy > 0 && vy < sp.H - 1 && vx > 0 && vx < sp.W - 1) {
        for (int i = 0; i < gp.k; ++i) {
            const int dyi = vy - gp.sy[i] + gp.R, dxi = vx - gp.sx[i] + gp.R;   // >= 0 for the taps below
            const int p0 = -gp.R + ((dyi % mag) + mag) % mag;
            const int q0 = -gp.R + ((dxi % mag) + mag) % mag;
            const float* wi = w + (size_t)i * gp.lr_h * gp.lr_w;
            for (int Pp = p0; Pp <= gp.R + 1; Pp += mag) {
                const int ny = vy - gp.sy[i] - Pp;
                if (ny < 0) continue;
                const int a = ny / mag;
                if (a >= gp.lr_h) continue;
                for (int Qq = q0; Qq <= gp.R + 1; Qq += mag) {
                    const int nx = vx - gp.sx[i] - Qq;
                    if (nx < 0) continue;
                    const int b = nx / mag;
                    if (b >= gp.lr_w) continue;
                    g = fmaf(tapk(gp, i, Pp, Qq), __ldg(wi + (size_t)a * gp.lr_w + b), g);
                }
            }
        }
        return g;
    }
    const int ylo = vy == 0 ? gp.fy_lo : vy, yhi = vy == sp.H - 1 ? gp.fy_hi : vy;
    const int xlo = vx == 0 ? gp.fx_lo : vx, xhi = vx == sp.W - 1 ? gp.fx_hi : vx;
    for (int yy = ylo; yy <= yhi; ++yy)
        for (int xx = xlo; xx <= xhi; ++xx)
            for (int i = 0; i < gp.k; ++i)
                for (int Pp = -gp.R; Pp <= gp.R + 1; ++Pp) {
                    const int ny = yy - gp.sy[i] - Pp;
                    if (ny < 0 || ny % mag) continue;
                    const int a = ny / mag;
                    if (a >= gp.lr_h) continue;
                    for (int Qq = -gp.R; Qq <= gp.R + 1; ++Qq) {
                        const int nx = xx - gp.sx[i] - Qq;
                        if (nx < 0 || nx % mag) continue;
                        const int b = nx / mag;
                        if (b >= gp.lr_w) continue;
                        g = fmaf(tapk(gp, i, Pp, Qq), __ldg(w + ((size_t)i * gp.lr_h + a) * gp.lr_w + b), g);
                    }
                }
    return g;
}

// ---- value + gradient ---------------------------------------------------------------------------
template <int PN>
__global__ void __launch_bounds__(GT) k_gen_residual(StencilParams sp, GenParams gp, Buffers b, int phase) {
    ScgState* st = b.st;
    if (phase != PH_DEBUG && st->done) return;
    const float alpha = (phase == PH_ITER) ? st->alpha_f : 0.0f;
    const float* X = pick(b.X, st->xcur);
    const float* P = pick(b.P, st->xcur);
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};
    const long long n = (long long)gp.k * gp.lr_h * gp.lr_w;
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx < n) {
        const int i = (int)(idx / ((long long)gp.lr_h * gp.lr_w));
        const int rem = (int)(idx - (long long)i * gp.lr_h * gp.lr_w);
        const int a = rem / gp.lr_w, c = rem - a * gp.lr_w;
        const float e = fwd_sample(sp, gp, X, P, alpha, i, a, c) - __ldg(gp.lr + idx);
        float v, d1;
        Pen<PN>::val_d1(e, sp.eps, sp.eps2, v, d1);
        gp.w[idx] = d1;
        acc[0] = v;
    }
    block_partials(acc, gp.part_a, gridDim.x, blockIdx.x);
}

template <int PN>
__global__ void __launch_bounds__(GT) k_gen_grad(StencilParams sp, GenParams gp, Buffers b, int phase) {
    ScgState* st = b.st;
    if (phase != PH_DEBUG && st->done) return;
    const float alpha = (phase == PH_ITER) ? st->alpha_f : 0.0f;
    const int xcur = st->xcur, rcur = st->rcur;
    const float* X = pick(b.X, xcur);
    const float* P = pick(b.P, xcur);
    const float* Ro = pick(b.R, rcur);
    float* Rn = pick(b.R, rcur ^ 1);
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // -, R, <r',r'>, <r',r_old>
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx < (long long)sp.H * sp.W) {
        const int vy = (int)(idx / sp.W), vx = (int)(idx - (long long)vy * sp.W);
        float g = adj_gather(sp, gp, gp.w, vy, vx);
        float gb = 0.0f;
        const float xv = xval(sp, X, P, alpha, vy, vx);
        for (int o = 0; o < gp.noff; ++o) {   // BTV offset list (quadrant or Farsiu), valid pairs only
            const int dy = gp.offy[o], dx = gp.offx[o];
            const float gm = gp.ogam[o];
            if (vy + dy < sp.H && vx + dx >= 0 && vx + dx < sp.W) {      // pair (v, v + d)
                float v, d1;
                charb_val_d1(xv - xval(sp, X, P, alpha, vy + dy, vx + dx), sp.eps, sp.eps2, v, d1);
                acc[1] = fmaf(gm, v, acc[1]);
                gb = fmaf(gm, d1, gb);
            }
            if (vy - dy >= 0 && vx - dx >= 0 && vx - dx < sp.W)          // pair (v - d, v)
                gb = fmaf(-gm, charb_d1(xval(sp, X, P, alpha, vy - dy, vx - dx) - xv, sp.eps2), gb);
        }
        const float rn = -fmaf(sp.lam, gb, g);
        const size_t o = (size_t)(vy - sp.store_lo) * sp.pitch + vx;
        Rn[o] = rn;
        acc[2] = rn * rn;
        acc[3] = rn * __ldg(Ro + o);
    }
    double accd[NSLOT] = {acc[0], acc[1], acc[2], acc[3]}, tot[NSLOT];
    if (reduce_partials(accd, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        const double d = sum_slot(gp.part_a, 0, gp.nblk_lr);
        tot[0] = d;
        finish_scalars<0>(sp, b, tot, phase);
    }
}

// ---- update + curvature -------------------------------------------------------------------------
template <int PN>
__global__ void __launch_bounds__(GT) k_gen_update(StencilParams sp, GenParams gp, Buffers b, int phase) {
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
    const float* P = pick(b.P, xcur);
    const float* R = pick(b.R, rcur);
    float* Xn = pick(b.X, xcur ^ 1);
    float* Pn = pick(b.P, xcur ^ 1);
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // -, curv BTV, <p,p>, <p,r>
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx < (long long)sp.H * sp.W) {
        const int uy = (int)(idx / sp.W), ux = (int)(idx - (long long)uy * sp.W);
        auto newx = [&](int y, int x) {
            const size_t o = (size_t)(y - sp.store_lo) * sp.pitch + x;
            return fmaf(au, __ldg(P + o), __ldg(X + o));
        };
        auto newp = [&](int y, int x) {
            const size_t o = (size_t)(y - sp.store_lo) * sp.pitch + x;
            return fmaf(be, __ldg(P + o), __ldg(R + o));
        };
        const size_t o = (size_t)(uy - sp.store_lo) * sp.pitch + ux;
        const float xn = newx(uy, ux), pn = newp(uy, ux);
        Xn[o] = xn;
        Pn[o] = pn;
        acc[2] = pn * pn;
        acc[3] = pn * __ldg(R + o);
        for (int o = 0; o < gp.noff; ++o) {
            const int dy = gp.offy[o], dx = gp.offx[o];
            if (uy + dy < sp.H && ux + dx >= 0 && ux + dx < sp.W) {
                const float t = xn - newx(uy + dy, ux + dx), dp = pn - newp(uy + dy, ux + dx);
                acc[1] = fmaf(gp.ogam[o] * charb_d2(t, sp.eps2), dp * dp, acc[1]);
            }
        }
    }
    block_partials(acc, gp.part_a, gridDim.x, blockIdx.x);
}

template <int PN>
__global__ void __launch_bounds__(GT) k_gen_curv_data(StencilParams sp, GenParams gp, Buffers b, int phase) {
    ScgState* st = b.st;
    if (phase != PH_DEBUG && (st->done || !st->success)) return;
    const int xcur = st->xcur;
    const float* Xn = pick(b.X, xcur ^ 1);
    const float* Pn = pick(b.P, xcur ^ 1);
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};
    const long long n = (long long)gp.k * gp.lr_h * gp.lr_w;
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx < n) {
        const int i = (int)(idx / ((long long)gp.lr_h * gp.lr_w));
        const int rem = (int)(idx - (long long)i * gp.lr_h * gp.lr_w);
        const int a = rem / gp.lr_w, c = rem - a * gp.lr_w;
        const float e = fwd_sample(sp, gp, Xn, Pn, 0.0f, i, a, c) - __ldg(gp.lr + idx);
        // A p: the forward sample of p_new (fwd_sample with alpha = 1 on (0, p) would need a zero buffer;
        // evaluate directly)
        const int by = gp.mag * a + gp.sy[i], bx = gp.mag * c + gp.sx[i];
        float ap = 0.0f;
        for (int Pp = -gp.R; Pp <= gp.R + 1; ++Pp) {
            const int u = clampi(by + Pp, 0, sp.H - 1);
            for (int Qq = -gp.R; Qq <= gp.R + 1; ++Qq) {
                const float k = tapk(gp, i, Pp, Qq);
                if (k == 0.0f) continue;
                ap = fmaf(k, __ldg(Pn + (size_t)(u - sp.store_lo) * sp.pitch + clampi(bx + Qq, 0, sp.W - 1)), ap);
            }
        }
        acc[0] = Pen<PN>::d2(e, sp.eps2) * ap * ap;
    }
    double accd[NSLOT] = {acc[0], 0.0, 0.0, 0.0}, tot[NSLOT];
    if (reduce_partials(accd, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        tot[1] = sum_slot(gp.part_a, 1, gp.nblk_hr);
        tot[2] = sum_slot(gp.part_a, 2, gp.nblk_hr);
        tot[3] = sum_slot(gp.part_a, 3, gp.nblk_hr);
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

// ================================================================================================
// Tiled general-path kernels (the hot loop).  Same arithmetic as the per-pixel reference kernels
// above (which stay for the debug entries and the image-border folds), with the operands staged
// in shared memory: LR tiles of 32 x 8 pixels of one frame read their HR footprint of x' once;
// HR tiles of 64 x 16 pixels read x' (+ halo 2) and, frame by frame, the LR window of rho' that
// reaches them.  R = PSF radius (kappa offsets [-R, R+1]); mag is a runtime stride <= 4.
// ================================================================================================
constexpr int LTX = 32, LTY = 8;                  // LR tile
constexpr int HTX = 64, HTY = 16, HH = 2;         // HR tile, BTV halo
constexpr int MAXMAG = 4;

__device__ __forceinline__ int floordiv(int a, int m) { return a >= 0 ? a / m : -((-a + m - 1) / m); }

// HR footprint of an LR tile of frame i: rows hy0 .. hy0 + nr - 1, cols hx0 .. hx0 + nc - 1 (clamped reads)
template <int R>
struct Foot {
    static constexpr int KD = 2 * R + 2;
    static constexpr int NR = MAXMAG * (LTY - 1) + KD, NC = MAXMAG * (LTX - 1) + KD;
};

// stage fma(a, B, A) (or A when B == nullptr) of the footprint into xs (row stride nc).  Fixed trip
// counts (warp w: rows w, w + LTY, ...; lane: columns lane, lane + 32, ...) so every load of a thread
// is issued before the first store (the loads are latency-bound, not bandwidth-bound)
template <int R, int MAG>
__device__ __forceinline__ void load_foot(const StencilParams& sp, const float* __restrict__ A,
                                          const float* __restrict__ B, float a, int hy0, int hx0, float* xs) {
    constexpr int KD = 2 * R + 2;
    constexpr int NR = MAG * (LTY - 1) + KD, NC = MAG * (LTX - 1) + KD;
    constexpr int NRJ = (NR + LTY - 1) / LTY, NCQ = (NC + 31) / 32;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float v[NRJ][NCQ];
#pragma unroll
    for (int j = 0; j < NRJ; ++j) {
        const int r = w + LTY * j;
        const int u = clampi(hy0 + r, 0, sp.H - 1);
        const float* ra = A + (size_t)(u - sp.store_lo) * sp.pitch;
        const float* rb = B ? B + (size_t)(u - sp.store_lo) * sp.pitch : nullptr;
#pragma unroll
        for (int q = 0; q < NCQ; ++q) {
            const int c = lane + 32 * q;
            const int vv = clampi(hx0 + c, 0, sp.W - 1);
            v[j][q] = (r < NR && c < NC) ? (rb ? fmaf(a, __ldg(rb + vv), __ldg(ra + vv)) : __ldg(ra + vv)) : 0.0f;
        }
    }
#pragma unroll
    for (int j = 0; j < NRJ; ++j)
#pragma unroll
        for (int q = 0; q < NCQ; ++q) {
            const int r = w + LTY * j, c = lane + 32 * q;
            if (r < NR && c < NC) xs[r * NC + c] = v[j][q];
        }
}

template <int R, int MAG>
__device__ __forceinline__ float foot_dot(const float* ks, const float* xs, int r0, int c0) {
    constexpr int KD = 2 * R + 2;
    constexpr int nc = MAG * (LTX - 1) + KD;
    float z = 0.0f;
#pragma unroll
    for (int P = 0; P < KD; ++P)
#pragma unroll
        for (int Q = 0; Q < KD; ++Q) z = fmaf(ks[P * KD + Q], xs[(r0 + P) * nc + c0 + Q], z);
    return z;
}

// LR tile t of the grid-stride loops: frame, first LR row and column
__device__ __forceinline__ void lr_tile(const GenParams& gp, int t, int& i, int& a0, int& b0) {
    const int ntx = (gp.lr_w + LTX - 1) / LTX, nty = (gp.lr_h + LTY - 1) / LTY;
    i = t / (ntx * nty);
    const int rem = t - i * ntx * nty, by = rem / ntx;
    a0 = by * LTY;
    b0 = (rem - by * ntx) * LTX;
}
__device__ __forceinline__ int lr_tiles(const GenParams& gp) {
    return ((gp.lr_w + LTX - 1) / LTX) * ((gp.lr_h + LTY - 1) / LTY) * gp.k;
}

template <int PN, int R, int MAG>
__global__ void __launch_bounds__(LTX * LTY) k_gen2_residual(StencilParams sp, GenParams gp, Buffers b, int phase) {
    constexpr int KD = 2 * R + 2;
    constexpr int mag = MAG;   // compile-time stride: divisions and residues become shifts / multiplies
    __shared__ float xs[Foot<R>::NR * Foot<R>::NC];
    __shared__ float ks[KD * KD];
    ScgState* st = b.st;
    if (phase != PH_DEBUG && st->done) return;
    const float alpha = (phase == PH_ITER) ? st->alpha_f : 0.0f;
    const float* X = pick(b.X, st->xcur);
    const float* P = pick(b.P, st->xcur);
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};
    for (int t = blockIdx.x; t < lr_tiles(gp); t += gridDim.x) {   // grid-stride: few CTAs, few partials
        int i, a0, b0;
        lr_tile(gp, t, i, a0, b0);
        __syncthreads();   // the previous tile's footprint is consumed
        load_foot<R, MAG>(sp, X, P, alpha, mag * a0 + gp.sy[i] - R, mag * b0 + gp.sx[i] - R, xs);
        if (tid < KD * KD) ks[tid] = __ldg(gp.taps + (size_t)i * KD * KD + tid);
        __syncthreads();
        const int a = a0 + ty, c = b0 + tx;
        if (a < gp.lr_h && c < gp.lr_w) {
            const size_t idx = ((size_t)i * gp.lr_h + a) * gp.lr_w + c;
            const float e = foot_dot<R, MAG>(ks, xs, mag * ty, mag * tx) - __ldg(gp.lr + idx);
            float v, d1;
            Pen<PN>::val_d1(e, sp.eps, sp.eps2, v, d1);
            gp.w[idx] = d1;
            acc[0] += v;
        }
    }
    block_partials(acc, gp.part_a, gridDim.x, blockIdx.x);
}

template <int PN, int R, int MAG>
__global__ void __launch_bounds__(LTX * LTY) k_gen2_curv_data(StencilParams sp, GenParams gp, Buffers b, int phase) {
    constexpr int KD = 2 * R + 2;
    constexpr int mag = MAG;
    __shared__ float xs[Foot<R>::NR * Foot<R>::NC];
    __shared__ float ps[Foot<R>::NR * Foot<R>::NC];
    __shared__ float ks[KD * KD];
    ScgState* st = b.st;
    if (phase != PH_DEBUG && (st->done || !st->success)) return;
    const int xcur = st->xcur;
    const float* Xn = pick(b.X, xcur ^ 1);
    const float* Pn = pick(b.P, xcur ^ 1);
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    double accd[NSLOT] = {0.0, 0.0, 0.0, 0.0}, tot[NSLOT];
    float cd = 0.0f;
    for (int t = blockIdx.x; t < lr_tiles(gp); t += gridDim.x) {
        int i, a0, b0;
        lr_tile(gp, t, i, a0, b0);
        __syncthreads();
        const int hy0 = mag * a0 + gp.sy[i] - R, hx0 = mag * b0 + gp.sx[i] - R;
        load_foot<R, MAG>(sp, Xn, nullptr, 0.0f, hy0, hx0, xs);
        load_foot<R, MAG>(sp, Pn, nullptr, 0.0f, hy0, hx0, ps);
        if (tid < KD * KD) ks[tid] = __ldg(gp.taps + (size_t)i * KD * KD + tid);
        __syncthreads();
        const int a = a0 + ty, c = b0 + tx;
        if (a < gp.lr_h && c < gp.lr_w) {
            const size_t idx = ((size_t)i * gp.lr_h + a) * gp.lr_w + c;
            const float e = foot_dot<R, MAG>(ks, xs, mag * ty, mag * tx) - __ldg(gp.lr + idx);
            const float ap = foot_dot<R, MAG>(ks, ps, mag * ty, mag * tx);
            cd = fmaf(Pen<PN>::d2(e, sp.eps2) * ap, ap, cd);
        }
    }
    accd[0] = cd;
    if (reduce_partials(accd, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        tot[1] = sum_slot(gp.part_a, 1, gp.nblk_hr);
        tot[2] = sum_slot(gp.part_a, 2, gp.nblk_hr);
        tot[3] = sum_slot(gp.part_a, 3, gp.nblk_hr);
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

// thread t of an HR tile handles column t % HTX of rows t / HTX + {0, 4, 8, 12}
constexpr int HNT = 256, HRPT = HTY * HTX / HNT;   // 4 pixels per thread
constexpr int XSC = HTX + 2 * HH;                   // x' tile row stride (halo HH each side)

template <int PN, int R, int MAG>
__global__ void __launch_bounds__(HNT) k_gen2_grad(StencilParams sp, GenParams gp, Buffers b, int phase) {
    constexpr int KD = 2 * R + 2;
    constexpr int WR = HTY + KD + 1, WC = HTX + KD + 1;   // LR window bound for mag >= 1
    constexpr int FC = 4;                                   // frames per staged chunk
    __shared__ float xs[(HTY + 2 * HH) * XSC];
    __shared__ float ws[FC][WR * WC];
    __shared__ float ts[GMAXK * KD * KD];   // every frame's taps
    ScgState* st = b.st;
    if (phase != PH_DEBUG && st->done) return;
    const float alpha = (phase == PH_ITER) ? st->alpha_f : 0.0f;
    const int xcur = st->xcur, rcur = st->rcur;
    const float* X = pick(b.X, xcur);
    const float* P = pick(b.P, xcur);
    const float* Ro = pick(b.R, rcur);
    float* Rn = pick(b.R, rcur ^ 1);
    constexpr int mag = MAG;
    const int tid = threadIdx.x;
    for (int e = tid; e < gp.k * KD * KD; e += HNT) ts[e] = __ldg(gp.taps + e);   // ordered by the tile loop's barriers
    const int ntx = (sp.W + HTX - 1) / HTX, nty = (sp.row_hi - sp.row_lo + HTY - 1) / HTY;
    const int cx = tid % HTX, ry = tid / HTX;
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // -, R, <r',r'>, <r',r_old>
    for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {   // grid-stride over HR tiles
    const int ty0 = sp.row_lo + (t / ntx) * HTY, tx0 = (t % ntx) * HTX;
    const bool inner = ty0 >= HH && ty0 + HTY + HH <= sp.H && tx0 >= HH && tx0 + HTX + HH <= sp.W;
    __syncthreads();   // the previous tile's x' and windows are consumed
    const int w8 = tid >> 5, lane = tid & 31;
    {   // x' on the tile + halo: warp w rows w, w + 8, w + 16; lanes columns (every load before any store)
        constexpr int XR = HTY + 2 * HH, XRJ = (XR + 7) / 8, XCQ = (XSC + 31) / 32;
        float v[XRJ][XCQ];
#pragma unroll
        for (int j = 0; j < XRJ; ++j) {
            const int r = w8 + 8 * j;
            const int u = clampi(ty0 - HH + r, 0, sp.H - 1);
            const size_t ro = (size_t)(u - sp.store_lo) * sp.pitch;
#pragma unroll
            for (int q = 0; q < XCQ; ++q) {
                const int c = lane + 32 * q;
                const size_t o = ro + clampi(tx0 - HH + c, 0, sp.W - 1);
                v[j][q] = (r < XR && c < XSC) ? fmaf(alpha, __ldg(P + o), __ldg(X + o)) : 0.0f;
            }
        }
#pragma unroll
        for (int j = 0; j < XRJ; ++j)
#pragma unroll
            for (int q = 0; q < XCQ; ++q) {
                const int r = w8 + 8 * j, c = lane + 32 * q;
                if (r < XR && c < XSC) xs[r * XSC + c] = v[j][q];
            }
    }
    float g[HRPT];
#pragma unroll
    for (int k = 0; k < HRPT; ++k) g[k] = 0.0f;
    // data term: rho' of every frame gathered through the residue-class taps (interior pixels), the
    // frames' LR windows staged FC at a time (one barrier pair per chunk)
    const int vx = tx0 + cx;
    for (int i0 = 0; i0 < gp.k; i0 += FC) {
        if (i0 > 0) __syncthreads();   // the previous chunk's windows are consumed
        constexpr int WRJ = (WR + 7) / 8, WCQ = (WC + 31) / 32;
#pragma unroll
        for (int f = 0; f < FC; ++f) {
            const int i = i0 + f;
            if (i >= gp.k) break;
            const int sy = gp.sy[i], sx = gp.sx[i];
            const int alo = floordiv(ty0 - sy - (R + 1), mag), ahi = floordiv(ty0 + HTY - 1 - sy + R, mag);
            const int blo = floordiv(tx0 - sx - (R + 1), mag), bhi = floordiv(tx0 + HTX - 1 - sx + R, mag);
            const int wr = ahi - alo + 1, wc = bhi - blo + 1;
            const float* wi = gp.w + (size_t)i * gp.lr_h * gp.lr_w;
            float v[WRJ][WCQ];
#pragma unroll
            for (int j = 0; j < WRJ; ++j)
#pragma unroll
                for (int q = 0; q < WCQ; ++q) {
                    const int r = w8 + 8 * j, c = lane + 32 * q;
                    const int la = alo + r, lb = blo + c;
                    v[j][q] = (r < wr && c < wc && (unsigned)la < (unsigned)gp.lr_h && (unsigned)lb < (unsigned)gp.lr_w)
                                  ? __ldg(wi + (size_t)la * gp.lr_w + lb) : 0.0f;
                }
#pragma unroll
            for (int j = 0; j < WRJ; ++j)
#pragma unroll
                for (int q = 0; q < WCQ; ++q) {
                    const int r = w8 + 8 * j, c = lane + 32 * q;
                    if (r < wr && c < wc) ws[f][r * WC + c] = v[j][q];
                }
        }
        __syncthreads();
#pragma unroll
        for (int f = 0; f < FC; ++f) {
            const int i = i0 + f;
            if (i >= gp.k) break;
            const int sy = gp.sy[i], sx = gp.sx[i];
            const int alo = floordiv(ty0 - sy - (R + 1), mag), blo = floordiv(tx0 - sx - (R + 1), mag);
            const float* ti = ts + i * KD * KD;
            const float* wf = ws[f];
            const int q0 = ((vx - sx + R) % mag + mag) % mag;   // first Q' (= Q + R) in the residue class
#pragma unroll
            for (int k = 0; k < HRPT; ++k) {
                const int vy = ty0 + ry + 4 * k;
                const int p0 = ((vy - sy + R) % mag + mag) % mag;
                float ga = 0.0f;
                constexpr int NT = (KD + mag - 1) / mag;   // taps per axis in one residue class (at most)
#pragma unroll
                for (int jp = 0; jp < NT; ++jp) {
                    const int Pp = p0 + jp * mag;
                    if (Pp >= KD) break;
                    const int a = (vy - sy - (Pp - R) - alo * mag) / mag;   // window row (exact division)
#pragma unroll
                    for (int jq = 0; jq < NT; ++jq) {
                        const int Qq = q0 + jq * mag;
                        if (Qq >= KD) break;
                        const int c = (vx - sx - (Qq - R) - blo * mag) / mag;
                        ga = fmaf(ti[Pp * KD + Qq], wf[a * WC + c], ga);
                    }
                }
                g[k] += ga;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < HRPT; ++k) {
        const int vy = ty0 + ry + 4 * k, vx = tx0 + cx;
        if (vy >= sp.row_hi || vx >= sp.W) continue;
        float gd = g[k];
        if (vy == 0 || vy == sp.H - 1 || vx == 0 || vx == sp.W - 1) gd = adj_gather(sp, gp, gp.w, vy, vx);   // folds
        const int ly = ry + 4 * k + HH, lx = cx + HH;
        const float xv = xs[ly * XSC + lx];
        float gb = 0.0f;
        if (inner) {   // every pair of the tile lies inside the image: no validity tests
            for (int o = 0; o < gp.noff; ++o) {
                const int dy = gp.offy[o], dx = gp.offx[o];
                const float gm = gp.ogam[o];
                float v, d1;
                charb_val_d1(xv - xs[(ly + dy) * XSC + lx + dx], sp.eps, sp.eps2, v, d1);
                acc[1] = fmaf(gm, v, acc[1]);
                gb = fmaf(gm, d1, gb);
                gb = fmaf(-gm, charb_d1(xs[(ly - dy) * XSC + lx - dx] - xv, sp.eps2), gb);
            }
        } else {
            for (int o = 0; o < gp.noff; ++o) {   // BTV offset list, valid pairs only (|dx|, dy <= HH)
                const int dy = gp.offy[o], dx = gp.offx[o];
                const float gm = gp.ogam[o];
                if (vy + dy < sp.H && vx + dx >= 0 && vx + dx < sp.W) {
                    float v, d1;
                    charb_val_d1(xv - xs[(ly + dy) * XSC + lx + dx], sp.eps, sp.eps2, v, d1);
                    acc[1] = fmaf(gm, v, acc[1]);
                    gb = fmaf(gm, d1, gb);
                }
                if (vy - dy >= 0 && vx - dx >= 0 && vx - dx < sp.W)
                    gb = fmaf(-gm, charb_d1(xs[(ly - dy) * XSC + lx - dx] - xv, sp.eps2), gb);
            }
        }
        const float rn = -fmaf(sp.lam, gb, gd);
        const size_t o = (size_t)(vy - sp.store_lo) * sp.pitch + vx;
        Rn[o] = rn;
        acc[2] = fmaf(rn, rn, acc[2]);
        acc[3] = fmaf(rn, __ldg(Ro + o), acc[3]);
    }
    }   // tiles
    double accd[NSLOT] = {acc[0], acc[1], acc[2], acc[3]}, tot[NSLOT];
    if (reduce_partials(accd, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        tot[0] = sum_slot(gp.part_a, 0, gp.nblk_lr);
        finish_scalars<0>(sp, b, tot, phase);
    }
}

template <int PN>
__global__ void __launch_bounds__(HNT) k_gen2_update(StencilParams sp, GenParams gp, Buffers b, int phase) {
    __shared__ float xs[(HTY + 2 * HH) * XSC];
    __shared__ float ps[(HTY + 2 * HH) * XSC];
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
    const float* P = pick(b.P, xcur);
    const float* R = pick(b.R, rcur);
    float* Xn = pick(b.X, xcur ^ 1);
    float* Pn = pick(b.P, xcur ^ 1);
    const int tid = threadIdx.x;
    const int ntx = (sp.W + HTX - 1) / HTX, nty = (sp.row_hi - sp.row_lo + HTY - 1) / HTY;
    const int cx = tid % HTX, ry = tid / HTX;
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // -, curv BTV, <p,p>, <p,r>
    for (int t = blockIdx.x; t < ntx * nty; t += gridDim.x) {   // grid-stride over HR tiles
    const int ty0 = sp.row_lo + (t / ntx) * HTY, tx0 = (t % ntx) * HTX;
    __syncthreads();
#pragma unroll
    for (int e = tid; e < (HTY + 2 * HH) * XSC; e += HNT) {   // new x, p on the tile + halo
        const int r = e / XSC, c = e - r * XSC;
        const int u = clampi(ty0 - HH + r, 0, sp.H - 1), v = clampi(tx0 - HH + c, 0, sp.W - 1);
        const size_t o = (size_t)(u - sp.store_lo) * sp.pitch + v;
        const float pv = __ldg(P + o);
        xs[e] = fmaf(au, pv, __ldg(X + o));
        ps[e] = fmaf(be, pv, __ldg(R + o));
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < HRPT; ++k) {
        const int uy = ty0 + ry + 4 * k, ux = tx0 + cx;
        if (uy >= sp.row_hi || ux >= sp.W) continue;
        const int ly = ry + 4 * k + HH, lx = cx + HH;
        const float xn = xs[ly * XSC + lx], pn = ps[ly * XSC + lx];
        const size_t o = (size_t)(uy - sp.store_lo) * sp.pitch + ux;
        Xn[o] = xn;
        Pn[o] = pn;
        acc[2] = fmaf(pn, pn, acc[2]);
        acc[3] = fmaf(pn, __ldg(R + o), acc[3]);
        for (int q = 0; q < gp.noff; ++q) {
            const int dy = gp.offy[q], dx = gp.offx[q];
            if (uy + dy < sp.H && ux + dx >= 0 && ux + dx < sp.W) {
                const int j = (ly + dy) * XSC + lx + dx;
                const float tt = xn - xs[j], dp = pn - ps[j];
                acc[1] = fmaf(gp.ogam[q] * charb_d2(tt, sp.eps2), dp * dp, acc[1]);
            }
        }
    }
    }   // tiles
    block_partials(acc, gp.part_a, gridDim.x, blockIdx.x);
}

// ================================================================================================
// Paper-literal finite-difference curvature (NEXT-4, Alg. 1 lines 6-11):
//   sigma = sigma0 / |p|,  delta = p^T (grad J(x + sigma p) - grad J(x)) / sigma
// with both gradients evaluated per pixel in fp64 from the fp32 iterate (in fp32 the probe
// displacement sigma p is below one ulp of x, reading 16).  Replaces the data-curvature pass.
// ================================================================================================
__device__ __forceinline__ double fd_rho1(int pn, double eps, double t) {
    return pn == 2 ? 2.0 * t : t / sqrt(fma(t, t, eps * eps));
}
__device__ __forceinline__ double fd_psi1(double eps, double t) { return t / sqrt(fma(t, t, eps * eps)); }

// sigma of this pass from the update pass's per-CTA <p,p> slots (same fixed order in every CTA)
__device__ double fd_sigma(const GenParams& gp) {
    __shared__ double s_sig;
    if (threadIdx.x == 0) {
        double pp = 0.0;
        for (int j = 0; j < gp.nblk_hr; ++j) pp += __ldcg(gp.part_a + (size_t)2 * gp.nblk_hr + j);
        s_sig = gp.sigma0 / sqrt(pp);
    }
    __syncthreads();
    return s_sig;
}

__device__ double fd_fwd(const StencilParams& sp, const GenParams& gp, const float* X, const float* P, double sig,
                         int i, int a, int b) {
    const int by = gp.mag * a + gp.sy[i], bx = gp.mag * b + gp.sx[i];
    double z = 0.0;
    for (int Pp = -gp.R; Pp <= gp.R + 1; ++Pp) {
        const int u = clampi(by + Pp, 0, sp.H - 1);
        for (int Qq = -gp.R; Qq <= gp.R + 1; ++Qq) {
            const size_t o = (size_t)(u - sp.store_lo) * sp.pitch + clampi(bx + Qq, 0, sp.W - 1);
            z = fma((double)tapk(gp, i, Pp, Qq), fma(sig, (double)__ldg(P + o), (double)__ldg(X + o)), z);
        }
    }
    return z;
}

template <int PN>
__global__ void __launch_bounds__(GT) k_gen_fd_residual(StencilParams sp, GenParams gp, Buffers b, int phase) {
    ScgState* st = b.st;
    if (phase != PH_DEBUG && (st->done || !st->success)) return;
    const int xcur = st->xcur;
    const float* Xn = pick(b.X, xcur ^ 1);
    const float* Pn = pick(b.P, xcur ^ 1);
    const double sig = fd_sigma(gp);
    const long long n = (long long)gp.k * gp.lr_h * gp.lr_w;
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx >= n) return;
    const int i = (int)(idx / ((long long)gp.lr_h * gp.lr_w));
    const int rem = (int)(idx - (long long)i * gp.lr_h * gp.lr_w);
    const int a = rem / gp.lr_w, c = rem - a * gp.lr_w;
    const double y = (double)__ldg(gp.lr + idx);
    const double e1 = fd_fwd(sp, gp, Xn, Pn, 0.0, i, a, c) - y;
    const double e2 = fd_fwd(sp, gp, Xn, Pn, sig, i, a, c) - y;
    gp.wd[idx] = fd_rho1(PN, (double)sp.eps, e2) - fd_rho1(PN, (double)sp.eps, e1);
}

template <int PN>
__global__ void __launch_bounds__(GT) k_gen_fd_grad(StencilParams sp, GenParams gp, Buffers b, int phase) {
    ScgState* st = b.st;
    if (phase != PH_DEBUG && (st->done || !st->success)) return;
    const int xcur = st->xcur;
    const float* Xn = pick(b.X, xcur ^ 1);
    const float* Pn = pick(b.P, xcur ^ 1);
    const double sig = fd_sigma(gp), eps = sp.eps;
    double accd[NSLOT] = {0.0, 0.0, 0.0, 0.0}, tot[NSLOT];
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx < (long long)sp.H * sp.W) {
        const int vy = (int)(idx / sp.W), vx = (int)(idx - (long long)vy * sp.W);
        // data term: transpose of the clamped correlation applied to rho'(e2) - rho'(e1), in fp64
        const int ylo = vy == 0 ? gp.fy_lo : vy, yhi = vy == sp.H - 1 ? gp.fy_hi : vy;
        const int xlo = vx == 0 ? gp.fx_lo : vx, xhi = vx == sp.W - 1 ? gp.fx_hi : vx;
        double gd = 0.0;
        for (int yy = ylo; yy <= yhi; ++yy)
            for (int xx = xlo; xx <= xhi; ++xx)
                for (int i = 0; i < gp.k; ++i)
                    for (int Pp = -gp.R; Pp <= gp.R + 1; ++Pp) {
                        const int ny = yy - gp.sy[i] - Pp;
                        if (ny < 0 || ny % gp.mag) continue;
                        const int a = ny / gp.mag;
                        if (a >= gp.lr_h) continue;
                        for (int Qq = -gp.R; Qq <= gp.R + 1; ++Qq) {
                            const int nx = xx - gp.sx[i] - Qq;
                            if (nx < 0 || nx % gp.mag) continue;
                            const int bb = nx / gp.mag;
                            if (bb >= gp.lr_w) continue;
                            gd = fma((double)tapk(gp, i, Pp, Qq), gp.wd[((size_t)i * gp.lr_h + a) * gp.lr_w + bb], gd);
                        }
                    }
        // BTV: psi'(D x2) - psi'(D x1) per valid pair, x2 = x + sigma p
        auto X1 = [&](int y, int x) { return (double)__ldg(Xn + (size_t)(y - sp.store_lo) * sp.pitch + x); };
        auto X2 = [&](int y, int x) {
            const size_t o = (size_t)(y - sp.store_lo) * sp.pitch + x;
            return fma(sig, (double)__ldg(Pn + o), (double)__ldg(Xn + o));
        };
        double gb = 0.0;
        const double x1 = X1(vy, vx), x2 = X2(vy, vx);
        for (int o = 0; o < gp.noff; ++o) {
            const int dy = gp.offy[o], dx = gp.offx[o];
            const double gm = (double)gp.ogam[o];
            if (vy + dy < sp.H && vx + dx >= 0 && vx + dx < sp.W)
                gb += gm * (fd_psi1(eps, x2 - X2(vy + dy, vx + dx)) - fd_psi1(eps, x1 - X1(vy + dy, vx + dx)));
            if (vy - dy >= 0 && vx - dx >= 0 && vx - dx < sp.W)
                gb -= gm * (fd_psi1(eps, X2(vy - dy, vx - dx) - x2) - fd_psi1(eps, X1(vy - dy, vx - dx) - x1));
        }
        const double pv = (double)__ldg(Pn + (size_t)(vy - sp.store_lo) * sp.pitch + vx);
        accd[0] = pv * (gd + (double)sp.lam * gb);
    }
    if (reduce_partials(accd, b.part, gridDim.x, blockIdx.x, &st->counter, tot)) {
        tot[0] = tot[0] / sig;   // delta = p^T (grad J(x + sigma p) - grad J(x)) / sigma (BTV included)
        tot[1] = 0.0;
        tot[2] = sum_slot(gp.part_a, 2, gp.nblk_hr);
        tot[3] = sum_slot(gp.part_a, 3, gp.nblk_hr);
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

// ---- debug: forward and adjoint on natural-layout HR buffers -------------------------------------
__global__ void k_gen_forward(StencilParams sp, GenParams gp, const float* __restrict__ x, float* __restrict__ y) {
    const long long n = (long long)gp.k * gp.lr_h * gp.lr_w;
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx >= n) return;
    const int i = (int)(idx / ((long long)gp.lr_h * gp.lr_w));
    const int rem = (int)(idx - (long long)i * gp.lr_h * gp.lr_w);
    const int a = rem / gp.lr_w, c = rem - a * gp.lr_w;
    y[idx] = fwd_sample(sp, gp, x, x, 0.0f, i, a, c);
}

__global__ void k_gen_adjoint(StencilParams sp, GenParams gp, const float* __restrict__ w, float* __restrict__ g) {
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx >= (long long)sp.H * sp.W) return;
    const int vy = (int)(idx / sp.W), vx = (int)(idx - (long long)vy * sp.W);
    g[(size_t)(vy - sp.store_lo) * sp.pitch + vx] = adj_gather(sp, gp, w, vy, vx);
}

// multi-image interpolation fusion for any geometry: the first integer-phase frame covering
// an HR site wins, uncovered sites keep the bilinear estimate already in `out` (natural layout)
__global__ void k_gen_interp(StencilParams sp, GenParams gp, float* __restrict__ out, int out_pitch) {
    const long long idx = (long long)blockIdx.x * GT + threadIdx.x;
    if (idx >= (long long)sp.H * sp.W) return;
    const int u = (int)(idx / sp.W), v = (int)(idx - (long long)u * sp.W);
    for (int i = 0; i < gp.k; ++i) {
        if (!gp.integer_phase[i]) continue;
        const int ny = u - gp.sy[i], nx = v - gp.sx[i];
        if (ny < 0 || nx < 0 || ny % gp.mag || nx % gp.mag) continue;
        const int a = ny / gp.mag, b = nx / gp.mag;
        if (a >= gp.lr_h || b >= gp.lr_w) continue;
        out[(size_t)u * out_pitch + v] = __ldg(gp.lr + ((size_t)i * gp.lr_h + a) * gp.lr_w + b);
        return;
    }
}

inline unsigned nblk(long long n) { return (unsigned)((n + GT - 1) / GT); }

}  // namespace

namespace {
dim3 lr_grid(const GenParams& gp) { return dim3(gp.nblk_lr); }
dim3 hr_grid(const StencilParams&, const GenParams& gp) { return dim3(gp.nblk_hr); }
}  // namespace

// grid-stride CTAs of the tiled passes: all tiles, capped at `cap` CTAs (a few waves of the device)
unsigned gen_blocks_lr(int k, int lr_h, int lr_w, int cap) {
    const long long n = (long long)((lr_w + LTX - 1) / LTX) * ((lr_h + LTY - 1) / LTY) * k;
    return (unsigned)std::min<long long>(n, cap);
}
unsigned gen_blocks_hr(int W, int rows, int cap) {
    const long long n = (long long)((W + HTX - 1) / HTX) * ((rows + HTY - 1) / HTY);
    return (unsigned)std::min<long long>(n, cap);
}

#define FL_GEN_RM(KERNEL, PN_, R_, GRID, BLOCK)                                                      \
    switch (gp.mag) {                                                                               \
        case 1: KERNEL<PN_, R_, 1><<<GRID, BLOCK, 0, s>>>(sp, gp, b, phase); break;                \
        case 2: KERNEL<PN_, R_, 2><<<GRID, BLOCK, 0, s>>>(sp, gp, b, phase); break;                \
        case 3: KERNEL<PN_, R_, 3><<<GRID, BLOCK, 0, s>>>(sp, gp, b, phase); break;                \
        case 4: KERNEL<PN_, R_, 4><<<GRID, BLOCK, 0, s>>>(sp, gp, b, phase); break;                \
        default: return cudaErrorInvalidValue;                                                      \
    }
#define FL_GEN_R(KERNEL, PN_, GRID, BLOCK)                                                            \
    switch (gp.R) {                                                                                 \
        case 0: FL_GEN_RM(KERNEL, PN_, 0, GRID, BLOCK) break;                                      \
        case 1: FL_GEN_RM(KERNEL, PN_, 1, GRID, BLOCK) break;                                      \
        case 2: FL_GEN_RM(KERNEL, PN_, 2, GRID, BLOCK) break;                                      \
        default: return cudaErrorInvalidValue;                                                      \
    }

cudaError_t launch_gen_value_grad(int bw, int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b,
                                  int phase, cudaStream_t s) {
    (void)bw;   // the general kernels walk the plan's BTV offset list (quadrant or Farsiu)
    if (gp.fused) return launch_gen3_vg(pn, sp, gp, b, phase, s);
    const dim3 lb(LTX * LTY);
    if (pn == 2) { FL_GEN_R(k_gen2_residual, 2, lr_grid(gp), lb) } else { FL_GEN_R(k_gen2_residual, 1, lr_grid(gp), lb) }
    if (pn == 2) { FL_GEN_R(k_gen2_grad, 2, hr_grid(sp, gp), HNT) } else { FL_GEN_R(k_gen2_grad, 1, hr_grid(sp, gp), HNT) }
    return cudaGetLastError();
}

cudaError_t launch_gen_update_curv(int bw, int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b,
                                   int phase, cudaStream_t s) {
    (void)bw;
    if (gp.fused && !gp.fd) return launch_gen3_uc(pn, sp, gp, b, phase, s);
    const dim3 lb(LTX * LTY);
    if (pn == 2) k_gen2_update<2><<<hr_grid(sp, gp), HNT, 0, s>>>(sp, gp, b, phase);
    else k_gen2_update<1><<<hr_grid(sp, gp), HNT, 0, s>>>(sp, gp, b, phase);
    if (gp.fd) {   // paper-literal finite-difference curvature in fp64 instead of the exact data curvature
        const unsigned nl = nblk((long long)gp.k * gp.lr_h * gp.lr_w), nh = nblk((long long)sp.H * sp.W);
        if (pn == 2) {
            k_gen_fd_residual<2><<<nl, GT, 0, s>>>(sp, gp, b, phase);
            k_gen_fd_grad<2><<<nh, GT, 0, s>>>(sp, gp, b, phase);
        } else {
            k_gen_fd_residual<1><<<nl, GT, 0, s>>>(sp, gp, b, phase);
            k_gen_fd_grad<1><<<nh, GT, 0, s>>>(sp, gp, b, phase);
        }
        return cudaGetLastError();
    }
    if (pn == 2) { FL_GEN_R(k_gen2_curv_data, 2, lr_grid(gp), lb) } else { FL_GEN_R(k_gen2_curv_data, 1, lr_grid(gp), lb) }
    return cudaGetLastError();
}
#undef FL_GEN_R
#undef FL_GEN_RM

cudaError_t launch_gen_forward(const StencilParams& sp, const GenParams& gp, const float* x, float* y, cudaStream_t s) {
    k_gen_forward<<<nblk((long long)gp.k * gp.lr_h * gp.lr_w), GT, 0, s>>>(sp, gp, x, y);
    return cudaGetLastError();
}
cudaError_t launch_gen_adjoint(const StencilParams& sp, const GenParams& gp, const float* w, float* g, cudaStream_t s) {
    k_gen_adjoint<<<nblk((long long)sp.H * sp.W), GT, 0, s>>>(sp, gp, w, g);
    return cudaGetLastError();
}
cudaError_t launch_gen_interp(const StencilParams& sp, const GenParams& gp, float* out, int out_pitch, cudaStream_t s) {
    k_gen_interp<<<nblk((long long)sp.H * sp.W), GT, 0, s>>>(sp, gp, out, out_pitch);
    return cudaGetLastError();
}
unsigned gen_blocks(long long n) { return nblk(n); }   // CTAs of a one-pixel-per-thread pass

}  // namespace flmisr
