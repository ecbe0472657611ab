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

// transpose of the clamped strided correlation at HR pixel (vy, vx), from LR-layout weights w
__device__ float adj_gather(const StencilParams& sp, const GenParams& gp, const float* __restrict__ w, int vy, int vx) {
    const int ylo = vy == 0 ? gp.fy_lo : vy, yhi = vy == sp.H - 1 ? gp.fy_hi : vy;
    const int xlo = vx == 0 ? gp.fx_lo : vx, xhi = vx == sp.W - 1 ? gp.fx_hi : vx;
    float g = 0.0f;
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
                        const int b = nx / gp.mag;
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

cudaError_t launch_gen_value_grad(int bw, int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b,
                                  int phase, cudaStream_t s) {
    const long long nlr = (long long)gp.k * gp.lr_h * gp.lr_w, nhr = (long long)sp.H * sp.W;
    if (pn == 2) k_gen_residual<2><<<nblk(nlr), GT, 0, s>>>(sp, gp, b, phase);
    else k_gen_residual<1><<<nblk(nlr), GT, 0, s>>>(sp, gp, b, phase);
    (void)bw;   // the general kernels walk the plan's BTV offset list (quadrant or Farsiu)
    if (pn == 2) k_gen_grad<2><<<nblk(nhr), GT, 0, s>>>(sp, gp, b, phase);
    else k_gen_grad<1><<<nblk(nhr), GT, 0, s>>>(sp, gp, b, phase);
    return cudaGetLastError();
}

cudaError_t launch_gen_update_curv(int bw, int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b,
                                   int phase, cudaStream_t s) {
    const long long nlr = (long long)gp.k * gp.lr_h * gp.lr_w, nhr = (long long)sp.H * sp.W;
    (void)bw;
    if (pn == 2) k_gen_update<2><<<nblk(nhr), GT, 0, s>>>(sp, gp, b, phase);
    else k_gen_update<1><<<nblk(nhr), GT, 0, s>>>(sp, gp, b, phase);
    if (pn == 2) k_gen_curv_data<2><<<nblk(nlr), GT, 0, s>>>(sp, gp, b, phase);
    else k_gen_curv_data<1><<<nblk(nlr), GT, 0, s>>>(sp, gp, b, phase);
    return cudaGetLastError();
}

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
