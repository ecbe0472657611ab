// flmisr_kernels.cu -- sm_100a kernels of the FL-MISR SCG hot path (arXiv 2108.04315).
//
// Polyphase fast path: the K = mag^2 LR frames are interleaved once into an
// HR-grid image Y with Y(mag*a + s_i) = y_i(a) (ingest), so every HR pixel u carries exactly one LR
// sample and the forward model A_i = D B M_i (Eq. sisr) becomes a unit-stride HR stencil
//     z(u) = sum_{P,Q} kappa(P,Q) x~(u + (P,Q))         (x~ = clamp-extended x, reading 4)
// with residual e(u) = z(u) - Y(u).  Its adjoint (zero-fill upsample, transposed blur, inverse
// shift; north_star) is the kappa-correlation of the zero-padded weight image w = rho'(e), folded
// back onto the edge pixels where the forward clamped.
//
// Per accepted SCG pass there are two stencil kernels (both HBM-bound):
//   k_update_curv : x <- x + alpha p, p <- r + beta p (Alg. 1 lines 14, 20) and the
//                   exact directional curvature delta = p^T Hess J p, <p,p>, <p,r> (lines 6-12).
//   k_value_grad  : f_new = J(x + alpha p) (line 16) and, speculatively in the same pass,
//                   r_new = -grad J(x + alpha p) with <r_new,r_new>, <r_new,r_old> (line 18).
// Each CTA reduces its partials with warp shuffles into one fp64 slot; the last CTA to finish sums
// the slots in a fixed order (deterministic, no float atomics) and runs Moller's scalar logic on
// device (single GPU), so there is no host round-trip inside the loop.
#include <cstdint>
#include <cuda_runtime.h>

#include "flmisr_common.cuh"
#include "flmisr_internal.h"

namespace flmisr {

// ------------------------------------------------------------------------------------------------
// Tile staging helpers.  A region of RH x RW floats whose origin is global (gr0, gc0) is loaded
// with clamp-to-image indexing (reading 4: x~ is the clamp extension), from storage rows
// [store_lo, store_hi).  gc0 and RW are multiples of 4 so interior chunks move as float4.
// ------------------------------------------------------------------------------------------------
template <int RH, int RW, typename F>
__device__ __forceinline__ void load_region(const StencilParams& sp, int gr0, int gc0, F&& fn) {
    constexpr int CH = RW / 4;
    for (int idx = threadIdx.x; idx < RH * CH; idx += NTHREADS) {
        int lr = idx / CH, ch = idx - lr * CH;
        int gr = clampi(gr0 + lr, 0, sp.H - 1);
        gr = clampi(gr, sp.store_lo, sp.store_hi - 1);
        size_t rowoff = (size_t)(gr - sp.store_lo) * sp.pitch;
        int gc = gc0 + 4 * ch;
        if (gc >= 0 && gc + 3 < sp.W) {
            fn(lr, 4 * ch, rowoff + gc, true, 0, 0, 0, 0);
        } else {
            int c0 = clampi(gc, 0, sp.W - 1), c1 = clampi(gc + 1, 0, sp.W - 1);
            int c2 = clampi(gc + 2, 0, sp.W - 1), c3 = clampi(gc + 3, 0, sp.W - 1);
            fn(lr, 4 * ch, rowoff, false, c0, c1, c2, c3);
        }
    }
}

__device__ __forceinline__ float4 ld4(const float* p, size_t off, bool vec, int c0, int c1, int c2, int c3) {
    if (vec) return __ldg(reinterpret_cast<const float4*>(p + off));
    return make_float4(__ldg(p + off + c0), __ldg(p + off + c1), __ldg(p + off + c2), __ldg(p + off + c3));
}

// ------------------------------------------------------------------------------------------------
// Kernel: value + gradient at x' = x + alpha p (one pass; Alg. 1 lines 14-19).
// ------------------------------------------------------------------------------------------------
template <int KR, int BW, int PN>
__global__ void __launch_bounds__(NTHREADS) k_value_grad(StencilParams sp, Buffers b, int phase) {
    constexpr int HX = (2 * KR > BW - 1) ? 2 * KR : BW - 1;   // x' halo
    constexpr int HXC = (HX + 3) / 4 * 4;                     // column halo rounded to float4
    constexpr int SXH = TY + 2 * HX, SXW = TX + 2 * HXC;
    constexpr int SWH = TY + 2 * KR, SWW = TX + 2 * KR;
    constexpr int KD = 2 * KR + 1;
    __shared__ float sX[SXH * SXW];
    __shared__ float sW[SWH * SWW];

    ScgState* st = b.st;
    if (phase != PH_DEBUG && st->done) return;
    const int xcur = st->xcur, rcur = st->rcur;
    const float alpha = (phase == PH_ITER) ? st->alpha_f : 0.0f;
    const float* __restrict__ X = pick(b.X, xcur);
    const float* __restrict__ P = pick(b.P, xcur);
    const float* __restrict__ Rold = pick(b.R, rcur);
    float* __restrict__ Rnew = pick(b.R, rcur ^ 1);

    const int tile = blockIdx.y * sp.tiles_x + blockIdx.x;
    const int ntiles = sp.tiles_x * sp.tiles_y;
    const int r0 = sp.tile_row0 + blockIdx.y * TY, c0 = blockIdx.x * TX;
    const int H = sp.H, W = sp.W;

    // stage 1: x' = x + alpha p on the tile + HX halo (clamp-extended)
    load_region<SXH, SXW>(sp, r0 - HX, c0 - HXC,
                          [&](int lr, int lc, size_t off, bool vec, int a0, int a1, int a2, int a3) {
                              float4 xv = ld4(X, off, vec, a0, a1, a2, a3);
                              float4 pv = ld4(P, off, vec, a0, a1, a2, a3);
                              float* d = sX + lr * SXW + lc;
                              d[0] = fmaf(alpha, pv.x, xv.x);
                              d[1] = fmaf(alpha, pv.y, xv.y);
                              d[2] = fmaf(alpha, pv.z, xv.z);
                              d[3] = fmaf(alpha, pv.w, xv.w);
                          });
    __syncthreads();

    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // D, R, <r',r'>, <r',r_old>
    const float eps = sp.eps, eps2 = sp.eps2;

    // stage 2: w = rho'(z - Y) on the tile + KR halo (zero outside the image); data value on the tile
    for (int idx = threadIdx.x; idx < SWH * SWW; idx += NTHREADS) {
        int i = idx / SWW, j = idx - i * SWW;
        int gr = r0 - KR + i, gc = c0 - KR + j;
        float wv = 0.0f;
        if (gr >= 0 && gr < H && gc >= 0 && gc < W) {
            float z = 0.0f;
            const float* base = sX + (i - KR + HX - KR) * SXW + (j - KR + HXC - KR);
#pragma unroll
            for (int P_ = 0; P_ < KD; ++P_)
#pragma unroll
                for (int Q_ = 0; Q_ < KD; ++Q_) z = fmaf(sp.taps[P_ * KD + Q_], base[P_ * SXW + Q_], z);
            float e = z - __ldg(b.Y + (size_t)(gr - sp.store_lo) * sp.pitch + gc);
            float v, d1;
            Pen<PN>::val_d1(e, eps, eps2, v, d1);
            wv = d1;
            if (i >= KR && i < KR + TY && j >= KR && j < KR + TX && gr >= sp.row_lo && gr < sp.row_hi) acc[0] += v;
        }
        sW[idx] = wv;
    }
    __syncthreads();

    // stage 3: g = A^T w (+ border fold) + lambda grad R; BTV value; r' = -g
    const float lam = sp.lam;
    for (int idx = threadIdx.x; idx < TY * TX; idx += NTHREADS) {
        int ly = idx / TX, lx = idx - ly * TX;
        int vy = r0 + ly, vx = c0 + lx;
        if (vy >= sp.row_hi || vx >= W) continue;
        // adjoint: g(v) = sum_{P,Q} kappa(P,Q) w(v - (P,Q))  (zero-padded w)
        float g = 0.0f;
        {
            const float* base = sW + (ly + KR + KR) * SWW + (lx + KR + KR);
#pragma unroll
            for (int P_ = 0; P_ < KD; ++P_)
#pragma unroll
                for (int Q_ = 0; Q_ < KD; ++Q_) g = fmaf(sp.taps[P_ * KD + Q_], base[-P_ * SWW - Q_], g);
        }
        if (KR > 0 && (vy == 0 || vy == H - 1 || vx == 0 || vx == W - 1)) {
            // fold: add g_ext(v') for virtual v' != v outside the image with clamp(v') = v
            int ylo = (vy == 0) ? -KR : vy, yhi = (vy == H - 1) ? H - 1 + KR : vy;
            int xlo = (vx == 0) ? -KR : vx, xhi = (vx == W - 1) ? W - 1 + KR : vx;
            for (int yy = ylo; yy <= yhi; ++yy)
                for (int xx = xlo; xx <= xhi; ++xx) {
                    if (yy == vy && xx == vx) continue;
                    for (int P_ = 0; P_ < KD; ++P_)
                        for (int Q_ = 0; Q_ < KD; ++Q_) {
                            int uy = yy - (P_ - KR), ux = xx - (Q_ - KR);
                            if (uy < 0 || uy >= H || ux < 0 || ux >= W) continue;
                            g = fmaf(sp.taps[P_ * KD + Q_], sW[(uy - r0 + KR) * SWW + (ux - c0 + KR)], g);
                        }
                }
        }
        // BTV: pairs (v, v+d) owned by v (value + both endpoints' gradient), pairs (v-d, v) gradient
        float gb = 0.0f;
        const float xv = sX[(ly + HX) * SXW + lx + HXC];
#pragma unroll
        for (int dy = 0; dy < BW; ++dy)
#pragma unroll
            for (int dx = 0; dx < BW; ++dx) {
                if (dy == 0 && dx == 0) continue;
                const float gm = sp.gam[dy * MAXBW + dx];
                if (vy + dy < H && vx + dx < W) {
                    float t = xv - sX[(ly + HX + dy) * SXW + lx + HXC + dx];
                    float v, d1;
                    charb_val_d1(t, eps, eps2, v, d1);
                    acc[1] = fmaf(gm, v, acc[1]);
                    gb = fmaf(gm, d1, gb);
                }
                if (vy - dy >= 0 && vx - dx >= 0) {
                    float t = sX[(ly + HX - dy) * SXW + lx + HXC - dx] - xv;
                    gb = fmaf(-gm, charb_d1(t, eps2), gb);
                }
            }
        float rn = -fmaf(lam, gb, g);
        size_t off = (size_t)(vy - sp.store_lo) * sp.pitch + vx;
        float ro = __ldg(Rold + off);
        Rnew[off] = rn;
        acc[2] = fmaf(rn, rn, acc[2]);
        acc[3] = fmaf(rn, ro, acc[3]);
        // band mode: owned boundary rows of the candidate go to the neighbours (inner border)
        if (b.send_top && vy - sp.row_lo < b.eta) b.send_top[(size_t)(vy - sp.row_lo) * sp.pitch + vx] = rn;
        if (b.send_bot && sp.row_hi - 1 - vy < b.eta) b.send_bot[(size_t)(vy - (sp.row_hi - b.eta)) * sp.pitch + vx] = rn;
    }

    double tot[NSLOT], accd[NSLOT] = {acc[0], acc[1], acc[2], acc[3]};
    if (reduce_partials(accd, b.part, ntiles, tile, &st->counter, tot)) finish_scalars<0>(sp, b, tot, phase);
}

// ------------------------------------------------------------------------------------------------
// Kernel: update x <- x + alpha_upd p, p <- r + beta p, and curvature at the new (x, p).
// ------------------------------------------------------------------------------------------------
template <int KR, int BW, int PN>
__global__ void __launch_bounds__(NTHREADS) k_update_curv(StencilParams sp, Buffers b, int phase) {
    constexpr int HK = (KR > BW - 1) ? KR : BW - 1;
    constexpr int HKC = (HK + 3) / 4 * 4;
    constexpr int SH = TY + 2 * HK, SW = TX + 2 * HKC;
    constexpr int KD = 2 * KR + 1;
    __shared__ float sXn[SH * SW];
    __shared__ float sPn[SH * SW];

    ScgState* st = b.st;
    if (phase != PH_DEBUG) {
        if (st->done) return;
        if (!st->success) {   // rejected step: delta is reused, only the scalar pre-value step runs
            if (sp.world == 1 && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) scg_pre_value(st);
            return;
        }
    }
    const int xcur = st->xcur, rcur = st->rcur;
    const float au = (phase == PH_DEBUG) ? 0.0f : st->alpha_upd_f;
    const float be = (phase == PH_DEBUG) ? 0.0f : st->beta_f;
    const float* __restrict__ X = pick(b.X, xcur);
    const float* __restrict__ P = pick(b.P, xcur);
    const float* __restrict__ R = pick(b.R, rcur);
    float* __restrict__ Xn = pick(b.X, xcur ^ 1);
    float* __restrict__ Pn = pick(b.P, xcur ^ 1);

    const int tile = blockIdx.y * sp.tiles_x + blockIdx.x;
    const int ntiles = sp.tiles_x * sp.tiles_y;
    const int r0 = sp.tile_row0 + blockIdx.y * TY, c0 = blockIdx.x * TX;
    const int H = sp.H, W = sp.W;
    float acc[NSLOT] = {0.f, 0.f, 0.f, 0.f};   // curv data, curv BTV, <p,p>, <p,r>

    load_region<SH, SW>(sp, r0 - HK, c0 - HKC, [&](int lr, int lc, size_t off, bool vec, int a0, int a1, int a2, int a3) {
        float4 xv = ld4(X, off, vec, a0, a1, a2, a3);
        float4 pv = ld4(P, off, vec, a0, a1, a2, a3);
        float4 rv = ld4(R, off, vec, a0, a1, a2, a3);
        float xn[4] = {fmaf(au, pv.x, xv.x), fmaf(au, pv.y, xv.y), fmaf(au, pv.z, xv.z), fmaf(au, pv.w, xv.w)};
        float pn[4] = {fmaf(be, pv.x, rv.x), fmaf(be, pv.y, rv.y), fmaf(be, pv.z, rv.z), fmaf(be, pv.w, rv.w)};
        float rr[4] = {rv.x, rv.y, rv.z, rv.w};
        float* dx_ = sXn + lr * SW + lc;
        float* dp_ = sPn + lr * SW + lc;
#pragma unroll
        for (int e = 0; e < 4; ++e) { dx_[e] = xn[e]; dp_[e] = pn[e]; }
        // owned interior element: write the new iterate, accumulate <p,p>, <p,r>
        int gr = r0 - HK + lr;
        if (lr >= HK && lr < HK + TY && gr < sp.row_hi && vec && lc >= HKC && lc < HKC + TX) {
            *reinterpret_cast<float4*>(Xn + off) = make_float4(xn[0], xn[1], xn[2], xn[3]);
            *reinterpret_cast<float4*>(Pn + off) = make_float4(pn[0], pn[1], pn[2], pn[3]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                acc[2] = fmaf(pn[e], pn[e], acc[2]);
                acc[3] = fmaf(pn[e], rr[e], acc[3]);
            }
        } else if (lr >= HK && lr < HK + TY && gr < sp.row_hi && !vec && lc >= HKC && lc < HKC + TX) {
            // partial float4 at the right image edge: element-wise, skip clamped duplicates
            int gc = c0 - HKC + lc;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (gc + e < W) {
                    Xn[off + gc + e] = xn[e];
                    Pn[off + gc + e] = pn[e];
                    acc[2] = fmaf(pn[e], pn[e], acc[2]);
                    acc[3] = fmaf(pn[e], rr[e], acc[3]);
                }
            }
        }
    });
    __syncthreads();

    const float eps2 = sp.eps2;
    {
        for (int idx = threadIdx.x; idx < TY * TX; idx += NTHREADS) {
            int ly = idx / TX, lx = idx - ly * TX;
            int uy = r0 + ly, ux = c0 + lx;
            if (uy >= sp.row_hi || ux >= W) continue;
            float z = 0.0f, ap = 0.0f;
            const float* bx = sXn + (ly + HK - KR) * SW + (lx + HKC - KR);
            const float* bp = sPn + (ly + HK - KR) * SW + (lx + HKC - KR);
#pragma unroll
            for (int P_ = 0; P_ < KD; ++P_)
#pragma unroll
                for (int Q_ = 0; Q_ < KD; ++Q_) {
                    float kk = sp.taps[P_ * KD + Q_];
                    z = fmaf(kk, bx[P_ * SW + Q_], z);
                    ap = fmaf(kk, bp[P_ * SW + Q_], ap);
                }
            float e = z - __ldg(b.Y + (size_t)(uy - sp.store_lo) * sp.pitch + ux);
            acc[0] = fmaf(Pen<PN>::d2(e, eps2), ap * ap, acc[0]);
            const float xu = sXn[(ly + HK) * SW + lx + HKC], pu = sPn[(ly + HK) * SW + lx + HKC];
#pragma unroll
            for (int dy = 0; dy < BW; ++dy)
#pragma unroll
                for (int dx = 0; dx < BW; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    if (uy + dy < H && ux + dx < W) {
                        float t = xu - sXn[(ly + HK + dy) * SW + lx + HKC + dx];
                        float dp = pu - sPn[(ly + HK + dy) * SW + lx + HKC + dx];
                        acc[1] = fmaf(sp.gam[dy * MAXBW + dx] * charb_d2(t, eps2), dp * dp, acc[1]);
                    }
                }
        }
    }
    (void)H;
    double tot[NSLOT], accd[NSLOT] = {acc[0], acc[1], acc[2], acc[3]};
    if (reduce_partials(accd, b.part, ntiles, tile, &st->counter, tot)) {
        if (threadIdx.x == 0 && phase != PH_DEBUG) st->xcur = xcur ^ 1;
        finish_scalars<1>(sp, b, tot, phase);
    }
}

// ------------------------------------------------------------------------------------------------
// Multi-GPU scalar kernels: the rank sums were allgathered into b.part[0 .. world*NSLOT); sum them
// in rank order (identical on every rank) and run the scalar logic (Alg. 1 "Central" lines).
// ------------------------------------------------------------------------------------------------
// rank sums -> consensus sums.  Default: fp64 records of NSLOT (band affine applied), summed in rank
// order.  det mode (sp.det): records of FXW exact 128-bit words, summed exactly, converted once, with
// the whole image's affine correction -- the same bits at every band count.
__device__ void rank_totals(const StencilParams& sp, const Buffers& b, int world, int which, double (&t)[NSLOT]) {
    if (!sp.det) {
        for (int k = 0; k < NSLOT; ++k) t[k] = 0.0;
        for (int r = 0; r < world; ++r)
            for (int k = 0; k < NSLOT; ++k) t[k] += b.part[r * NSLOT + k];
        return;
    }
    const __int128* w = reinterpret_cast<const __int128*>(b.part);
    __int128 s[FXW];
    for (int k = 0; k < FXW; ++k) s[k] = 0;
    for (int r = 0; r < world; ++r)
        for (int k = 0; k < FXW; ++k) s[k] += w[r * FXW + k];
    const double* aff = which == 0 ? sp.aff_vg : sp.aff_uc;
    const double* off = which == 0 ? sp.det_off_vg : sp.det_off_uc;
    for (int k = 0; k < NSLOT; ++k)
        t[k] = s[NSLOT] != 0 ? __longlong_as_double(0x7ff8000000000000ll) : fx_to_double(s[k]) * aff[k] + off[k];
}

__global__ void k_scalar_after_value(const __grid_constant__ StencilParams sp, Buffers b, int world, int phase) {
    ScgState* s = b.st;
    if (s->done) return;
    double t[NSLOT];
    rank_totals(sp, b, world, 0, t);
    scg_after_value(s, t, b.trace, phase);
}

__global__ void k_scalar_after_curv(const __grid_constant__ StencilParams sp, Buffers b, int world) {
    ScgState* s = b.st;
    if (s->done) return;
    if (!s->success) { scg_pre_value(s); return; }
    double t[NSLOT];
    rank_totals(sp, b, world, 1, t);
    scg_after_curv(s, t);
}

__global__ void k_state_init(ScgState* s, double lam0, double lambda_reg, int n_iter, long long npix, int rules,
                             unsigned* gbar, double* part) {
    if (gbar) *gbar = 0u;
    // the loop kernels' grid_sum accumulator sets 0 and 1 (25 words each; set 2 is zeroed in the loop)
    if (part)
        for (int i = 0; i < 2 * (6 * NSLOT + 1); ++i) reinterpret_cast<unsigned long long*>(part)[i] = 0ull;
    s->f = 0; s->f_new = 0; s->lam = lam0; s->lamb = 0; s->delta = 0; s->pp = 0; s->mu = 0;
    s->alpha = 0; s->beta = 0; s->rr = 0; s->lambda_reg = lambda_reg;
    for (int i = 0; i < 8; ++i) s->dbg[i] = 0;
    s->alpha_f = 0; s->alpha_upd_f = 0; s->beta_f = 0;
    s->npix = npix; s->k = 0; s->n_iter = n_iter; s->success = 1; s->done = 0;
    s->xcur = 0; s->rcur = 0; s->accepted = 0; s->converged_at = -1; s->failed_stage = 0; s->failed_iter = -1;
    s->counter = 0;
    s->rules = rules; s->curv = 0;
    s->pend = 0; s->pend_n = 0; s->seq = 0;
}

// ------------------------------------------------------------------------------------------------
// Ingest (polyphase relayout), bilinear initial estimate, finalize, debug forward/adjoint.
// ------------------------------------------------------------------------------------------------
__global__ void k_ingest(IngestParams ip, const float* __restrict__ lr, float* __restrict__ Y) {
    int gx = blockIdx.x * blockDim.x + threadIdx.x;
    int gy = ip.store_lo + blockIdx.y;
    if (gx >= ip.W || gy >= ip.store_hi) return;
    int ph = (gy % ip.mag) * ip.mag + (gx % ip.mag);
    int f = ip.frame_of_phase[ph];
    if (f < 0) {   // missing phase (per-phase path): zero sample under a zero kappa
        Y[(size_t)(gy - ip.store_lo) * ip.pitch + phys_col(gx, ip.perm)] = 0.0f;
        return;
    }
    int a = (gy - ip.sy[f]) / ip.mag, c = (gx - ip.sx[f]) / ip.mag;
    Y[(size_t)(gy - ip.store_lo) * ip.pitch + phys_col(gx, ip.perm)] =
        __ldg(lr + ((size_t)f * ip.lr_h + a) * ip.lr_w + c);
}

__global__ void k_egest(IngestParams ip, const float* __restrict__ Yhr, float* __restrict__ lr) {
    int gx = blockIdx.x * blockDim.x + threadIdx.x;
    int gy = ip.store_lo + blockIdx.y;
    if (gx >= ip.W || gy >= ip.store_hi) return;
    int ph = (gy % ip.mag) * ip.mag + (gx % ip.mag);
    int f = ip.frame_of_phase[ph];
    if (f < 0) return;
    int a = (gy - ip.sy[f]) / ip.mag, c = (gx - ip.sx[f]) / ip.mag;
    lr[((size_t)f * ip.lr_h + a) * ip.lr_w + c] = Yhr[(size_t)(gy - ip.store_lo) * ip.pitch + phys_col(gx, ip.perm)];
}

__global__ void k_hr_copy(const float* __restrict__ src, int sp_, int sperm, float* __restrict__ dst, int dp, int dperm,
                          int W) {
    int gx = blockIdx.x * blockDim.x + threadIdx.x;
    int gy = blockIdx.y;
    if (gx >= W) return;
    dst[(size_t)gy * dp + phys_col(gx, dperm)] = src[(size_t)gy * sp_ + phys_col(gx, sperm)];
}

// x0(u,v) = bilerp(y_0, (u - t0y)/mag, (v - t0x)/mag), LR indices clamped (reading 14).
__global__ void k_init_x0(IngestParams ip, const float* __restrict__ lr, float* __restrict__ X) {
    int gx = blockIdx.x * blockDim.x + threadIdx.x;
    int gy = ip.store_lo + blockIdx.y;
    if (gx >= ip.W || gy >= ip.store_hi) return;
    float a = ((float)gy - ip.t0y) / (float)ip.mag, c = ((float)gx - ip.t0x) / (float)ip.mag;
    float a0 = floorf(a), c0 = floorf(c);
    float fa = a - a0, fc = c - c0;
    int ia0 = clampi((int)a0, 0, ip.lr_h - 1), ia1 = clampi((int)a0 + 1, 0, ip.lr_h - 1);
    int ic0 = clampi((int)c0, 0, ip.lr_w - 1), ic1 = clampi((int)c0 + 1, 0, ip.lr_w - 1);
    const float* y = lr;
    float v = (1.f - fa) * (1.f - fc) * __ldg(y + (size_t)ia0 * ip.lr_w + ic0) +
              (1.f - fa) * fc * __ldg(y + (size_t)ia0 * ip.lr_w + ic1) +
              fa * (1.f - fc) * __ldg(y + (size_t)ia1 * ip.lr_w + ic0) + fa * fc * __ldg(y + (size_t)ia1 * ip.lr_w + ic1);
    X[(size_t)(gy - ip.store_lo) * ip.pitch + phys_col(gx, ip.perm)] = v;
}

// out = x + alpha_upd p when the last step was accepted and not yet applied (fused with the copy
// into the caller's buffer; Alg. 1 line 24 for the owned rows).
__global__ void k_finalize(StencilParams sp, Buffers b, float* __restrict__ out, int out_pitch, int row_lo, int row_hi) {
    int gx = blockIdx.x * blockDim.x + threadIdx.x;
    int gy = row_lo + blockIdx.y;
    if (gx >= sp.W || gy >= row_hi) return;
    const ScgState* s = b.st;
    float a = s->success ? s->alpha_upd_f : 0.0f;
    size_t off = (size_t)(gy - sp.store_lo) * sp.pitch + phys_col(gx, sp.perm);
    out[(size_t)gy * out_pitch + gx] = fmaf(a, pick(b.P, s->xcur)[off], pick(b.X, s->xcur)[off]);
}

template <int KR>
__global__ void k_forward_debug(StencilParams sp, const float* __restrict__ x, float* __restrict__ z) {
    int gx = blockIdx.x * blockDim.x + threadIdx.x;
    int gy = sp.row_lo + blockIdx.y;
    if (gx >= sp.W || gy >= sp.row_hi) return;
    constexpr int KD = 2 * KR + 1;
    float acc = 0.0f;
    for (int P_ = 0; P_ < KD; ++P_)
        for (int Q_ = 0; Q_ < KD; ++Q_) {
            int uy = clampi(gy + P_ - KR, 0, sp.H - 1), ux = clampi(gx + Q_ - KR, 0, sp.W - 1);
            acc = fmaf(sp.taps[P_ * KD + Q_], x[(size_t)(uy - sp.store_lo) * sp.pitch + ux], acc);
        }
    z[(size_t)(gy - sp.store_lo) * sp.pitch + gx] = acc;
}

template <int KR>
__global__ void k_adjoint_debug(StencilParams sp, const float* __restrict__ w, float* __restrict__ g) {
    int gx = blockIdx.x * blockDim.x + threadIdx.x;
    int gy = sp.row_lo + blockIdx.y;
    if (gx >= sp.W || gy >= sp.row_hi) return;
    constexpr int KD = 2 * KR + 1;
    const int H = sp.H, W = sp.W;
    int ylo = (gy == 0) ? -KR : gy, yhi = (gy == H - 1) ? H - 1 + KR : gy;
    int xlo = (gx == 0) ? -KR : gx, xhi = (gx == W - 1) ? W - 1 + KR : gx;
    float acc = 0.0f;
    for (int yy = ylo; yy <= yhi; ++yy)
        for (int xx = xlo; xx <= xhi; ++xx)
            for (int P_ = 0; P_ < KD; ++P_)
                for (int Q_ = 0; Q_ < KD; ++Q_) {
                    int uy = yy - (P_ - KR), ux = xx - (Q_ - KR);
                    if (uy < 0 || uy >= H || ux < 0 || ux >= W) continue;
                    acc = fmaf(sp.taps[P_ * KD + Q_], w[(size_t)(uy - sp.store_lo) * sp.pitch + ux], acc);
                }
    g[(size_t)(gy - sp.store_lo) * sp.pitch + gx] = acc;
}

// ------------------------------------------------------------------------------------------------
// Launchers
// ------------------------------------------------------------------------------------------------
#define FL_DISPATCH(KERNEL, KR_, BW_, PN_, GRID, ...)                                                  \
    do {                                                                                               \
        switch ((KR_) * 100 + (BW_) * 10 + (PN_)) {                                                    \
            FL_CASE(KERNEL, 0, 1, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 0, 1, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 0, 2, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 0, 2, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 0, 3, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 0, 3, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 1, 1, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 1, 1, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 1, 2, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 1, 2, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 1, 3, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 1, 3, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 2, 1, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 2, 1, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 2, 2, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 2, 2, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 2, 3, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 2, 3, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 3, 1, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 3, 1, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 3, 2, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 3, 2, 2, GRID, __VA_ARGS__)    \
            FL_CASE(KERNEL, 3, 3, 1, GRID, __VA_ARGS__) FL_CASE(KERNEL, 3, 3, 2, GRID, __VA_ARGS__)    \
            default: return cudaErrorInvalidValue;                                                     \
        }                                                                                              \
    } while (0)
#define FL_CASE(KERNEL, A, B, C, GRID, ...) \
    case A * 100 + B * 10 + C: KERNEL<A, B, C><<<GRID, NTHREADS, 0, s>>>(__VA_ARGS__); break;

cudaError_t launch_value_grad(int kr, int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                              cudaStream_t s) {
    dim3 grid(sp.tiles_x, sp.tiles_y);
    FL_DISPATCH(k_value_grad, kr, bw, pn, grid, sp, b, phase);
    return cudaGetLastError();
}

cudaError_t launch_update_curv(int kr, int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                               cudaStream_t s) {
    dim3 grid(sp.tiles_x, sp.tiles_y);
    FL_DISPATCH(k_update_curv, kr, bw, pn, grid, sp, b, phase);
    return cudaGetLastError();
}

cudaError_t launch_scalar_after_value(const StencilParams& sp, const Buffers& b, int world, int phase, cudaStream_t s) {
    k_scalar_after_value<<<1, 1, 0, s>>>(sp, b, world, phase);
    return cudaGetLastError();
}
cudaError_t launch_scalar_after_curv(const StencilParams& sp, const Buffers& b, int world, cudaStream_t s) {
    k_scalar_after_curv<<<1, 1, 0, s>>>(sp, b, world);
    return cudaGetLastError();
}

cudaError_t launch_state_init(const Buffers& b, double lam0, double lambda_reg, int n_iter, long long npix,
                              int rules, cudaStream_t s) {
    k_state_init<<<1, 1, 0, s>>>(b.st, lam0, lambda_reg, n_iter, npix, rules, b.gbar, b.part);
    return cudaGetLastError();
}

static dim3 rowgrid(int W, int rows) { return dim3((W + 255) / 256, rows); }

// Vectorised setup/output kernels for the streaming path's permuted layout (W % 4 == 0): one thread
// per group of four HR columns, 16-byte stores.
// mag = 2: the group (c0, c2 | c1, c3) of HR row u holds LR columns (2q, 2q+1) of the frames with
// phases (u & 1, 0) and (u & 1, 1) -- two 8-byte loads, one 16-byte store.
__global__ void k_ingest_m2(IngestParams ip, const float* __restrict__ lr, float* __restrict__ Y) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = ip.store_lo + blockIdx.y;
    if (4 * q >= ip.W || gy >= ip.store_hi) return;
    const int py = gy & 1;
    // a phase no frame covers (per-phase path with missing phases: its kappa is zero) holds 0
    const int f0 = ip.frame_of_phase[py * 2], f1 = ip.frame_of_phase[py * 2 + 1];
    const int a0 = (gy - py) >> 1, a1 = (gy - py) >> 1;
    const float2 v0 = f0 < 0 ? make_float2(0.f, 0.f)
                             : __ldg(reinterpret_cast<const float2*>(lr + ((size_t)f0 * ip.lr_h + a0) * ip.lr_w + 2 * q));
    const float2 v1 = f1 < 0 ? make_float2(0.f, 0.f)
                             : __ldg(reinterpret_cast<const float2*>(lr + ((size_t)f1 * ip.lr_h + a1) * ip.lr_w + 2 * q));
    *reinterpret_cast<float4*>(Y + (size_t)(gy - ip.store_lo) * ip.pitch + 4 * q) = make_float4(v0.x, v0.y, v1.x, v1.y);
}

// x3 polyphase ingest (complete phases, lr_w % 4 == 0): a thread turns four LR columns of the three
// frames of its row phase into twelve HR columns -- three 16-byte loads, three 16-byte stores
__global__ void k_ingest_m3(IngestParams ip, const float* __restrict__ lr, float* __restrict__ Y) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = ip.store_lo + blockIdx.y;
    if (12 * k >= ip.W || gy >= ip.store_hi) return;
    const int py = gy % 3, a = (gy - py) / 3;
    float4 L[3];
#pragma unroll
    for (int px = 0; px < 3; ++px) {
        const int f = ip.frame_of_phase[py * 3 + px];
        L[px] = __ldg(reinterpret_cast<const float4*>(lr + ((size_t)f * ip.lr_h + a) * ip.lr_w + 4 * k));
    }
    auto at = [&](int c) -> float {   // HR column 12k + c = 3 (4k + c / 3) + c % 3
        const float4& v = L[c % 3];
        const int m = c / 3;
        return m == 0 ? v.x : m == 1 ? v.y : m == 2 ? v.z : v.w;
    };
    float* row = Y + (size_t)(gy - ip.store_lo) * ip.pitch + 12 * k;
#pragma unroll
    for (int i = 0; i < 3; ++i)
        *reinterpret_cast<float4*>(row + 4 * i) = make_float4(at(4 * i), at(4 * i + 2), at(4 * i + 1), at(4 * i + 3));
}

// polyphase ingest for any magnification in the permuted layout: one 16-byte store per group of four
// HR columns, each column's LR sample from its phase's frame (a missing phase holds 0)
template <int MAG>
__global__ void k_ingest_v4(IngestParams ip, const float* __restrict__ lr, float* __restrict__ Y) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = ip.store_lo + blockIdx.y;
    if (4 * q >= ip.W || gy >= ip.store_hi) return;
    const int py = gy % MAG;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int gx = 4 * q + j, px = gx % MAG;
        const int f = ip.frame_of_phase[py * MAG + px];
        v[j] = f < 0 ? 0.0f
                     : __ldg(lr + ((size_t)f * ip.lr_h + (gy - ip.sy[f]) / MAG) * ip.lr_w + (gx - ip.sx[f]) / MAG);
    }
    *reinterpret_cast<float4*>(Y + (size_t)(gy - ip.store_lo) * ip.pitch + 4 * q) = make_float4(v[0], v[2], v[1], v[3]);
}

// x0 (reading 14) when frame 0's HR shift is integral: integer floor division by the magnification and
// exact fractions j / MAG (no float division of the coordinates), four columns per thread, permuted
// layout, p0 = 0 in the same pass
template <int MAG>
__global__ void k_init_x0_int(IngestParams ip, int t0y, int t0x, const float* __restrict__ lr, float* __restrict__ X,
                              float* __restrict__ P0) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = ip.store_lo + blockIdx.y;
    if (4 * q >= ip.W || gy >= ip.store_hi) return;
    const int an = gy - t0y;
    const int a0 = an >= 0 ? an / MAG : -((-an + MAG - 1) / MAG);
    const float fa = (float)(an - a0 * MAG) * (1.0f / MAG);
    const float* r0 = lr + (size_t)clampi(a0, 0, ip.lr_h - 1) * ip.lr_w;
    const float* r1 = lr + (size_t)clampi(a0 + 1, 0, ip.lr_h - 1) * ip.lr_w;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int cn = 4 * q + j - t0x;
        const int c0 = cn >= 0 ? cn / MAG : -((-cn + MAG - 1) / MAG);
        const float fc = (float)(cn - c0 * MAG) * (1.0f / MAG);
        const int ic0 = clampi(c0, 0, ip.lr_w - 1), ic1 = clampi(c0 + 1, 0, ip.lr_w - 1);
        v[j] = (1.f - fa) * (1.f - fc) * __ldg(r0 + ic0) + (1.f - fa) * fc * __ldg(r0 + ic1) +
               fa * (1.f - fc) * __ldg(r1 + ic0) + fa * fc * __ldg(r1 + ic1);
    }
    const size_t o = (size_t)(gy - ip.store_lo) * ip.pitch + 4 * q;
    *reinterpret_cast<float4*>(X + o) = make_float4(v[0], v[2], v[1], v[3]);
    if (P0) *reinterpret_cast<float4*>(P0 + o) = make_float4(0.f, 0.f, 0.f, 0.f);
}

// x0 at x2 / x3 when frame 0's HR column shift is a multiple of the magnification: a thread's HR columns
// (4 at x2, 12 at x3) read a fixed window of 3 / 5 consecutive LR columns per LR row, so every tap is a
// compile-time register (vector loads, no per-column address arithmetic)
template <int MAG>
__global__ void k_init_x0_vec(IngestParams ip, int t0y, int t0x, const float* __restrict__ lr, float* __restrict__ X) {
    constexpr int NC = MAG == 2 ? 4 : 12;          // HR columns per thread
    constexpr int NL = NC / MAG + 1;               // LR columns read per row
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = ip.store_lo + blockIdx.y;
    if (NC * k >= ip.W || gy >= ip.store_hi) return;
    const int an = gy - t0y;
    const int a0 = an >= 0 ? an / MAG : -((-an + MAG - 1) / MAG);
    const float fa = (float)(an - a0 * MAG) * (1.0f / MAG);
    const float* r0 = lr + (size_t)clampi(a0, 0, ip.lr_h - 1) * ip.lr_w;
    const float* r1 = lr + (size_t)clampi(a0 + 1, 0, ip.lr_h - 1) * ip.lr_w;
    const int b0 = (NC * k - t0x) / MAG;           // exact: t0x % MAG == 0
    float c[NL];
#pragma unroll
    for (int m = 0; m < NL; ++m) {
        const int ic = clampi(b0 + m, 0, ip.lr_w - 1);
        c[m] = (1.f - fa) * __ldg(r0 + ic) + fa * __ldg(r1 + ic);   // the row interpolation at LR column b0 + m
    }
    float v[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        const int m = j / MAG;
        const float fc = (float)(j % MAG) * (1.0f / MAG);
        v[j] = (1.f - fc) * c[m] + fc * c[m + 1];
    }
    float* row = X + (size_t)(gy - ip.store_lo) * ip.pitch + NC * k;
#pragma unroll
    for (int i = 0; i < NC / 4; ++i)
        *reinterpret_cast<float4*>(row + 4 * i) = make_float4(v[4 * i], v[4 * i + 2], v[4 * i + 1], v[4 * i + 3]);
}

__device__ __forceinline__ float bilerp_x0(const IngestParams& ip, const float* __restrict__ y, int gy, int gx) {
    float a = ((float)gy - ip.t0y) / (float)ip.mag, c = ((float)gx - ip.t0x) / (float)ip.mag;
    float a0 = floorf(a), c0 = floorf(c);
    float fa = a - a0, fc = c - c0;
    int ia0 = clampi((int)a0, 0, ip.lr_h - 1), ia1 = clampi((int)a0 + 1, 0, ip.lr_h - 1);
    int ic0 = clampi((int)c0, 0, ip.lr_w - 1), ic1 = clampi((int)c0 + 1, 0, ip.lr_w - 1);
    return (1.f - fa) * (1.f - fc) * __ldg(y + (size_t)ia0 * ip.lr_w + ic0) +
           (1.f - fa) * fc * __ldg(y + (size_t)ia0 * ip.lr_w + ic1) +
           fa * (1.f - fc) * __ldg(y + (size_t)ia1 * ip.lr_w + ic0) + fa * fc * __ldg(y + (size_t)ia1 * ip.lr_w + ic1);
}

// x0 (reading 14) for one group of four columns of one row, in the permuted layout, plus p0 = 0 in the
// same pass (P0 nullable).  The row interpolation (a0, a1, fa) is shared by the four columns.
__global__ void k_init_x0_perm(IngestParams ip, const float* __restrict__ lr, float* __restrict__ X,
                               float* __restrict__ P0) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = ip.store_lo + blockIdx.y;
    if (4 * q >= ip.W || gy >= ip.store_hi) return;
    const float a = ((float)gy - ip.t0y) / (float)ip.mag;
    const float a0 = floorf(a), fa = a - a0;
    const float* r0 = lr + (size_t)clampi((int)a0, 0, ip.lr_h - 1) * ip.lr_w;
    const float* r1 = lr + (size_t)clampi((int)a0 + 1, 0, ip.lr_h - 1) * ip.lr_w;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float c = ((float)(4 * q + j) - ip.t0x) / (float)ip.mag;
        const float c0 = floorf(c), fc = c - c0;
        const int ic0 = clampi((int)c0, 0, ip.lr_w - 1), ic1 = clampi((int)c0 + 1, 0, ip.lr_w - 1);
        v[j] = (1.f - fa) * (1.f - fc) * __ldg(r0 + ic0) + (1.f - fa) * fc * __ldg(r0 + ic1) +
               fa * (1.f - fc) * __ldg(r1 + ic0) + fa * fc * __ldg(r1 + ic1);
    }
    const size_t o = (size_t)(gy - ip.store_lo) * ip.pitch + 4 * q;
    *reinterpret_cast<float4*>(X + o) = make_float4(v[0], v[2], v[1], v[3]);
    if (P0) *reinterpret_cast<float4*>(P0 + o) = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void k_finalize_perm(StencilParams sp, Buffers b, float* __restrict__ out, int out_pitch, int row_lo,
                                int row_hi) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = row_lo + blockIdx.y;
    if (4 * q >= sp.W || gy >= row_hi) return;
    const ScgState* s = b.st;
    const float a = s->success ? s->alpha_upd_f : 0.0f;
    const size_t off = (size_t)(gy - sp.store_lo) * sp.pitch + 4 * q;
    const float4 x = *reinterpret_cast<const float4*>(pick(b.X, s->xcur) + off);
    const float4 p = *reinterpret_cast<const float4*>(pick(b.P, s->xcur) + off);
    // stored (c0, c2, c1, c3) -> natural (c0, c1, c2, c3)
    *reinterpret_cast<float4*>(out + (size_t)gy * out_pitch + 4 * q) =
        make_float4(fmaf(a, p.x, x.x), fmaf(a, p.z, x.z), fmaf(a, p.y, x.y), fmaf(a, p.w, x.w));
}

static bool vec4_ok(int perm, int W, int pitch) { return perm && W % 4 == 0 && pitch % 4 == 0; }

cudaError_t launch_ingest(const IngestParams& ip, const float* lr, float* Y, cudaStream_t s) {
    const dim3 g4 = rowgrid(ip.W / 4, ip.store_hi - ip.store_lo);
    if (vec4_ok(ip.perm, ip.W, ip.pitch) && ip.mag == 2 && ip.lr_w % 2 == 0)
        k_ingest_m2<<<g4, 256, 0, s>>>(ip, lr, Y);
    else if (vec4_ok(ip.perm, ip.W, ip.pitch) && ip.mag == 3 && ip.lr_w % 4 == 0 && ip.complete)
        k_ingest_m3<<<rowgrid(ip.W / 12, ip.store_hi - ip.store_lo), 256, 0, s>>>(ip, lr, Y);
    else if (vec4_ok(ip.perm, ip.W, ip.pitch) && ip.mag == 3)
        k_ingest_v4<3><<<g4, 256, 0, s>>>(ip, lr, Y);
    else if (vec4_ok(ip.perm, ip.W, ip.pitch) && ip.mag == 4)
        k_ingest_v4<4><<<g4, 256, 0, s>>>(ip, lr, Y);
    else
        k_ingest<<<rowgrid(ip.W, ip.store_hi - ip.store_lo), 256, 0, s>>>(ip, lr, Y);
    return cudaGetLastError();
}
cudaError_t launch_egest(const IngestParams& ip, const float* Yhr, float* lr, cudaStream_t s) {
    k_egest<<<rowgrid(ip.W, ip.store_hi - ip.store_lo), 256, 0, s>>>(ip, Yhr, lr);
    return cudaGetLastError();
}
cudaError_t launch_hr_copy(const float* src, int src_pitch, int src_perm, float* dst, int dst_pitch, int dst_perm,
                           int rows, int W, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    k_hr_copy<<<rowgrid(W, rows), 256, 0, s>>>(src, src_pitch, src_perm, dst, dst_pitch, dst_perm, W);
    return cudaGetLastError();
}
static bool x0_int_path(const IngestParams& ip) {
    return vec4_ok(ip.perm, ip.W, ip.pitch) && ip.t0y == floorf(ip.t0y) && ip.t0x == floorf(ip.t0x) && ip.mag >= 1 &&
           ip.mag <= 4;
}
// the integer-phase x0 kernel writes X only (p0 = 0 by a memset: measured faster than a second
// 16-byte store stream from the same kernel, 41 -> ~25 us at C3)
bool init_x0_zeroes_p(const IngestParams& ip) { return vec4_ok(ip.perm, ip.W, ip.pitch) && !x0_int_path(ip); }
cudaError_t launch_init_x0(const IngestParams& ip, const float* lr, float* X, cudaStream_t s, float* P0) {
    const dim3 g4 = rowgrid(ip.W / 4, ip.store_hi - ip.store_lo);
    if (x0_int_path(ip)) {
        const int ty = (int)ip.t0y, tx = (int)ip.t0x;
        if (ip.mag == 2 && tx % 2 == 0) {
            k_init_x0_vec<2><<<g4, 256, 0, s>>>(ip, ty, tx, lr, X);
            return cudaGetLastError();
        }
        if (ip.mag == 3 && tx % 3 == 0 && ip.W % 12 == 0) {
            k_init_x0_vec<3><<<rowgrid(ip.W / 12, ip.store_hi - ip.store_lo), 256, 0, s>>>(ip, ty, tx, lr, X);
            return cudaGetLastError();
        }
        switch (ip.mag) {
            case 1: k_init_x0_int<1><<<g4, 256, 0, s>>>(ip, ty, tx, lr, X, nullptr); break;
            case 2: k_init_x0_int<2><<<g4, 256, 0, s>>>(ip, ty, tx, lr, X, nullptr); break;
            case 3: k_init_x0_int<3><<<g4, 256, 0, s>>>(ip, ty, tx, lr, X, nullptr); break;
            default: k_init_x0_int<4><<<g4, 256, 0, s>>>(ip, ty, tx, lr, X, nullptr); break;
        }
    } else if (vec4_ok(ip.perm, ip.W, ip.pitch))
        k_init_x0_perm<<<rowgrid(ip.W / 4, ip.store_hi - ip.store_lo), 256, 0, s>>>(ip, lr, X, P0);
    else
        k_init_x0<<<rowgrid(ip.W, ip.store_hi - ip.store_lo), 256, 0, s>>>(ip, lr, X);
    return cudaGetLastError();
}
cudaError_t launch_finalize(const StencilParams& sp, const Buffers& b, float* out, int out_pitch, int row_lo,
                            int row_hi, cudaStream_t s) {
    if (vec4_ok(sp.perm, sp.W, sp.pitch) && out_pitch % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0)
        k_finalize_perm<<<rowgrid(sp.W / 4, row_hi - row_lo), 256, 0, s>>>(sp, b, out, out_pitch, row_lo, row_hi);
    else
        k_finalize<<<rowgrid(sp.W, row_hi - row_lo), 256, 0, s>>>(sp, b, out, out_pitch, row_lo, row_hi);
    return cudaGetLastError();
}
cudaError_t launch_forward_debug(int kr, const StencilParams& sp, const float* x, float* z, cudaStream_t s) {
    dim3 g = rowgrid(sp.W, sp.row_hi - sp.row_lo);
    switch (kr) {
        case 0: k_forward_debug<0><<<g, 256, 0, s>>>(sp, x, z); break;
        case 1: k_forward_debug<1><<<g, 256, 0, s>>>(sp, x, z); break;
        case 2: k_forward_debug<2><<<g, 256, 0, s>>>(sp, x, z); break;
        case 3: k_forward_debug<3><<<g, 256, 0, s>>>(sp, x, z); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
cudaError_t launch_adjoint_debug(int kr, const StencilParams& sp, const float* w, float* g, cudaStream_t s) {
    dim3 gr = rowgrid(sp.W, sp.row_hi - sp.row_lo);
    switch (kr) {
        case 0: k_adjoint_debug<0><<<gr, 256, 0, s>>>(sp, w, g); break;
        case 1: k_adjoint_debug<1><<<gr, 256, 0, s>>>(sp, w, g); break;
        case 2: k_adjoint_debug<2><<<gr, 256, 0, s>>>(sp, w, g); break;
        case 3: k_adjoint_debug<3><<<gr, 256, 0, s>>>(sp, w, g); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// uint16 detector codes -> fp32 (value = scale * code): 8 codes (16 B) per thread, two 16-B stores
__global__ void k_u16_to_f32(const uint16_t* __restrict__ in, float* __restrict__ out, long long n, float scale) {
    const long long i8 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (i8 + 8 <= n) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(in + i8));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        float o[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            o[2 * j] = scale * (float)(w[j] & 0xffffu);
            o[2 * j + 1] = scale * (float)(w[j] >> 16);
        }
        reinterpret_cast<float4*>(out + i8)[0] = make_float4(o[0], o[1], o[2], o[3]);
        reinterpret_cast<float4*>(out + i8)[1] = make_float4(o[4], o[5], o[6], o[7]);
    } else {
        for (long long i = i8; i < n; ++i) out[i] = scale * (float)in[i];
    }
}
cudaError_t launch_u16_to_f32(const uint16_t* in, float* out, long long n, float scale, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const long long nt = (n + 7) / 8;
    k_u16_to_f32<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(in, out, n, scale);
    return cudaGetLastError();
}

}  // namespace flmisr
