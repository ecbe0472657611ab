// flmisr_internal.h -- shared declarations between the host plan/driver (flmisr_api.cpp) and the
// sm_100a kernels (flmisr_kernels.cu).  Not part of the public ABI (include/flmisr.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace flmisr {

// Output tile of one CTA in the stencil kernels (rows x columns of HR pixels).
constexpr int TX = 64;
constexpr int TY = 16;
constexpr int NTHREADS = 256;
constexpr int MAXKR = 3;                                 // kappa radius (PSF radius, +1 for a common fractional phase)
constexpr int MAXTAPS = (2 * MAXKR + 1) * (2 * MAXKR + 1);
constexpr int MAXBW = 3;                                 // BTV window w
constexpr int NSLOT = 4;                                 // fp64 partial sums per CTA

// Device-resident SCG state (Moller SCG scalars).  fp64 scalars; the fp32
// copies are what the per-pixel kernels use.
struct ScgState {
    double f, f_new, lam, lamb, delta, pp, mu, alpha, beta, rr;
    double lambda_reg;           // BTV weight lambda (Eq. objective)
    double dbg[8];               // debug-entry sums
    float alpha_f;               // step alpha for the value/gradient pass (x + alpha p)
    float alpha_upd_f;           // alpha of the pending accepted step, applied by the next update pass
    float beta_f;                // conjugate-direction beta for the next update pass
    float pad0;
    long long npix;              // H*W (Moller restart period)
    int k, n_iter, success, done;
    int xcur, rcur;              // ping-pong indices of x/p and r buffers
    int accepted, converged_at, failed_stage, failed_iter;
    unsigned int counter;        // CTA arrival counter (last-CTA reduction), reset by the last CTA
    int rules;                   // SCG variant bits (flmisr_config.scg_rules): 1 PR+ restart, 2 Netlab scale rules
    double curv;                 // last exact curvature p^T Hess J p (Netlab rules recompute delta from it)
    // deferred reduction (streaming kernels, world == 1): the kernel that produced per-CTA slots leaves
    // them pending; the next kernel reduces them in every CTA and applies the scalar step on entry
    int pend;                    // 0 none, PEND_VG_INIT, PEND_VG_ITER, PEND_UC
    int pend_n;                  // CTAs (slots) of the producing kernel
    int seq;                     // producing-kernel counter: slots live in part[(seq & 1) * NSLOT * pend_n ...]
    int pad2;
};
enum Pending : int { PEND_NONE = 0, PEND_VG_INIT = 1, PEND_VG_ITER = 2, PEND_UC = 3 };

struct StencilParams {
    int H, W, pitch;             // global HR size, row pitch (floats) of every HR buffer
    int row_lo, row_hi;          // owned global rows [row_lo, row_hi)
    int store_lo, store_hi;      // rows held in device storage [store_lo, store_hi) (owned + halo)
    int tile_row0;               // global row of the first tile row
    int tiles_x, tiles_y;
    int world;                   // 1: scalar logic in the last CTA; >1: rank sums for the allgather
    int perm;                    // HR buffers use the permuted column layout (streaming path)
    float eps, eps2, lam;        // Charbonnier eps, eps^2, BTV weight lambda (fp32 copies)
    float taps[MAXTAPS];         // kappa, (2KR+1)^2 centred, row-major, correlation orientation
    float gam[MAXBW * MAXBW];    // gamma(dy,dx) = alpha^(dx+dy) at [dy*MAXBW + dx], gam[0] unused
    // streaming (separable-kappa) kernels, flmisr_stream.cu
    float ka[3], kb[3];          // kappa(P,Q) = ka[P+1] * kb[Q+1] (KR <= 1; KR = 0 zero-padded)
    float lgam[MAXBW * MAXBW];   // lambda * gamma(dy,dx)
    float lgc[4];                // lambda * alpha^c of BTV class c = dx + dy (1..4): 4 distinct weights
    int nstrips, nsegs, seg_rows, wpb;   // 128-column warp strips (step 124), row segments, warps/CTA
    // work items (one warp each): n_int = ni * nseg_i segments of seg_rows rows on the ni interior
    // strips, then ne * nseg_b segments of seg_b rows on the ne edge strips (column 0 / column W-1),
    // which run the slower border code and therefore get shorter segments (one balanced wave)
    int ni, ne, nseg_i, nseg_b, seg_b, n_int, nitems;
    double gcls[4];              // gamma of BTV class dx+dy = 1..4 (fp64, applied to the CTA sums)
    // affine correction of the raw CTA sums before the scalar logic: tot = raw * aff[k] + aff[4+k]
    double aff_vg[2 * NSLOT], aff_uc[2 * NSLOT];
    int deferred;                // streaming kernels: deferred reduction (world == 1), see ScgState::pend
    // det mode (flmisr_config.det_rows > 0): work items are fixed global tiles, sums exact 128-bit fixed
    // point; the affine offsets are the whole image's (applied once to the exact all-band total)
    int det;                     // 1: det mode; det_rows = T, the tile height (segments are unions of tiles)
    int det_rows;
    int loop_warps;              // warps of the persistent loop kernels: nitems, or (det) at most one wave
    double det_off_vg[NSLOT], det_off_uc[NSLOT];
};
// det mode: 128-bit words per CTA partial (NSLOT exact sums + the count of non-finite tile values)
constexpr int FXW = NSLOT + 1;
constexpr int RSW = 2 * FXW;   // doubles per rank-sum record (det mode: FXW 128-bit words; else NSLOT fp64)

// Streaming kernels (flmisr_stream.cu): strips of SCOLS columns per warp, stepping by SSTEP.
#ifndef FLMISR_SWPB
#define FLMISR_SWPB 16
#endif
#ifndef FLMISR_SMINB
#define FLMISR_SMINB 1
#endif
constexpr int SWPB = FLMISR_SWPB;    // warps per CTA of the streaming kernels
constexpr int SMINB = FLMISR_SMINB;  // resident CTAs per SM they are compiled for (register budget)
constexpr int SCOLS = 128;
constexpr int SHALO = 2;
constexpr int SSTEP = SCOLS - 2 * SHALO;

// Per-phase streaming path (flmisr_stream4.cu): K = 4 frames at x2 with complete integer phases and a
// composed kernel per frame; strips overlap by 4 columns per side.
constexpr int PC_SSTEP = SCOLS - 8;
#ifndef FLMISR_PC_WPB
#define FLMISR_PC_WPB 12
#endif
constexpr int PC_WPB = FLMISR_PC_WPB;    // warps per CTA of the per-phase kernels (one CTA per SM)
struct PcTaps {
    float k[4][16];              // kappa of phase class 2 (u mod 2) + (v mod 2) at [(P+1)*4 + (Q+1)], P, Q in [-1, 2]
};

struct Buffers {
    const float* Y;              // polyphase-interleaved LR stack on the HR grid (storage base)
    float* X[2];                 // x ping-pong
    float* P[2];                 // p ping-pong
    float* R[2];                 // r = -grad J ping-pong (R[rcur] accepted, R[1-rcur] candidate)
    double* part;                // NSLOT x ntiles fp64 CTA partials (slot-major)
    double* rank_sums;           // NSLOT fp64 rank-local sums (world > 1)
    ScgState* st;
    double* trace;               // (n_iter+1) x 6 rows (k, f, rr, alpha, lambda_scg, accepted)
    const float* halo_top;       // world > 1: received r rows above the band (eta x pitch) or null
    const float* halo_bot;       // received r rows below the band or null
    float* send_top;             // owned top eta rows of the r candidate, for the upper neighbour
    float* send_bot;
    int eta;                     // halo rows per side
    unsigned* gbar;              // grid-barrier arrival counter of the persistent loop kernel (zeroed per call)
    const float* mem_lo;         // the plan's HR allocation [mem_lo, mem_hi) (all seven buffers + padding
    const float* mem_hi;         // rows): bounds of every streaming-kernel access in FLMISR_BOUNDS builds
};

// Row bands over peer memory (flmisr_stream.cu k_scg_peer_loop*).  Pointers
// indexed by absolute rank q are the rank's memory as mapped on this device (CUDA IPC over NVLink;
// plain device pointers when all bands share one device); those indexed by the launch-local band l
// are this device's own.
constexpr int PMAX = 8;                  // ranks of a peer group
struct PeerLoop {
    int g;                       // bands in this launch: 1 (one per GPU) or world (all on one device)
    int rank0;                   // rank of band l = 0 of this launch
    int world;
    int ctas;                    // CTAs per band (identical on every rank)
    double* mbox[PMAX];          // rank q's mailbox [2][world][ctas][NSLOT]: every CTA's partial sums
    unsigned long long* cnt[PMAX];   // rank q's arrival counter (monotonic across calls)
    unsigned* epoch_word[PMAX];  // band l: phases completed over all calls
    unsigned long long timeout_ns;   // a barrier wait longer than this abandons the loop (failed_stage 3)
    int drop_band;               // test hook (FLMISR_PEER_TEST_DROP, emulation): this band never arrives; -1 none
};
enum FailStage : int { FAIL_NONE = 0, FAIL_CURV = 1, FAIL_VALUE = 2, FAIL_PEER_TIMEOUT = 3 };
struct PeerBands {               // g > 1 (one device): every band's parameters, kernel-parameter space
    StencilParams sp[PMAX];
    Buffers b[PMAX];
};

enum Phase : int { PH_ITER = 0, PH_INIT = 1, PH_DEBUG = 2 };

// Launchers (flmisr_kernels.cu).  Return cudaSuccess or the launch error; dispatch on (kr, bw, pn).
cudaError_t launch_value_grad(int kr, int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                              cudaStream_t s);
cudaError_t launch_update_curv(int kr, int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                               cudaStream_t s);
cudaError_t launch_value_grad_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                                     cudaStream_t s);
cudaError_t launch_update_curv_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, int phase,
                                      cudaStream_t s);
// deferred mode: apply the last kernel's pending scalar step (one CTA) before the state is read back
cudaError_t launch_settle(const StencilParams& sp, const Buffers& b, cudaStream_t s);
// the whole SCG loop (init pass + n_iter passes) as one cooperative persistent kernel (world == 1)
cudaError_t launch_scg_loop_stream(int bw, int pn, const StencilParams& sp, const Buffers& b, cudaStream_t s);
cudaError_t launch_scg_peer_loop(int bw, int pn, const StencilParams& sp, const Buffers& b, const PeerLoop& pl,
                                 const PeerBands* pb, cudaStream_t s);
cudaError_t launch_pc_vg(int bw, int pn, const StencilParams& sp, const Buffers& b, const PcTaps& T, int phase,
                         cudaStream_t s);
cudaError_t launch_pc_uc(int bw, int pn, const StencilParams& sp, const Buffers& b, const PcTaps& T, int phase,
                         cudaStream_t s);
cudaError_t launch_pc_loop(int bw, int pn, const StencilParams& sp, const Buffers& b, const PcTaps& T, cudaStream_t s);
cudaError_t launch_pc_forward_debug(const StencilParams& sp, const PcTaps& T, const float* x, float* z, cudaStream_t s);
cudaError_t launch_pc_adjoint_debug(const StencilParams& sp, const PcTaps& T, const float* w, float* g, cudaStream_t s);
cudaError_t launch_scalar_after_value(const StencilParams& sp, const Buffers& b, int world, int phase,
                                      cudaStream_t s);   // world > 1
cudaError_t launch_scalar_after_curv(const StencilParams& sp, const Buffers& b, int world, cudaStream_t s);   // world > 1
cudaError_t launch_state_init(const Buffers& b, double lam0, double lambda_reg, int n_iter, long long npix,
                              int rules, cudaStream_t s);

struct IngestParams {
    int H, W, pitch, k, lr_h, lr_w, mag;
    int store_lo, store_hi;
    int frame_of_phase[16];      // residue (u mod mag, v mod mag) -> frame index
    int sy[16], sx[16];          // integer phase of frame i
    float t0y, t0x;              // HR shift of frame 0 (bilinear initial estimate)
    int perm;                    // 1: HR buffers use the streaming path's permuted column layout
    int complete;                // 1: every phase class holds a frame (no missing phase)
};

// General-geometry path (flmisr_general.cu): per-frame integer phase and composed kernel.
constexpr int GMAXK = 64;                                // frames supported by the general path
constexpr int GMAXOFF = 16;                              // BTV offsets (w <= 3: quadrant 8, Farsiu 11)
struct GenParams {
    int k, lr_h, lr_w, mag;
    int R, kd;                   // kappa offsets [-R, R+1] per axis, kd = 2R + 2
    int fy_lo, fy_hi, fx_lo, fx_hi;   // virtual HR rows/cols any forward sample reads (clamp folding)
    int nblk_lr, nblk_hr;        // CTAs of the LR-pixel and HR-pixel passes
    const float* taps;           // k x kd x kd, kappa_i(P, Q) at [i][P + R][Q + R] (correlation orientation)
    const float* lr;             // plan-owned copy of the LR stack (k x lr_h x lr_w)
    float* w;                    // rho'(e) per LR pixel (k x lr_h x lr_w)
    double* part_a;              // NSLOT x max(nblk) partials of the first pass of each pair
    int sy[GMAXK], sx[GMAXK];    // integer HR phase floor(mag * shift_i)
    int integer_phase[GMAXK];    // 1: mag * shift_i is integral (interpolation fusion inserts the frame)
    int fd;                      // 1: paper-literal FD curvature (NEXT-4) instead of the exact data curvature
    double sigma0;               // FD probe: sigma = sigma0 / |p|
    double* wd;                  // FD: rho'(e(x + sigma p)) - rho'(e(x)) per LR pixel (fp64)
    int noff;                    // BTV offsets d = (offy, offx), offy >= 0 (quadrant or Farsiu set)
    int offy[GMAXOFF], offx[GMAXOFF];
    float ogam[GMAXOFF];         // gamma(d)
    int fused;                   // 1: the fused tiled kernels k_gen3_* run the loop (phases in [-(R+1), mag-1+R])
    int btvq;                    // BTV offsets are the quadrant of window btvq (compile-time offsets), 0: the list
    int nblk3;                   // their CTAs
};
cudaError_t launch_gen_value_grad(int bw, int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b,
                                  int phase, cudaStream_t s);
cudaError_t launch_gen_update_curv(int bw, int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b,
                                   int phase, cudaStream_t s);
cudaError_t launch_gen_forward(const StencilParams& sp, const GenParams& gp, const float* x, float* y, cudaStream_t s);
cudaError_t launch_gen_adjoint(const StencilParams& sp, const GenParams& gp, const float* w, float* g, cudaStream_t s);
cudaError_t launch_gen_interp(const StencilParams& sp, const GenParams& gp, float* out, int out_pitch, cudaStream_t s);
unsigned gen_blocks(long long n);
unsigned gen_blocks_lr(int k, int lr_h, int lr_w, int cap);   // CTAs of the tiled LR-pixel passes
unsigned gen_blocks_hr(int W, int rows, int cap);             // CTAs of the tiled HR-pixel passes
unsigned gen3_blocks(int W, int H, int cap);                  // CTAs of the fused general kernels
size_t gen3_smem(int R, int mag, int k);                      // their dynamic shared memory (max of the two)
cudaError_t launch_gen3_vg(int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b, int phase,
                           cudaStream_t s);
cudaError_t launch_gen3_uc(int pn, const StencilParams& sp, const GenParams& gp, const Buffers& b, int phase,
                           cudaStream_t s);

// Streaming-path column layout: each aligned group of 4 columns is stored as (c0, c2, c1, c3).
__host__ __device__ __forceinline__ int phys_col(int c, int perm) {
    return perm ? ((c & ~3) | ((c & 1) << 1) | ((c >> 1) & 1)) : c;
}
// pitched HR copy between the natural layout (dst_perm = 0) and a buffer layout (perm)
cudaError_t launch_hr_copy(const float* src, int src_pitch, int src_perm, float* dst, int dst_pitch, int dst_perm,
                           int rows, int W, cudaStream_t s);
cudaError_t launch_ingest(const IngestParams& ip, const float* lr, float* Y, cudaStream_t s);
cudaError_t launch_egest(const IngestParams& ip, const float* Yhr, float* lr, cudaStream_t s);   // debug
// x0 into X (buffer layout); P0 non-null: also zero it in the same pass (returns whether it did)
cudaError_t launch_init_x0(const IngestParams& ip, const float* lr, float* X, cudaStream_t s, float* P0 = nullptr);
bool init_x0_zeroes_p(const IngestParams& ip);
// uint16 detector frames -> fp32 (pipeline input; in and out 16-B aligned)
cudaError_t launch_u16_to_f32(const uint16_t* in, float* out, long long n, float scale, cudaStream_t s);
cudaError_t launch_finalize(const StencilParams& sp, const Buffers& b, float* out, int out_pitch, int row_lo,
                            int row_hi, cudaStream_t s);
cudaError_t launch_forward_debug(int kr, const StencilParams& sp, const float* x, float* zhr, cudaStream_t s);
cudaError_t launch_adjoint_debug(int kr, const StencilParams& sp, const float* whr, float* g, cudaStream_t s);

}  // namespace flmisr
