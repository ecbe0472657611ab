/*
 * flmisr.h -- C ABI of the B200-native FL-MISR SCG reconstruction (arXiv 2108.04315).
 *
 * One call reconstructs one high-resolution (HR) projection x from K low-resolution (LR)
 * projections y_i taken at sub-pixel detector shifts, by minimising the MAP objective
 *
 *     J(x) = sum_i || A_i x - y_i ||_p^p  +  lambda * sum_d gamma(d) || x - S_d x ||_1
 *
 * (Eq. objective; forward model y = A x + eps with A = D B M, Eq. sisr
 * P:65-71; BTV prior Eq. prior) with Moller's scaled conjugate gradient (SCG, the
 * [SCG] citation of P:186/P:206), run as in Algorithm 1: the HR image is
 * row-partitioned over `world` GPUs (Eq. subfunction), SCG scalars are consensus sums
 * of per-partition inner products (tab:parameters P:140-160), and partition borders
 * are exchanged every iteration (inner-outer border exchange, fig:communication).
 * The readings of everything the paper leaves open are in DESIGN.md section 3 ("reading k").
 *
 * Types are C99 only; pointers are plain host or device pointers as stated per argument.
 * All entry points are thread-compatible (a plan must not be used from two threads at once;
 * different plans may run concurrently on different streams).
 */
#ifndef FLMISR_H
#define FLMISR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct flmisr_plan_s* flmisr_plan_t;

typedef enum {
    FLMISR_OK = 0,
    FLMISR_ERR_CONFIG = -1,  /* invalid configuration (raised by flmisr_plan, before any GPU work)  */
    FLMISR_ERR_SHAPE = -2,   /* argument shape / pointer error (raised before any launch)           */
    FLMISR_ERR_CUDA = -3,    /* CUDA runtime error (message in flmisr_last_error)                   */
    FLMISR_ERR_NCCL = -4,    /* NCCL error (multi-GPU)                                              */
    FLMISR_ERR_NUMERIC = -5  /* non-finite consensus scalar: loop frozen on device   */
} flmisr_status;

typedef struct {
    /* LR stack: k frames of lr_h x lr_w, fp32 row-major, intensities normalised to [0,1]
     * (reading 20).  Requirements: k >= 1, lr_h, lr_w >= 1.                          */
    int32_t k, lr_h, lr_w;
    /* host, k x 2 doubles: detector shift (dy, dx) of frame i in LR pixels; frame i samples the
     * HR image at HR position mag*(a,b) + mag*shift_i (reading 3: +dx = lattice moved right). */
    const double* shifts;
    /* host, psf_h x psf_w doubles, odd sizes <= 5, entries >= 0, sum 1 (+-1e-6); centred,
     * applied as correlation on the HR grid (B of Eq. sisr; reading 2).                      */
    const double* psf;
    int32_t psf_h, psf_w;
    int32_t mag;         /* SR factor r in [1, 4]; HR = (mag*lr_h) x (mag*lr_w) (D of Eq. sisr) */
    int32_t p_norm;      /* 1: Charbonnier-smoothed L1 (the paper's choice); 2: squared L2 */
    double l1_eps;       /* Charbonnier epsilon > 0 for the data term and BTV (reading 8); 1e-3  */
    double lambda;       /* regularisation weight >= 0 (Eq. objective; 0.05 at P:271)           */
    double btv_alpha;    /* 0 < alpha < 1, gamma(d) = alpha^(dx+dy) (Eq. prior; 0.4 at P:271)   */
    int32_t btv_window;  /* w in [1, 3]: offsets dx, dy in [0, w-1] (Eq. prior, reading 6/7)   */
    int32_t n_iter;      /* SCG loop passes incl. rejected ones (20 at P:271)      */
    double scg_sigma0;   /* Moller sigma0 of the FD curvature probe (curv_mode = 1)      */
    double scg_lambda0;  /* Moller initial scale lambda_1 > 0; 1e-6                      */
    int32_t rank, world; /* row band `rank` of `world` partitions; world = 1: no NCCL    */
    const void* nccl_unique_id; /* host, 128-byte ncclUniqueId (same on all ranks) or NULL if world == 1 */
    int32_t device;      /* CUDA device ordinal for this rank                                    */
    /* Variants (0 = the readings of DESIGN.md section 3):                      */
    int32_t btv_offsets; /* 0: the paper's quadrant dx, dy in [0, w-1] (reading 6);
                            1: Farsiu's set dy = m in [0, w-1], dx = l in [-(w-1), w-1], l + m >= 0,
                            gamma = alpha^(|l|+m) (the [BTV] citation); general path, world 1 */
    int32_t curv_mode;   /* 0: exact curvature p^T Hess J p (reading 16); 1: the paper's finite-difference
                            probe sigma = scg_sigma0 / |p|, delta = p^T (grad J(x + sigma p) - grad J(x))
                            / sigma, both gradients in fp64 (general path, world 1)     */
    int32_t scg_rules;   /* bit mask: 1 = PR+ restart (beta <- max(beta, 0)); 2 = Netlab scale
                            rules (delta = curv + lam |p|^2 each pass; lam x4 at Delta < 0.25, x1/2 at
                            Delta > 0.75, bounded to [1e-15, 1e100]); 0 = Moller literal (reading 11) */
    int32_t x0_mode;     /* initial estimate when flmisr_reconstruct* gets x0 == NULL: 0 = bilinear
                            upsample of frame 0 (reading 14); 1 = multi-image interpolation
                            fusion (reading 24: the flmisr_interp_fuse image)                */
    int32_t det_rows;    /* 0 = off.  T in [3, 4095], a multiple of 3: results bit-identical for
                            every band count g (SURVEY 8(e) "bit-stable"; "consensus equals
                            centralised"): rows are cut into fixed global tiles of T HR rows, band
                            boundaries are multiples of lcm(T, mag), every warp segment is a union
                            of whole tiles, each tile's partial sums are committed separately and
                            every sum (tile -> lane -> CTA -> band -> all bands) is an exact 128-bit
                            fixed-point sum (grid 2^-64), independent of order and grouping, over
                            both band transports (peer memory and NCCL).  Needs the streaming path
                            (fast_path 2); else FLMISR_ERR_CONFIG.  ~1.45x the loop time on one GPU
                                                                                      */
} flmisr_config;

typedef struct {
    int32_t iters_run;    /* SCG loop passes executed (<= n_iter)                                 */
    int32_t accepted;     /* passes whose step was accepted (runtime grows with these)     */
    int32_t converged_at; /* pass at which <r,r> == 0 stopped the loop, or -1                     */
    int32_t failed_stage; /* 0 none; 1 curvature/step, 2 value/accept (non-finite consensus)      */
    int32_t failed_iter;  /* pass index of the numeric failure, or -1                             */
    double* f_trace;      /* optional caller-owned host array of (n_iter+1)*6 doubles, or NULL:
                             rows (k, f, <r,r>, alpha, lambda_scg, accepted); row 0 = init */
} flmisr_report;

/*
 * flmisr_plan: validate `cfg`, derive the per-frame taps kappa_i = PSF (*) bilinear(frac(mag*shift_i))
 * and integer phases, choose the polyphase fast path (K = mag^2 distinct phases in [0,mag)^2 with one
 * common kappa) or the general-geometry path (any k <= 64, missing, repeated or
 * fractional phases, per-frame kappa_i; world == 1 only), compute the row band and halo, allocate all
 * device scratch on cfg->device and (world > 1) initialise the NCCL communicator from
 * cfg->nccl_unique_id.
 * Ownership: the plan copies everything it needs from cfg (shifts/psf may be freed afterwards).
 * Errors: FLMISR_ERR_CONFIG for invalid parameters or an unsupported geometry (message names the
 * violated rule, e.g. the minimum band height); FLMISR_ERR_CUDA / _NCCL for runtime failures.
 * On error *out is set to NULL.  A plan is reusable for any number of projections.
 */
flmisr_status flmisr_plan(const flmisr_config* cfg, flmisr_plan_t* out);

/*
 * flmisr_reconstruct: run SCG for cfg.n_iter passes on one projection (Alg. 1).
 *   lr_stack  device pointer, k x lr_h x lr_w fp32, full frames on every rank (read only).
 *   x0        device pointer, H x W fp32 initial estimate, or NULL for the bilinear upsample of
 *             frame 0 (reading 14).  Read only.
 *   hr_out    device pointer, H x W fp32 (world == 1 or rank 0: the fused image, Alg. 1 line 24,
 *             P:227); on other ranks rows of the owned band only are written (may be NULL).
 *   cuda_stream  cudaStream_t to enqueue on, or NULL for the plan's own stream.
 *   report    nullable; filled after the end-of-call stream synchronisation.
 * Blocking: returns after the stream has drained (matches SPEC's function semantics).
 * Returns FLMISR_ERR_NUMERIC when a consensus scalar became non-finite (the device froze the loop;
 * hr_out then holds the last finite iterate), FLMISR_ERR_SHAPE on NULL required pointers.
 */
flmisr_status flmisr_reconstruct(flmisr_plan_t plan, const float* lr_stack, const float* x0, float* hr_out,
                                 void* cuda_stream, flmisr_report* report);

/*
 * flmisr_interp_fuse: the paper's non-iterative baseline, multi-image interpolation fusion ("we
 * inserted the pixel values of the LR images into the corresponding integer location in the HR grid";
 * tab:runtime's "Multi-image interp." row; reading 24): every LR pixel of a frame with an
 * integer HR phase is written at its HR site mag*(a,b) + s_i (the first such frame in index order wins);
 * HR sites no frame covers keep the bilinear upsample of frame 0 (reading 14).  On a polyphase-complete
 * stack every HR site holds exactly one LR pixel.
 *   lr_stack  device pointer, k x lr_h x lr_w fp32 (caller-owned, read only)
 *   hr_out    device pointer, H x W fp32 row-major (caller-owned, written)
 *   cuda_stream  cudaStream_t the kernels are enqueued on (0 = the plan's stream); asynchronous
 *             (no host synchronisation).  Uses the plan's scratch buffers: do not overlap it with a
 *             reconstruction on the same plan.
 * Errors: FLMISR_ERR_SHAPE on NULL pointers, FLMISR_ERR_CONFIG for a band plan (world > 1),
 * FLMISR_ERR_CUDA on a launch failure.
 */
flmisr_status flmisr_interp_fuse(flmisr_plan_t plan, const float* lr_stack, float* hr_out, void* cuda_stream);

/*
 * flmisr_reconstruct_async / flmisr_finish: the two halves of flmisr_reconstruct.  _async enqueues the
 * whole reconstruction (same arguments and errors as flmisr_reconstruct) plus the status read-back and
 * returns without synchronising; flmisr_finish waits for it and fills `report` (nullable).  Exactly one
 * _finish per _async; the caller's buffers must stay valid until _finish returns.  Used for streamed
 * acquisition and for timing the device work without host latency.
 */
flmisr_status flmisr_reconstruct_async(flmisr_plan_t plan, const float* lr_stack, const float* x0, float* hr_out,
                                       void* cuda_stream);
flmisr_status flmisr_finish(flmisr_plan_t plan, flmisr_report* report);

/*
 * flmisr_profile: per-kernel CUDA-event timing on the launching stream.  enable = 1 turns it on and
 * resets the counters, 0 turns it off and resets, -1 only reads.  out8 (nullable, host, 8 doubles)
 * receives {launches, total ms} for: [0] value+gradient kernel (or, when the plan runs the SCG loop as
 * one persistent kernel, that kernel: one launch per reconstruction), [1] update+curvature kernel
 * (0 launches in the persistent mode), [2] setup+finalize (ingest, x0, state, output), [3] whole
 * reconstructions.
 */
flmisr_status flmisr_profile(flmisr_plan_t plan, int32_t enable, double* out8);

/*
 * flmisr_reconstruct_host:flmisr_reconstruct for HOST buffers (end-to-end path): lr_stack_host
 * (k x lr_h x lr_w fp32) is staged through the plan's pinned buffer and copied H2D, hr_out_host
 * (H x W fp32; rank 0 / world 1) receives the D2H copy.  Same errors as flmisr_reconstruct.
 */
flmisr_status flmisr_reconstruct_host(flmisr_plan_t plan, const float* lr_stack_host, float* hr_out_host,
                                      flmisr_report* report);

/* flmisr_destroy: free all device memory, the CUDA graph, streams and the NCCL communicator.
 * NULL is accepted.  Always returns FLMISR_OK unless a CUDA call fails. */
flmisr_status flmisr_destroy(flmisr_plan_t plan);

/* Thread-local message describing the last error returned on this thread ("" if none). */
const char* flmisr_last_error(void);

/* Row band of `rank` among `world` (Eq. subfunction): rows [row_lo, row_hi) of an H-row HR
 * image, boundaries rounded down to multiples of mag, remainder to the last band.  Host only. */
flmisr_status flmisr_band(int32_t H, int32_t world, int32_t rank, int32_t mag, int32_t* row_lo, int32_t* row_hi);

/*
 * Single-device band emulation (tests, no NCCL): flmisr_plan_virtual builds the plan of band
 * cfg->rank of cfg->world exactly like flmisr_plan but without a communicator (nccl_unique_id is
 * ignored); flmisr_reconstruct_virtual runs the `g` bands plans[0..g-1] (ranks 0..g-1 of one
 * configuration, same device) on plans[0]'s stream in Algorithm 1's order, with device-to-device
 * copies in place of the allgather and the halo send/recv, and writes the fused image to hr_out
 * (device, H x W).  lr_stack / x0 as in flmisr_reconstruct.  report: band 0's (all bands must agree;
 * FLMISR_ERR_NUMERIC otherwise).
 */
flmisr_status flmisr_plan_virtual(const flmisr_config* cfg, flmisr_plan_t* out);
flmisr_status flmisr_reconstruct_virtual(flmisr_plan_t* plans, int32_t g, const float* lr_stack, const float* x0,
                                         float* hr_out, flmisr_report* report);

/*
 * Row bands over peer memory (the inner-outer border exchange P:197 and the
 * consensus sums P:195 of Alg. 1).  Each band's whole SCG loop is ONE persistent
 * cooperative kernel; after every phase the bands meet through peer-mapped memory: each band stores
 * its fp64 band sums into every rank's mailbox and bumps a per-sender flag word, every rank sums the
 * world band sums in rank order (bit-identical consensus scalars everywhere), and the value+gradient
 * pass stores the candidate r's eta boundary rows straight into the neighbours' halo buffers.
 *
 * flmisr_reconstruct_virtual_peer: the g bands plans[0..g-1] (flmisr_plan_virtual, ranks 0..g-1 of one
 *   streaming-path configuration, same device; each virtual plan is sized for 1/g of the SMs) in ONE
 *   cooperative launch with local pointers in place of the peer mappings.  Arguments, output and report
 *   as flmisr_reconstruct_virtual.  FLMISR_ERR_CONFIG if the bands do not fit one cooperative wave.
 * flmisr_peer_export: a world > 1 plan (flmisr_plan) writes FLMISR_PEER_BLOB_BYTES bytes to out (host):
 *   CUDA IPC handles of its halo buffers and mailbox block, its geometry (H, W, n_iter, halo, pitch), a
 *   digest of its configuration and its device's PCI bus id.  The caller all-gathers the blobs of the
 *   world ranks (e.g. over the torch process group) in rank order.
 * flmisr_peer_connect: blobs = world x FLMISR_PEER_BLOB_BYTES bytes (host, rank order).  Maps every
 *   peer's mailbox block and the neighbours' halo buffers (same node, NVLink / NVSwitch), after which
 *   flmisr_reconstruct* on this plan runs the peer loop (the band gather to rank 0 stays on NCCL).
 *   Every rank of the group must call flmisr_reconstruct* the same number of times with the same
 *   n_iter.  Errors: FLMISR_ERR_CONFIG (not a streaming band plan, bad blobs, already connected, a
 *   peer that planned a different problem, a peer device without peer access or native peer
 *   atomics), FLMISR_ERR_CUDA (IPC mapping failed).  On any error the plan stays on the NCCL
 *   transport and remains usable.  A peer-loop reconstruction whose band barrier does not complete
 *   within 20 s (a lost rank, peer memory without working system-scope atomics) abandons the loop on
 *   every band and returns FLMISR_ERR_CUDA naming the timeout (failed_stage 3) instead of hanging;
 *   the device stays usable.  Status: EXPERIMENTAL on real multi-GPU nodes -- the kernel code
 *   is parity-tested in the single-device emulation (flmisr_reconstruct_virtual_peer); the IPC /
 *   system-scope path has not run on more than one GPU in this repository's test environment.
 */
#define FLMISR_PEER_BLOB_BYTES 256
flmisr_status flmisr_reconstruct_virtual_peer(flmisr_plan_t* plans, int32_t g, const float* lr_stack,
                                              const float* x0, float* hr_out, flmisr_report* report);
flmisr_status flmisr_peer_export(flmisr_plan_t plan, void* out);
flmisr_status flmisr_peer_connect(flmisr_plan_t plan, const void* blobs);

/* Fill out128 (128 bytes, host) with a fresh ncclUniqueId (rank 0 calls this and broadcasts the
 * bytes to the other ranks, e.g. over the torch process group; S:288 coordinator role). */
flmisr_status flmisr_nccl_unique_id(void* out128);

/* HR geometry of a plan: H, W, owned rows [row_lo, row_hi); fast_path = 0 general-geometry kernels
 * (unfused), 1 tiled polyphase kernels, 2 streaming polyphase kernels, 3 fused general-geometry
 * kernels (every integer phase in [-(R+1), mag-1+R]; FLMISR_GEN2=1 at plan time forces 0); loop_kernel = 1 when the SCG loop runs as
 * one persistent cooperative kernel (streaming path, world 1).  Any output may be NULL. */
flmisr_status flmisr_plan_info(flmisr_plan_t plan, int32_t* H, int32_t* W, int32_t* row_lo, int32_t* row_hi,
                               int32_t* fast_path, int32_t* loop_kernel);

/* ------------------------------------------------------------------------------------------
 * Streaming capture-reconstruct pipeline (fig:capture: each view is
 * super-resolved while the next one is acquired).  A pipeline owns `depth` device input and output
 * slots and two copy streams beside the plan's compute stream; for every submitted view it enqueues
 *   H2D of the LR stack (upload stream) -> [uint16 -> fp32 on the device] -> the plan's whole SCG
 *   reconstruction (compute stream) -> D2H of the HR image (download stream),
 * so view j+1's upload and view j-1's download overlap view j's reconstruction.
 *
 * flmisr_pipeline_create: plan = a world-1 plan or one band of a partitioned group (every rank of
 *   the group creates its pipeline and submits the same views in the same order); the pipeline uses
 *   the plan's buffers exclusively (no flmisr_reconstruct* on that plan until it is destroyed).
 *   depth >= 2 slots (views in flight).  input_u16: 0 = fp32 frames; 1 = uint16 frames, value =
 *   u16_scale * code, converted on the device (halves the H2D bytes; 16-bit detector data).
 *   Errors: FLMISR_ERR_SHAPE (bad arguments), FLMISR_ERR_CUDA (allocation).
 * flmisr_pipeline_submit: lr_host = host k x lr_h x lr_w frames (fp32 or uint16); hr_host = host
 *   H x W fp32 destination (world 1 / rank 0; may be NULL on other ranks).  Page-locked buffers are
 *   DMA'd in place and must stay valid until the view completes; pageable buffers are staged through
 *   per-slot pinned memory (the output is copied out when the slot is next reused or at _wait).
 *   Returns once the view is enqueued; blocks only while the slot it reuses is still in flight.
 * flmisr_pipeline_wait: drain every submitted view.  n_done (nullable) = views completed since
 *   create; report (nullable; f_trace is not filled) = the most recent view's.  Returns the first
 *   error any view hit since the last _wait (FLMISR_ERR_NUMERIC if a view's loop froze).
 * flmisr_pipeline_destroy: drain and free (NULL accepted); the plan stays valid.  A plan drives at
 *   most one pipeline; flmisr_destroy(plan) drains and frees it too (its handle is then invalid).
 * ------------------------------------------------------------------------------------------ */
typedef struct flmisr_pipeline_s* flmisr_pipeline_t;
flmisr_status flmisr_pipeline_create(flmisr_plan_t plan, int32_t depth, int32_t input_u16, float u16_scale,
                                     flmisr_pipeline_t* out);
flmisr_status flmisr_pipeline_submit(flmisr_pipeline_t pipe, const void* lr_host, float* hr_host);
flmisr_status flmisr_pipeline_wait(flmisr_pipeline_t pipe, int64_t* n_done, flmisr_report* report);
flmisr_status flmisr_pipeline_destroy(flmisr_pipeline_t pipe);

/* ------------------------------------------------------------------------------------------
 * Debug entry points (parity tests).  Each runs the SAME kernels as the SCG loop (for VALUE,
 * GRAD and CURV) or shares their device stencil code (FORWARD, ADJOINT) on the plan's stream,
 * synchronises, and returns.  All array arguments are device pointers (fp32), scalars host.
 * ------------------------------------------------------------------------------------------ */
typedef enum {
    FLMISR_OP_FORWARD = 0, /* in0 = x (H x W)            -> out = A x as k x lr_h x lr_w frames          */
    FLMISR_OP_ADJOINT = 1, /* in0 = w (k x lr_h x lr_w)  -> out = sum_i A_i^T w_i (H x W)                */
    FLMISR_OP_GRAD = 2,    /* in0 = x, lr = y            -> out = -grad J(x) (H x W); s[0..1] = D, R      */
    FLMISR_OP_CURV = 3,    /* in0 = x, in1 = p, lr = y   -> s[0] = p^T Hess J(x) p, s[1] = <p,p>          */
    FLMISR_OP_VALUE = 4,   /* in0 = x, lr = y            -> s[0] = D(x), s[1] = R(x)  (J = D + lambda R)  */
    FLMISR_OP_X0 = 5,      /* lr = y                     -> out = bilinear initial estimate (H x W)       */
    FLMISR_OP_INTERP = 6   /* lr = y -> out = multi-image interpolation fusion: every LR pixel of an
                              integer-phase frame at its HR site (first frame wins), the bilinear initial
                              estimate on sites no frame covers (none on the fast path)                  */
} flmisr_op;

flmisr_status flmisr_debug_apply(flmisr_plan_t plan, int32_t op, const float* lr_stack, const float* in0,
                                 const float* in1, float* out, double* scalars_out);

#ifdef __cplusplus
}
#endif
#endif /* FLMISR_H */
