/*
 * flmisr_oracle.c -- plain, slow, single-threaded fp64 CPU oracle for the FL-MISR
 * SCG reconstruction (arXiv 2108.04315).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2108_04315_b200/) never imports, links or calls it, and shares no code with it.
 *
 * Every function cites the passage it follows.  P:n = /root/reference/PAPER.md line n,
 * S:n = /root/reference/SPEC.md line n, "reading k" = DESIGN.md section 3 ledger entry k.
 * There is no blocking, fusion or reordering beyond what the definitions state: each
 * quantity is evaluated straight from its definition with plain loops.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py against a
 * closed form, a library routine (scipy.ndimage / scipy.sparse.linalg.cg), a worked
 * example (tests/golden/) or brute force.  Against the paper's own numbers parity is
 * unpinned (the paper prints no image, trajectory or numeric SCG example).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t k, lr_h, lr_w;   /* K LR frames of lr_h x lr_w                                  */
    const double* shifts;    /* k x 2 (dy, dx) in LR pixels (reading 3)                      */
    const double* psf;       /* psf_h x psf_w, odd sizes, centred, applied as correlation   */
    int32_t psf_h, psf_w;
    int32_t mag;             /* SR factor r (reading: "magnification" of north_star)        */
    int32_t p_norm;          /* 1: Charbonnier-smoothed L1 (reading 8); 2: squared   */
    double eps;              /* Charbonnier epsilon (reading 8)                              */
    double lambda;           /* regularisation weight (Eq. objective; 0.05 at P:271) */
    double btv_alpha;        /* gamma(d) = alpha^(dx+dy) (Eq. prior)                  */
    int32_t btv_window;      /* w: dx, dy in [0, w-1] (reading 6/7)                  */
    int32_t btv_offsets;     /* 0: the paper's quadrant dx, dy in [0, w-1] (reading 6);
                                1: Farsiu's set dy = m in [0, w-1], dx = l in [-(w-1), w-1], l + m >= 0
                                (the [BTV] citation), gamma = alpha^(|l|+m) */
} orc_problem;

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
static int H_of(const orc_problem* pb) { return pb->mag * pb->lr_h; }
static int W_of(const orc_problem* pb) { return pb->mag * pb->lr_w; }

/* The BTV offset set Q of Eq. prior as an explicit list, (0,0) excluded:
 * quadrant (reading 6): d = (dy, dx), dy, dx in [0, w-1], gamma(d) = alpha^(dx+dy);
 * Farsiu (NEXT-4): d = (m, l), m in [0, w-1], l in [-(w-1), w-1], l + m >= 0, gamma = alpha^(|l|+m).
 * Returns the number of offsets (<= 3w^2). */
static int btv_offset_list(const orc_problem* pb, int* dys, int* dxs, double* gams)
{
    int w = pb->btv_window, n = 0;
    for (int dy = 0; dy < w; ++dy)
        for (int dx = pb->btv_offsets ? -(w - 1) : 0; dx < w; ++dx) {
            if (dy == 0 && dx == 0) continue;
            if (pb->btv_offsets && dx + dy < 0) continue;
            dys[n] = dy; dxs[n] = dx;
            gams[n] = pow(pb->btv_alpha, (dx < 0 ? -dx : dx) + dy);
            ++n;
        }
    return n;
}
#define BTV_MAXOFF 64

/* ---------------------------------------------------------------------------------
 * Per-frame operator A_i = D B M_i  (Eq. sisr; reading 1, 3, 4, 19).
 * M_i: bilinear translation by t_i = mag * shift_i HR px, s_i = floor(t_i), phi_i = t_i - s_i.
 * B:   correlation with the centred PSF h.
 * D:   point sampling at stride mag.
 * Composed: kappa_i = h (*) b_phi on offsets P in [-Ry, Ry+1], Q in [-Rx, Rx+1], and
 *   (A_i x)(a,b) = sum_{P,Q} kappa_i(P,Q) x[clamp(mag*a + s_y + P), clamp(mag*b + s_x + Q)].
 * --------------------------------------------------------------------------------- */
typedef struct {
    int sy, sx;          /* integer phase s_i                     */
    int ry, rx;          /* PSF radii                             */
    int kh, kw;          /* kappa storage (2Ry+2) x (2Rx+2)       */
    int py1, qx1;        /* support P in [-Ry, py1], Q in [-Rx, qx1]: py1 = Ry+1 if phi_y != 0
                            else Ry (kappa is identically zero on the extra row/column)   */
    double kap[64 * 64]; /* kappa(P,Q) at [(P+Ry)*kw + (Q+Rx)]    */
} orc_taps;

/* kappa_i = h (*) b_phi, with b_phi = {(1-fy)(1-fx), (1-fy)fx, fy(1-fx), fy fx} at offsets
 * (0,0), (0,1), (1,0), (1,1): M_i samples x at u + t_i by bilinear interpolation,
 * then B correlates with h, so x(u + PQ + s + ab) carries h(PQ) b_phi(ab). */
int orc_taps_build(const orc_problem* pb, int i, orc_taps* t)
{
    double ty = pb->mag * pb->shifts[2 * i + 0];
    double tx = pb->mag * pb->shifts[2 * i + 1];
    double fsy = floor(ty), fsx = floor(tx);
    double fy = ty - fsy, fx = tx - fsx;
    t->sy = (int)fsy; t->sx = (int)fsx;
    t->ry = pb->psf_h / 2; t->rx = pb->psf_w / 2;
    t->kh = 2 * t->ry + 2; t->kw = 2 * t->rx + 2;
    t->py1 = fy != 0.0 ? t->ry + 1 : t->ry;
    t->qx1 = fx != 0.0 ? t->rx + 1 : t->rx;
    if (t->kh * t->kw > 64 * 64) return -1;
    memset(t->kap, 0, sizeof(double) * (size_t)(t->kh * t->kw));
    double bw[2][2] = {{(1 - fy) * (1 - fx), (1 - fy) * fx}, {fy * (1 - fx), fy * fx}};
    for (int P = -t->ry; P <= t->ry; ++P)
        for (int Q = -t->rx; Q <= t->rx; ++Q) {
            double hv = pb->psf[(P + t->ry) * pb->psf_w + (Q + t->rx)];
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b)
                    t->kap[(P + a + t->ry) * t->kw + (Q + b + t->rx)] += hv * bw[a][b];
        }
    return 0;
}

/* (A_i x)(a,b) for one LR pixel -- the definition above, with clamp (reading 4). */
static double fwd_pixel(const orc_problem* pb, const orc_taps* t, const double* x, int a, int b)
{
    int H = H_of(pb), W = W_of(pb);
    double acc = 0.0;
    for (int P = -t->ry; P <= t->py1; ++P)
        for (int Q = -t->rx; Q <= t->qx1; ++Q) {
            int u = clampi(pb->mag * a + t->sy + P, 0, H - 1);
            int v = clampi(pb->mag * b + t->sx + Q, 0, W - 1);
            acc += t->kap[(P + t->ry) * t->kw + (Q + t->rx)] * x[(size_t)u * W + v];
        }
    return acc;
}

/* y_i = A_i x for all frames (Eq. sisr P:67 without noise; A = DBM P:71). y: k x lr_h x lr_w. */
int orc_forward(const orc_problem* pb, const double* x, double* y)
{
    orc_taps t;
    for (int i = 0; i < pb->k; ++i) {
        if (orc_taps_build(pb, i, &t)) return -1;
        for (int a = 0; a < pb->lr_h; ++a)
            for (int b = 0; b < pb->lr_w; ++b)
                y[((size_t)i * pb->lr_h + a) * pb->lr_w + b] = fwd_pixel(pb, &t, x, a, b);
    }
    return 0;
}

/* x = sum_i A_i^T y_i, scatter form: every (a,b,P,Q) adds kappa_i(P,Q) y_i(a,b) to the x index
 * the forward read from (clamped).  This is the exact transpose (S:37-63 spmv_transpose). */
int orc_adjoint(const orc_problem* pb, const double* y, double* x)
{
    int H = H_of(pb), W = W_of(pb);
    orc_taps t;
    memset(x, 0, sizeof(double) * (size_t)H * W);
    for (int i = 0; i < pb->k; ++i) {
        if (orc_taps_build(pb, i, &t)) return -1;
        for (int a = 0; a < pb->lr_h; ++a)
            for (int b = 0; b < pb->lr_w; ++b) {
                double yv = y[((size_t)i * pb->lr_h + a) * pb->lr_w + b];
                for (int P = -t.ry; P <= t.py1; ++P)
                    for (int Q = -t.rx; Q <= t.qx1; ++Q) {
                        int u = clampi(pb->mag * a + t.sy + P, 0, H - 1);
                        int v = clampi(pb->mag * b + t.sx + Q, 0, W - 1);
                        x[(size_t)u * W + v] += t.kap[(P + t.ry) * t.kw + (Q + t.rx)] * yv;
                    }
            }
    }
    return 0;
}

/* ---------------------------------------------------------------------------------
 * Robust penalties (reading 8): rho_1(t) = sqrt(t^2+eps^2) - eps, rho_2(t) = t^2.
 * --------------------------------------------------------------------------------- */
static double rho(int p, double e, double t)   { return p == 2 ? t * t : sqrt(t * t + e * e) - e; }
static double drho(int p, double e, double t)  { return p == 2 ? 2.0 * t : t / sqrt(t * t + e * e); }
static double d2rho(int p, double e, double t) { double q = t * t + e * e; return p == 2 ? 2.0 : e * e / (q * sqrt(q)); }
static double psi(double e, double t)   { return sqrt(t * t + e * e) - e; }
static double dpsi(double e, double t)  { return t / sqrt(t * t + e * e); }
static double d2psi(double e, double t) { double q = t * t + e * e; return e * e / (q * sqrt(q)); }

/* Row-range ownership used for partitioned partial sums (reading 18):
 * LR pixel (i,a,b) belongs to the band holding HR row clamp(mag*a + s_iy); a BTV pair (u, u+d)
 * belongs to the band holding u; a vector element belongs to the band holding its row.
 * [row_lo, row_hi) = [0, H) gives the centralised quantity. */

/* Data term D(x) = sum_i sum_{a,b} rho(A_i x - y_i)  (Eq. misr, p in {1,2}). */
static double data_value_rows(const orc_problem* pb, const double* x, const double* y, int lo, int hi)
{
    int H = H_of(pb);
    orc_taps t;
    double acc = 0.0;
    for (int i = 0; i < pb->k; ++i) {
        orc_taps_build(pb, i, &t);
        for (int a = 0; a < pb->lr_h; ++a) {
            int own = clampi(pb->mag * a + t.sy, 0, H - 1);
            if (own < lo || own >= hi) continue;
            for (int b = 0; b < pb->lr_w; ++b) {
                double e = fwd_pixel(pb, &t, x, a, b) - y[((size_t)i * pb->lr_h + a) * pb->lr_w + b];
                acc += rho(pb->p_norm, pb->eps, e);
            }
        }
    }
    return acc;
}

/* BTV R(x) = sum_{d in Q} gamma(d) sum_{u, u+d in Omega} psi(x_u - x_{u+d})
 * (Eq. prior; valid pairs only, reading 5; quadrant offsets, reading 6). */
static double btv_value_rows(const orc_problem* pb, const double* x, int lo, int hi)
{
    int H = H_of(pb), W = W_of(pb);
    int dys[BTV_MAXOFF], dxs[BTV_MAXOFF];
    double gams[BTV_MAXOFF];
    int no = btv_offset_list(pb, dys, dxs, gams);
    double acc = 0.0;
    for (int o = 0; o < no; ++o) {
        int dy = dys[o], dx = dxs[o];
        double s = 0.0;
        for (int u = lo; u < hi; ++u)
            for (int v = 0; v < W; ++v) {
                if (u + dy >= H || v + dx < 0 || v + dx >= W) continue;
                s += psi(pb->eps, x[(size_t)u * W + v] - x[(size_t)(u + dy) * W + v + dx]);
            }
        acc += gams[o] * s;
    }
    return acc;
}

/* D and R separately, over the whole image (Eq. objective: J = D + lambda R). */
void orc_value(const orc_problem* pb, const double* x, const double* y, double* D, double* R)
{
    *D = data_value_rows(pb, x, y, 0, H_of(pb));
    *R = btv_value_rows(pb, x, 0, H_of(pb));
}

double orc_objective(const orc_problem* pb, const double* x, const double* y)
{
    double D, R;
    orc_value(pb, x, y, &D, &R);
    return D + pb->lambda * R;
}

/* grad J = sum_i A_i^T rho'(A_i x - y_i) + lambda grad R  (Eq. objective P:166 differentiated;
 * A_i^T by the scatter of orc_adjoint; grad R by differentiating each pair term). */
int orc_grad(const orc_problem* pb, const double* x, const double* y, double* g)
{
    int H = H_of(pb), W = W_of(pb);
    int dys[BTV_MAXOFF], dxs[BTV_MAXOFF];
    double gams[BTV_MAXOFF];
    int no = btv_offset_list(pb, dys, dxs, gams);
    size_t M = (size_t)pb->k * pb->lr_h * pb->lr_w;
    double* res = (double*)malloc(sizeof(double) * M);
    if (!res) return -1;
    orc_forward(pb, x, res);
    for (size_t m = 0; m < M; ++m) res[m] = drho(pb->p_norm, pb->eps, res[m] - y[m]);
    orc_adjoint(pb, res, g);
    free(res);
    for (int o = 0; o < no; ++o) {
        int dy = dys[o], dx = dxs[o];
        double gam = pb->lambda * gams[o];
        for (int u = 0; u + dy < H; ++u)
            for (int v = 0; v < W; ++v) {
                if (v + dx < 0 || v + dx >= W) continue;
                size_t i0 = (size_t)u * W + v, i1 = (size_t)(u + dy) * W + v + dx;
                double d = gam * dpsi(pb->eps, x[i0] - x[i1]);
                g[i0] += d;
                g[i1] -= d;
            }
    }
    return 0;
}

/* Exact directional curvature p^T (Hess J)(x) p (reading 16: the sigma -> 0 limit of the paper's
 * probe, Alg. 1 lines 6-11):
 *   sum_i sum rho''(A_i x - y_i) (A_i p)^2 + lambda sum_d gamma_d sum_valid psi''(x_u-x_{u+d}) (p_u-p_{u+d})^2. */
static double curv_rows(const orc_problem* pb, const double* x, const double* y, const double* p, int lo, int hi)
{
    int H = H_of(pb), W = W_of(pb);
    int dys[BTV_MAXOFF], dxs[BTV_MAXOFF];
    double gams[BTV_MAXOFF];
    int no = btv_offset_list(pb, dys, dxs, gams);
    orc_taps t;
    double acc = 0.0;
    for (int i = 0; i < pb->k; ++i) {
        orc_taps_build(pb, i, &t);
        for (int a = 0; a < pb->lr_h; ++a) {
            int own = clampi(pb->mag * a + t.sy, 0, H - 1);
            if (own < lo || own >= hi) continue;
            for (int b = 0; b < pb->lr_w; ++b) {
                double e = fwd_pixel(pb, &t, x, a, b) - y[((size_t)i * pb->lr_h + a) * pb->lr_w + b];
                double ap = fwd_pixel(pb, &t, p, a, b);
                acc += d2rho(pb->p_norm, pb->eps, e) * ap * ap;
            }
        }
    }
    double reg = 0.0;
    for (int o = 0; o < no; ++o) {
        int dy = dys[o], dx = dxs[o];
        double s = 0.0;
        for (int u = lo; u < hi; ++u)
            for (int v = 0; v < W; ++v) {
                if (u + dy >= H || v + dx < 0 || v + dx >= W) continue;
                size_t i0 = (size_t)u * W + v, i1 = (size_t)(u + dy) * W + v + dx;
                double dp = p[i0] - p[i1];
                s += d2psi(pb->eps, x[i0] - x[i1]) * dp * dp;
            }
        reg += gams[o] * s;
    }
    return acc + pb->lambda * reg;
}

double orc_curv(const orc_problem* pb, const double* x, const double* y, const double* p)
{
    return curv_rows(pb, x, y, p, 0, H_of(pb));
}

/* Initial estimate x0 (reading 14): bilinear upsample of frame 0,
 * x0(u,v) = bilerp(y_0, (u - t_0y)/mag, (v - t_0x)/mag), LR indices clamped to the frame. */
void orc_init_x0(const orc_problem* pb, const double* y, double* x0)
{
    int H = H_of(pb), W = W_of(pb), h = pb->lr_h, w = pb->lr_w;
    double ty = pb->mag * pb->shifts[0], tx = pb->mag * pb->shifts[1];
    for (int u = 0; u < H; ++u)
        for (int v = 0; v < W; ++v) {
            double a = (u - ty) / pb->mag, b = (v - tx) / pb->mag;
            double a0 = floor(a), b0 = floor(b);
            double fa = a - a0, fb = b - b0;
            int ia0 = clampi((int)a0, 0, h - 1), ia1 = clampi((int)a0 + 1, 0, h - 1);
            int ib0 = clampi((int)b0, 0, w - 1), ib1 = clampi((int)b0 + 1, 0, w - 1);
            x0[(size_t)u * W + v] = (1 - fa) * (1 - fb) * y[(size_t)ia0 * w + ib0] + (1 - fa) * fb * y[(size_t)ia0 * w + ib1]
                                  + fa * (1 - fb) * y[(size_t)ia1 * w + ib0] + fa * fb * y[(size_t)ia1 * w + ib1];
        }
}

/* ---------------------------------------------------------------------------------
 * Moller SCG (the [SCG] citation at P:186 / P:206), with the consensus of P:195 / P:209-222
 * made exact (reading 11, 12): every scalar is a sum of per-band partials over owned elements,
 * summed in band order, and the SCG scalar logic runs once on the sums.
 *
 * Band simulation (g > 1): band h owns HR rows [lo_h, hi_h) and stores its own copy of rows
 * [lo_h - eta, hi_h + eta) of x, p, r.  The gradient is evaluated from that local copy for
 * owned rows only; afterwards the halo rows of r are replaced by the neighbours' owned rows
 * (inner-outer border exchange, fig:communication); x and p halos are updated with
 * the same arithmetic as owned rows.  Reads outside the local copy are impossible by
 * construction: a local copy is expanded into a full-size NaN-filled scratch image, so an
 * insufficient eta poisons the result (pinned by the g-invariance test).
 * --------------------------------------------------------------------------------- */
typedef struct {
    int32_t iters_run, accepted, converged_at, nonfinite;
} orc_stats;

enum { CURV_EXACT = 0, CURV_FD = 1 };

static void band_bounds(int H, int g, int mag, int h, int* lo, int* hi)
{
    /* rows [floor(h*H/g) rounded down to a multiple of mag, ...) (reading: bands multiples of mag) */
    long l = ((long)h * H / g) / mag * mag, u = ((long)(h + 1) * H / g) / mag * mag;
    if (h == g - 1) u = H;
    *lo = (int)l; *hi = (int)u;
}

/* local gradient of band [lo,hi) from a local copy of x restricted to rows [lo-eta, hi+eta). */
static int band_grad(const orc_problem* pb, const double* xfull, const double* y, int lo, int hi, int eta,
                     double* scratch, double* gfull_out)
{
    int H = H_of(pb), W = W_of(pb);
    size_t N = (size_t)H * W;
    for (size_t n = 0; n < N; ++n) scratch[n] = NAN;
    int rlo = lo - eta < 0 ? 0 : lo - eta, rhi = hi + eta > H ? H : hi + eta;
    memcpy(scratch + (size_t)rlo * W, xfull + (size_t)rlo * W, sizeof(double) * (size_t)(rhi - rlo) * W);
    double* g = (double*)malloc(sizeof(double) * N);
    if (!g) return -1;
    /* A^T rho'(A x - y) restricted to LR pixels whose residual can touch the owned rows; the
     * others read NaN rows and must not be used.  Compute residual per LR pixel only when its
     * sample row (before clamp) lies within the PSF reach of the band. */
    memset(g, 0, sizeof(double) * N);
    orc_taps t;
    for (int i = 0; i < pb->k; ++i) {
        orc_taps_build(pb, i, &t);
        for (int a = 0; a < pb->lr_h; ++a) {
            int base = pb->mag * a + t.sy;
            /* rows touched by this LR pixel: clamp(base + P), P in [-ry, py1] */
            int tlo = clampi(base - t.ry, 0, H - 1), thi = clampi(base + t.py1, 0, H - 1);
            if (thi < lo || tlo >= hi) continue;
            for (int b = 0; b < pb->lr_w; ++b) {
                double e = fwd_pixel(pb, &t, scratch, a, b) - y[((size_t)i * pb->lr_h + a) * pb->lr_w + b];
                double wv = drho(pb->p_norm, pb->eps, e);
                for (int P = -t.ry; P <= t.py1; ++P)
                    for (int Q = -t.rx; Q <= t.qx1; ++Q) {
                        int u = clampi(base + P, 0, H - 1);
                        int v = clampi(pb->mag * b + t.sx + Q, 0, W - 1);
                        g[(size_t)u * W + v] += t.kap[(P + t.ry) * t.kw + (Q + t.rx)] * wv;
                    }
            }
        }
    }
    int dys[BTV_MAXOFF], dxs[BTV_MAXOFF];
    double gams[BTV_MAXOFF];
    int no = btv_offset_list(pb, dys, dxs, gams);
    for (int o = 0; o < no; ++o) {
        int dy = dys[o], dx = dxs[o];
        double gam = pb->lambda * gams[o];
        for (int u = lo - dy; u < hi; ++u) {
            if (u < 0 || u + dy >= H) continue;
            for (int v = 0; v < W; ++v) {
                if (v + dx < 0 || v + dx >= W) continue;
                size_t i0 = (size_t)u * W + v, i1 = (size_t)(u + dy) * W + v + dx;
                double d = gam * dpsi(pb->eps, scratch[i0] - scratch[i1]);
                g[i0] += d;
                g[i1] -= d;
            }
        }
    }
    for (int u = lo; u < hi; ++u)
        memcpy(gfull_out + (size_t)u * W, g + (size_t)u * W, sizeof(double) * W);
    free(g);
    return 0;
}

static double dot_rows(const double* a, const double* b, int W, int lo, int hi)
{
    double s = 0.0;
    for (size_t n = (size_t)lo * W; n < (size_t)hi * W; ++n) s += a[n] * b[n];
    return s;
}

/* Central objective from per-band partials (Alg. 1 line 17: f_c = sum_h f_h). */
static double f_consensus(const orc_problem* pb, const double* x, const double* y, int g)
{
    int H = H_of(pb);
    double f = 0.0;
    for (int h = 0; h < g; ++h) {
        int lo, hi;
        band_bounds(H, g, pb->mag, h, &lo, &hi);
        f += data_value_rows(pb, x, y, lo, hi) + pb->lambda * btv_value_rows(pb, x, lo, hi);
    }
    return f;
}

/* -grad J assembled band by band (g = 1: one band, the centralised gradient). */
static int neg_grad_consensus(const orc_problem* pb, const double* x, const double* y, int g, int eta,
                              double* scratch, double* r)
{
    int H = H_of(pb), W = W_of(pb);
    size_t N = (size_t)H * W;
    if (g == 1) {
        if (orc_grad(pb, x, y, r)) return -1;
    } else {
        for (int h = 0; h < g; ++h) {
            int lo, hi;
            band_bounds(H, g, pb->mag, h, &lo, &hi);
            if (band_grad(pb, x, y, lo, hi, eta, scratch, r)) return -1;
        }
    }
    for (size_t n = 0; n < N; ++n) r[n] = -r[n];
    return 0;
}

static double dot_consensus(const orc_problem* pb, const double* a, const double* b, int g)
{
    int H = H_of(pb), W = W_of(pb);
    double s = 0.0;
    for (int h = 0; h < g; ++h) {
        int lo, hi;
        band_bounds(H, g, pb->mag, h, &lo, &hi);
        s += dot_rows(a, b, W, lo, hi);
    }
    return s;
}

static double curv_consensus(const orc_problem* pb, const double* x, const double* y, const double* p, int g)
{
    int H = H_of(pb);
    double s = 0.0;
    for (int h = 0; h < g; ++h) {
        int lo, hi;
        band_bounds(H, g, pb->mag, h, &lo, &hi);
        s += curv_rows(pb, x, y, p, lo, hi);
    }
    return s;
}

/*
 * orc_scg: Moller's SCG literally ("Algorithm"):
 *   x <- x0; r <- -grad J(x); p <- r; f <- J(x); lam <- lam0; lamb <- 0; success <- 1; k <- 0
 *   while k < n_iter:
 *     if success: pp <- <p,p>; delta <- CURV(x,p)     (EXACT: p^T Hess p; FD: sigma_k = sigma0/sqrt(pp),
 *                                                       delta <- <p, grad J(x + sigma_k p) - grad J(x)>/sigma_k)
 *     delta <- delta + (lam - lamb) pp
 *     if delta <= 0: lamb <- 2(lam - delta/pp); delta <- -delta + lam pp; lam <- lamb
 *     mu <- <p,r>; alpha <- mu/delta
 *     f_new <- J(x + alpha p); Delta <- 2 delta (f - f_new)/mu^2
 *     if Delta >= 0: x <- x + alpha p; r_old <- r; r <- -grad J(x); f <- f_new; lamb <- 0; success <- 1
 *                    if (k+1) mod N == 0: p <- r else beta <- (<r,r> - <r,r_old>)/mu; p <- r + beta p
 *                    if Delta >= 0.75: lam <- lam/4
 *     else: lamb <- lam; success <- 0
 *     if Delta < 0.25: lam <- lam + delta (1 - Delta)/pp
 *     k <- k + 1
 *     if <r,r> == 0: break
 * trace (nullable): (n_iter+1) rows of 6 doubles (k, f, <r,r>, alpha, lam, accepted);
 * row 0 is the initial state (alpha = 0, accepted = 1).
 * rules (SURVEY 8(f) NEXT-4 variants, bit mask; 0 = Moller literal as above):
 *   1  PR+ restart: beta <- max(beta, 0), i.e. p <- r on non-positive beta
 *   2  Netlab scale rules (Nabney's scg.m): every pass delta <- curv + lam pp with curv the last
 *      CURV(x,p); if delta <= 0: delta <- lam pp, lam <- lam - curv/pp (no lamb); after the
 *      comparison: Delta < 0.25 -> lam <- min(4 lam, 1e100); Delta > 0.75 -> lam <- max(lam/2, 1e-15)
 * x0 == NULL -> orc_init_x0 on frame 0.  g >= 1 bands, eta halo rows (band simulation above).
 * Returns 0, or -1 on allocation failure, -2 when a consensus scalar is non-finite.
 */
int orc_scg(const orc_problem* pb, const double* y, const double* x0, int n_iter, int curv_mode,
            double sigma0, double lambda0, int g, int eta, double* x_out, double* trace, orc_stats* st, int rules)
{
    const int pr_plus = rules & 1, netlab = rules & 2;
    double curv = 0.0;
    int H = H_of(pb), W = W_of(pb);
    size_t N = (size_t)H * W;
    double *x = x_out, *r = malloc(sizeof(double) * N), *p = malloc(sizeof(double) * N);
    double *rold = malloc(sizeof(double) * N), *xn = malloc(sizeof(double) * N);
    double *scratch = malloc(sizeof(double) * N), *gt = malloc(sizeof(double) * N);
    int rc = 0;
    if (!r || !p || !rold || !xn || !scratch || !gt) { rc = -1; goto out; }
    if (x0) memcpy(x, x0, sizeof(double) * N);
    else orc_init_x0(pb, y, x);
    if (neg_grad_consensus(pb, x, y, g, eta, scratch, r)) { rc = -1; goto out; }
    memcpy(p, r, sizeof(double) * N);
    double f = f_consensus(pb, x, y, g);
    double lam = lambda0, lamb = 0.0, delta = 0.0, pp = 0.0, rr = dot_consensus(pb, r, r, g);
    int success = 1, k = 0;
    if (st) { st->iters_run = 0; st->accepted = 0; st->converged_at = -1; st->nonfinite = 0; }
    if (trace) {
        for (int i = 0; i < (n_iter + 1) * 6; ++i) trace[i] = 0.0;
        trace[0] = 0; trace[1] = f; trace[2] = rr; trace[3] = 0; trace[4] = lam; trace[5] = 1;
    }
    if (rr == 0.0) { if (st) st->converged_at = 0; goto out; }
    while (k < n_iter) {
        if (success) {
            pp = dot_consensus(pb, p, p, g);
            if (curv_mode == CURV_FD) {
                double sig = sigma0 / sqrt(pp);
                for (size_t n = 0; n < N; ++n) xn[n] = x[n] + sig * p[n];
                if (neg_grad_consensus(pb, xn, y, g, eta, scratch, gt)) { rc = -1; goto out; }
                /* grad J(x+sig p) - grad J(x) = -gt + r */
                double s = 0.0;
                for (int h = 0; h < g; ++h) {
                    int lo, hi;
                    band_bounds(H, g, pb->mag, h, &lo, &hi);
                    double sh = 0.0;
                    for (size_t n = (size_t)lo * W; n < (size_t)hi * W; ++n) sh += p[n] * (r[n] - gt[n]);
                    s += sh;
                }
                delta = s / sig;
            } else {
                delta = curv_consensus(pb, x, y, p, g);
            }
            curv = delta;
        }
        if (netlab) {
            delta = curv + lam * pp;
            if (delta <= 0.0) {
                delta = lam * pp;
                lam = lam - curv / pp;
            }
        } else {
            delta = delta + (lam - lamb) * pp;
            if (delta <= 0.0) {
                lamb = 2.0 * (lam - delta / pp);
                delta = -delta + lam * pp;
                lam = lamb;
            }
        }
        double mu = dot_consensus(pb, p, r, g);
        double alpha = mu / delta;
        for (size_t n = 0; n < N; ++n) xn[n] = x[n] + alpha * p[n];
        double fnew = f_consensus(pb, xn, y, g);
        double Delta = 2.0 * delta * (f - fnew) / (mu * mu);
        if (!isfinite(delta) || !isfinite(alpha) || !isfinite(fnew) || !isfinite(Delta)) {
            if (st) st->nonfinite = 1;
            rc = -2;
            goto out;
        }
        int acc = Delta >= 0.0;
        if (acc) {
            memcpy(x, xn, sizeof(double) * N);
            memcpy(rold, r, sizeof(double) * N);
            if (neg_grad_consensus(pb, x, y, g, eta, scratch, r)) { rc = -1; goto out; }
            f = fnew;
            lamb = 0.0;
            success = 1;
            rr = dot_consensus(pb, r, r, g);
            if ((size_t)(k + 1) % N == 0) {
                memcpy(p, r, sizeof(double) * N);
            } else {
                double beta = (rr - dot_consensus(pb, r, rold, g)) / mu;
                if (pr_plus && beta < 0.0) beta = 0.0;
                for (size_t n = 0; n < N; ++n) p[n] = r[n] + beta * p[n];
            }
            if (!netlab && Delta >= 0.75) lam = lam / 4.0;
            if (st) st->accepted++;
        } else {
            lamb = lam;
            success = 0;
        }
        if (netlab) {
            if (Delta < 0.25) lam = fmin(4.0 * lam, 1e100);
            if (Delta > 0.75) lam = fmax(0.5 * lam, 1e-15);
        } else if (Delta < 0.25) {
            lam = lam + delta * (1.0 - Delta) / pp;
        }
        k = k + 1;
        if (st) st->iters_run = k;
        if (trace) {
            double* row = trace + (size_t)k * 6;
            row[0] = k; row[1] = f; row[2] = rr; row[3] = alpha; row[4] = lam; row[5] = acc;
        }
        if (rr == 0.0) { if (st) st->converged_at = k; break; }
    }
out:
    free(r); free(p); free(rold); free(xn); free(scratch); free(gt);
    return rc;
}

/* Partitioned partial sums exposed for the additivity pins. */
double orc_value_rows(const orc_problem* pb, const double* x, const double* y, int lo, int hi)
{
    return data_value_rows(pb, x, y, lo, hi) + pb->lambda * btv_value_rows(pb, x, lo, hi);
}

void orc_band_bounds(int H, int g, int mag, int h, int* lo, int* hi) { band_bounds(H, g, mag, h, lo, hi); }

/* Multi-image interpolation fusion (tab:runtime "interpolation" row P:432): every
 * LR pixel is inserted at its integer HR location r*(a,b) + s_i (frames with a fractional phase are
 * not inserted); HR sites no frame covers take the bilinear upsample of frame 0 (orc_init_x0).
 * The first frame (in index order) that covers a site wins. */
void orc_interp_fuse(const orc_problem* pb, const double* y, double* out)
{
    int H = H_of(pb), W = W_of(pb);
    orc_init_x0(pb, y, out);
    unsigned char* done = (unsigned char*)calloc((size_t)H * W, 1);
    for (int i = 0; i < pb->k; ++i) {
        double ty = pb->mag * pb->shifts[2 * i], tx = pb->mag * pb->shifts[2 * i + 1];
        if (ty != floor(ty) || tx != floor(tx)) continue;
        int sy = (int)ty, sx = (int)tx;
        for (int a = 0; a < pb->lr_h; ++a)
            for (int b = 0; b < pb->lr_w; ++b) {
                int u = pb->mag * a + sy, v = pb->mag * b + sx;
                if (u < 0 || u >= H || v < 0 || v >= W || (done && done[(size_t)u * W + v])) continue;
                out[(size_t)u * W + v] = y[((size_t)i * pb->lr_h + a) * pb->lr_w + b];
                if (done) done[(size_t)u * W + v] = 1;
            }
    }
    free(done);
}
