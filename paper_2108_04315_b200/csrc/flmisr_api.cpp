// flmisr_api.cpp -- C ABI (include/flmisr.h): plan validation and construction, device memory,
// the SCG driver that enqueues one reconstruction, NCCL plumbing for row bands, debug entries.
//
// Host-side design: the plan derives the per-frame taps kappa_i =
// PSF (*) bilinear(frac(mag*shift_i)) in fp64 (A_i = D B M_i, Eq. sisr), detects the
// polyphase fast path, fixes the row band + halo of this rank (Eq. subfunction; halo eta =
// max(2 KR, w-1), reading 17), and allocates every buffer once ("calculated once ... and
// shared by all rotation angles").  flmisr_reconstruct enqueues the whole SCG loop; every SCG
// decision is taken on the device (no host round-trip until the final synchronisation).
#include "flmisr.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "flmisr_internal.h"

using namespace flmisr;

namespace {

thread_local std::string g_last_error;

flmisr_status fail(flmisr_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(FLMISR_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));       \
    } while (0)

// ---- NCCL through dlopen (the torch-bundled libnccl.so.2 is already mapped in torch processes) ----
struct NcclApi {
    bool ok = false;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
};

static void nccl_load(NcclApi& api);
NcclApi& nccl() {   // loaded once, thread-safe (plans may be created from several host threads)
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] { nccl_load(api); });
    return api;
}
static void nccl_load(NcclApi& api) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.ok = api.CommInitRank && api.CommDestroy && api.AllGather && api.Send && api.Recv && api.GroupStart &&
             api.GroupEnd && api.GetErrorString;
}

#define NCCL_TRY(expr)                                                                              \
    do {                                                                                            \
        ncclResult_t r_ = (expr);                                                                   \
        if (r_ != ncclSuccess)                                                                      \
            return fail(FLMISR_ERR_NCCL, std::string(#expr) + ": " + nccl().GetErrorString(r_));   \
    } while (0)

}  // namespace

// Optional per-kernel timing with CUDA events on the launching stream (bench.py roofline).
struct Prof {
    bool enabled = false;
    std::vector<cudaEvent_t> ev;
    double ms[4] = {0, 0, 0, 0};   // value_grad, update_curv, other (setup + finalize), whole call
    long long n[4] = {0, 0, 0, 0};
};

struct flmisr_plan_s {
    flmisr_config cfg{};
    std::vector<double> shifts, psf;
    int H = 0, W = 0, pitch = 0, kr = 0, bw = 0, pn = 1, eta = 0;
    int row_lo = 0, row_hi = 0, store_lo = 0, store_hi = 0;
    int fast = 0;
    int stream_path = 0;   // 1: register-streaming kernels (flmisr_stream.cu), 0: tiled kernels
    int pc = 0;            // 1: per-phase streaming kernels (flmisr_stream4.cu): complete phases, kappa per frame
    int all_int = 0;       // 1: every frame's HR shift mag * shift_i is integral
    int complete = 0;      // 1: every phase class holds a frame (polyphase-complete)
    PcTaps pct{};          // their taps per phase class
    int virt = 0;          // 1: band of an in-process virtual group (flmisr_reconstruct_virtual), no NCCL
    float* halo_mem = nullptr;   // send/recv halo rows (world > 1)
    StencilParams sp{};
    IngestParams ip{};
    Buffers b{};
    GenParams gp{};          // general-geometry path (fast == 0)
    float* gmem = nullptr;   // general path: taps, LR copy, rho' weights
    double* gpart = nullptr; // general path: first-pass partials
    size_t hr_bytes = 0;     // bytes of one stored HR buffer
    float* mem = nullptr;    // one allocation for all HR buffers
    double* dmem = nullptr;  // partials + rank sums + trace + grid-barrier counter
    ScgState* st = nullptr;
    ScgState* st_host = nullptr;  // pinned
    double* trace_host = nullptr; // pinned
    float* pin_in = nullptr;      // pinned staging for the host entry point
    float* pin_out = nullptr;
    float* d_lr = nullptr;        // device LR stack for the host entry point
    float* d_out = nullptr;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    float* recv_top = nullptr;
    float* recv_bot = nullptr;
    cudaEvent_t done_ev = nullptr;
    cudaStream_t last_stream = nullptr;
    int pending = 0;
    int prof_marks = 0;
    Prof prof;
    cudaGraphExec_t graph_exec = nullptr;   // the captured SCG loop (world == 1)
    cudaGraphExec_t graph_exec_prof = nullptr;   // the same with per-kernel event records
    int no_graph = 0;                       // FLMISR_NO_GRAPH=1: always launch eagerly
    cudaGraphExec_t virt_graph = nullptr;   // band 0 of a virtual group: the group's captured loop
    std::vector<const void*> virt_key;      // ... and the bands (plan, buffers) it was captured for
    int persist = 0;                        // 1: the SCG loop runs as one persistent cooperative kernel
    int prof_mode = 0;                      // layout of the profiling marks of the last call (0 per-kernel, 1 loop)
    flmisr_pipeline_s* pipe = nullptr;      // the pipeline driving this plan, if any
    // row bands over peer memory (world > 1)
    unsigned char* peer_mem = nullptr;      // arrival counter, epoch word, mailbox (peer_mem layout below)
    int peer = 0;                           // 1: flmisr_peer_connect done, the SCG loop is k_scg_peer_loop
    PeerLoop pl{};                          // its parameters (g = 1)
    Buffers b_peer{};                       // b with the send rows pointing into the neighbours' halo buffers
    std::vector<void*> ipc_open;            // peer mappings to close
};

// peer_mem layout: arrival counter (u64), epoch word (u32), mailbox [2][world][PEER_MAXCTAS][NSLOT] fp64
// (det mode: [2][world][PEER_MAXCTAS][FXW] 128-bit words)
constexpr int PEER_MAXCTAS = 256;
size_t peer_mem_bytes(int world) { return 64 + (size_t)2 * world * PEER_MAXCTAS * FXW * 16; }
unsigned long long* peer_cnt(unsigned char* m) { return reinterpret_cast<unsigned long long*>(m); }
unsigned* peer_epoch(unsigned char* m) { return reinterpret_cast<unsigned*>(m + 8); }
double* peer_mbox(unsigned char* m) { return reinterpret_cast<double*>(m + 64); }
static flmisr_status failed_status(const ScgState& hs, const char* what) {
    if (hs.failed_stage == FAIL_PEER_TIMEOUT)
        return fail(FLMISR_ERR_CUDA, std::string(what) + ": the peer band barrier timed out at SCG pass " +
                                         std::to_string(hs.failed_iter) + " (a rank or its peer memory is unreachable)");
    return fail(FLMISR_ERR_NUMERIC, std::string(what) + ": non-finite consensus scalar at SCG pass " +
                                        std::to_string(hs.failed_iter) + " (stage " + std::to_string(hs.failed_stage) + ")");
}

namespace {

bool is_odd(int v) { return v > 0 && (v & 1); }

// kappa_i = h (*) b_phi on offsets P in [-R, R+1] x [-R, R+1] (A_i = D B M_i, reading 19).
void composed_taps(const flmisr_config& c, int i, std::vector<double>& kap, int& sy, int& sx, double& fy,
                   double& fx) {
    double ty = c.mag * c.shifts[2 * i], tx = c.mag * c.shifts[2 * i + 1];
    double fsy = std::floor(ty), fsx = std::floor(tx);
    sy = (int)fsy; sx = (int)fsx;
    fy = ty - fsy; fx = tx - fsx;
    int ry = c.psf_h / 2, rx = c.psf_w / 2, R = std::max(ry, rx);
    int KD = 2 * R + 2;
    kap.assign((size_t)KD * KD, 0.0);
    double bw[2][2] = {{(1 - fy) * (1 - fx), (1 - fy) * fx}, {fy * (1 - fx), fy * fx}};
    for (int P = -ry; P <= ry; ++P)
        for (int Q = -rx; Q <= rx; ++Q) {
            double h = c.psf[(P + ry) * c.psf_w + (Q + rx)];
            for (int a = 0; a < 2; ++a)
                for (int bb = 0; bb < 2; ++bb) kap[(size_t)(P + a + R) * KD + (Q + bb + R)] += h * bw[a][bb];
        }
}

flmisr_status validate(const flmisr_config* c, bool virt) {
    if (!c) return fail(FLMISR_ERR_CONFIG, "config is NULL");
    if (c->k < 1) return fail(FLMISR_ERR_CONFIG, "k must be >= 1 (S:96)");
    if (c->lr_h < 1 || c->lr_w < 1) return fail(FLMISR_ERR_CONFIG, "lr_h and lr_w must be >= 1");
    if (c->mag < 1 || c->mag > 4) return fail(FLMISR_ERR_CONFIG, "mag must be in [1, 4]");
    if (!c->shifts || !c->psf) return fail(FLMISR_ERR_CONFIG, "shifts and psf must be non-NULL host arrays");
    if (!is_odd(c->psf_h) || !is_odd(c->psf_w) || c->psf_h > 5 || c->psf_w > 5)
        return fail(FLMISR_ERR_CONFIG, "psf sizes must be odd and <= 5 (S:123)");
    double s = 0.0;
    for (int i = 0; i < c->psf_h * c->psf_w; ++i) {
        if (!(c->psf[i] >= 0.0) || !std::isfinite(c->psf[i]))
            return fail(FLMISR_ERR_CONFIG, "psf entries must be finite and >= 0 (S:95)");
        s += c->psf[i];
    }
    if (std::fabs(s - 1.0) > 1e-6) return fail(FLMISR_ERR_CONFIG, "psf must sum to 1 within 1e-6 (S:95)");
    for (int i = 0; i < 2 * c->k; ++i)
        if (!std::isfinite(c->shifts[i])) return fail(FLMISR_ERR_CONFIG, "shifts must be finite");
    if (c->p_norm != 1 && c->p_norm != 2) return fail(FLMISR_ERR_CONFIG, "p_norm must be 1 or 2 (Eq. misr, P:121)");
    if (!(c->l1_eps > 0.0) || !std::isfinite(c->l1_eps)) return fail(FLMISR_ERR_CONFIG, "l1_eps must be > 0 (S:183)");
    if (!(c->lambda >= 0.0) || !std::isfinite(c->lambda)) return fail(FLMISR_ERR_CONFIG, "lambda must be >= 0 (S:183)");
    if (!(c->btv_alpha > 0.0 && c->btv_alpha < 1.0))
        return fail(FLMISR_ERR_CONFIG, "btv_alpha must be in (0, 1) (P:138, S:183)");
    if (c->btv_window < 1 || c->btv_window > MAXBW) return fail(FLMISR_ERR_CONFIG, "btv_window must be in [1, 3]");
    if (c->n_iter < 0) return fail(FLMISR_ERR_CONFIG, "n_iter must be >= 0");
    if (c->x0_mode != 0 && c->x0_mode != 1)
        return fail(FLMISR_ERR_CONFIG, "x0_mode must be 0 (bilinear frame 0) or 1 (interpolation fusion)");
    if (c->det_rows != 0 && (c->det_rows < 3 || c->det_rows > 4095 || c->det_rows % 3 != 0))
        return fail(FLMISR_ERR_CONFIG, "det_rows must be 0 (off) or a multiple of 3 in [3, 4095] HR rows");
    if (!(c->scg_lambda0 > 0.0) || !std::isfinite(c->scg_lambda0))
        return fail(FLMISR_ERR_CONFIG, "scg_lambda0 must be > 0 (S:362)");
    if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return fail(FLMISR_ERR_CONFIG, "need 0 <= rank < world");
    if (c->world > 1 && !virt && !c->nccl_unique_id)
        return fail(FLMISR_ERR_CONFIG, "world > 1 needs nccl_unique_id");
    if (c->btv_offsets != 0 && c->btv_offsets != 1)
        return fail(FLMISR_ERR_CONFIG, "btv_offsets must be 0 (quadrant, P:136) or 1 (Farsiu)");
    if (c->scg_rules < 0 || c->scg_rules > 3) return fail(FLMISR_ERR_CONFIG, "scg_rules must be in [0, 3]");
    if (c->curv_mode != 0 && c->curv_mode != 1) return fail(FLMISR_ERR_CONFIG, "curv_mode must be 0 (exact) or 1 (FD)");
    if (c->curv_mode == 1 && !(c->scg_sigma0 > 0.0 && std::isfinite(c->scg_sigma0)))
        return fail(FLMISR_ERR_CONFIG, "curv_mode = 1 needs scg_sigma0 > 0 (S:362)");
    if (c->curv_mode == 1 && c->world > 1)
        return fail(FLMISR_ERR_CONFIG, "the finite-difference curvature (curv_mode = 1) runs on the general path: world must be 1");
    if (c->btv_offsets == 1 && c->world > 1)
        return fail(FLMISR_ERR_CONFIG, "Farsiu BTV offsets (btv_offsets = 1) run on the general path: world must be 1");
    return FLMISR_OK;
}

}  // namespace

extern "C" {

const char* flmisr_last_error(void) { return g_last_error.c_str(); }

static int world_of(const flmisr_config& c) { return c.world; }

static flmisr_status make_plan(const flmisr_config* cfg, flmisr_plan_t* out, bool virt) {
    if (!out) return fail(FLMISR_ERR_CONFIG, "out is NULL");
    *out = nullptr;
    flmisr_status vs = validate(cfg, virt);
    if (vs != FLMISR_OK) return vs;
    const flmisr_config& c = *cfg;

    // ---- taps, phases, fast-path detection ----
    const int mag = c.mag, K = c.k;
    const int R = std::max(c.psf_h / 2, c.psf_w / 2);
    std::vector<double> kap0;
    int sy0, sx0;
    double fy0, fx0;
    composed_taps(c, 0, kap0, sy0, sx0, fy0, fx0);
    bool fast = (K == mag * mag);
    std::vector<int> frame_of_phase(mag * mag, -1);
    std::vector<int> sy(K), sx(K);
    for (int i = 0; i < K; ++i) {
        std::vector<double> kap;
        double fy, fx;
        composed_taps(c, i, kap, sy[i], sx[i], fy, fx);
        for (size_t j = 0; j < kap.size(); ++j)   // common kappa up to fp64 rounding of mag*shift
            if (std::fabs(kap[j] - kap0[j]) > 1e-12) fast = false;
        if (sy[i] < 0 || sy[i] >= mag || sx[i] < 0 || sx[i] >= mag) { fast = false; continue; }
        int ph = sy[i] * mag + sx[i];
        if (frame_of_phase[ph] >= 0) fast = false;
        else frame_of_phase[ph] = i;
    }
    if (std::getenv("FLMISR_FORCE_GENERAL") || c.btv_offsets == 1 || c.curv_mode == 1) fast = false;
    // per-phase path (flmisr_stream4.cu): x2 with K <= 4 frames at distinct integer phases in [0,2)^2 whose
    // composed kernels differ (sub-pixel remainders per frame), PSF <= 3x3, one GPU: the polyphase Y with a
    // 4x4 kernel per phase class runs on streaming kernels instead of the general path.  A phase no frame
    // covers gets a zero kernel and a zero sample: its residual, penalty, weight and curvature are 0.
    bool pc = false;
    if (!fast && mag == 2 && K >= 1 && K <= 4 && std::max(c.psf_h, c.psf_w) <= 3 && c.world == 1 && !virt &&
        c.det_rows == 0 &&
        c.btv_offsets == 0 && c.curv_mode == 0 && (c.lr_w % 2) == 0 && c.lr_w >= 4 && c.lr_h >= 4 &&
        !std::getenv("FLMISR_FORCE_GENERAL") && !std::getenv("FLMISR_NO_PC")) {
        int seen[4] = {-1, -1, -1, -1};
        pc = true;
        for (int i = 0; i < K && pc; ++i) {
            if (sy[i] < 0 || sy[i] > 1 || sx[i] < 0 || sx[i] > 1 || seen[sy[i] * 2 + sx[i]] >= 0) pc = false;
            else seen[sy[i] * 2 + sx[i]] = i;
        }
        if (pc) {
            for (int ph = 0; ph < 4; ++ph) frame_of_phase[ph] = seen[ph];
            fast = true;
        }
    }
    if (!fast && c.world > 1)
        return fail(FLMISR_ERR_CONFIG,
                    "row-band partitioning (world > 1) needs the polyphase fast path (K = mag^2 frames with distinct "
                    "integer HR phases in [0,mag)^2 and one common sub-pixel remainder); general geometries run on "
                    "one GPU per projection");
    if (!fast && K > GMAXK) return fail(FLMISR_ERR_CONFIG, "the general-geometry path supports k <= 64 frames");
    const bool frac = (fy0 != 0.0 || fx0 != 0.0);
    const int kr = pc ? R + 1 : (fast ? (frac ? R + 1 : R) : R + 1);
    if (fast && kr > MAXKR) return fail(FLMISR_ERR_CONFIG, "kappa radius exceeds 3");
    if (c.world > 1 && !virt && !nccl().ok) return fail(FLMISR_ERR_NCCL, "libnccl.so.2 could not be loaded");

    auto* p = new flmisr_plan_s();
    p->cfg = c;
    p->shifts.assign(c.shifts, c.shifts + 2 * K);
    p->psf.assign(c.psf, c.psf + c.psf_h * c.psf_w);
    p->cfg.shifts = p->shifts.data();
    p->cfg.psf = p->psf.data();
    p->cfg.nccl_unique_id = nullptr;
    p->fast = fast ? 1 : 0;
    p->pc = pc ? 1 : 0;
    p->complete = 1;
    for (int ph = 0; ph < mag * mag; ++ph) if (frame_of_phase[ph] < 0) p->complete = 0;
    p->all_int = 1;
    for (int i = 0; i < 2 * K; ++i)
        if (mag * c.shifts[i] != std::floor(mag * c.shifts[i])) p->all_int = 0;
    if (c.x0_mode == 1 && world_of(c) > 1 && !p->all_int) {
        delete p;
        return fail(FLMISR_ERR_CONFIG, "x0_mode = 1 with fractional HR shifts needs world == 1");
    }
    if (pc) {   // kappa of each phase class, offsets [-R, R+1] placed in the 4x4 window [-1, 2]
        for (int ph = 0; ph < 4; ++ph) {
            for (int j = 0; j < 16; ++j) p->pct.k[ph][j] = 0.0f;
            if (frame_of_phase[ph] < 0) continue;   // missing phase: zero kernel
            std::vector<double> kap;
            int syi, sxi;
            double fy, fx;
            composed_taps(c, frame_of_phase[ph], kap, syi, sxi, fy, fx);
            const int KD = 2 * R + 2;
            for (int P = -R; P <= R + 1; ++P)
                for (int Q = -R; Q <= R + 1; ++Q)
                    p->pct.k[ph][(P + 1) * 4 + (Q + 1)] = (float)kap[(size_t)(P + R) * KD + (Q + R)];
        }
    }
    p->virt = virt ? 1 : 0;
    p->no_graph = std::getenv("FLMISR_NO_GRAPH") != nullptr;
    p->H = mag * c.lr_h;
    p->W = mag * c.lr_w;
    p->pitch = (p->W + 31) / 32 * 32;
    p->kr = kr;
    p->bw = c.btv_window;
    p->pn = c.p_norm;
    p->eta = std::max(2 * kr, c.btv_window - 1);

    // ---- row band (Eq. subfunction): multiples of mag (det mode: of lcm(det_rows, mag), so every
    // band is a union of the fixed global tiles), remainder to the last band ----
    const int world = c.world, rank = c.rank;
    const int bunit = c.det_rows ? c.det_rows / std::gcd(c.det_rows, mag) * mag : mag;
    auto band = [&](int h, int& lo, int& hi) {
        lo = (int)(((long long)h * p->H / world) / bunit * bunit);
        hi = (h == world - 1) ? p->H : (int)(((long long)(h + 1) * p->H / world) / bunit * bunit);
    };
    for (int h = 0; h < world && world > 1; ++h) {
        int lo, hi;
        band(h, lo, hi);
        if (hi - lo < std::max(p->eta, 1) || (c.det_rows && hi - lo < bunit)) {
            const int need = std::max(std::max(p->eta, 1), c.det_rows ? bunit : 1);
            const int minH = world * (c.det_rows ? bunit : need * mag);
            delete p;
            return fail(FLMISR_ERR_CONFIG, "image too small for " + std::to_string(world) +
                                               " partitions: every band needs >= eta = " + std::to_string(need) +
                                               " rows; minimum HR height " + std::to_string(minH) + " (S:254)");
        }
    }
    band(rank, p->row_lo, p->row_hi);
    p->store_lo = std::max(0, p->row_lo - p->eta);
    p->store_hi = std::min(p->H, p->row_hi + p->eta);
    const int srows = p->store_hi - p->store_lo;

    // ---- stencil parameters ----
    StencilParams& sp = p->sp;
    sp.H = p->H; sp.W = p->W; sp.pitch = p->pitch;
    sp.row_lo = p->row_lo; sp.row_hi = p->row_hi;
    sp.store_lo = p->store_lo; sp.store_hi = p->store_hi;
    sp.tile_row0 = p->row_lo;
    sp.tiles_x = (p->W + TX - 1) / TX;
    sp.tiles_y = (p->row_hi - p->row_lo + TY - 1) / TY;
    sp.world = world;
    sp.eps = (float)c.l1_eps;
    sp.eps2 = (float)(c.l1_eps * c.l1_eps);
    sp.lam = (float)c.lambda;
    {
        const int KD = 2 * R + 2, kd = 2 * kr + 1;
        for (int i = 0; i < MAXTAPS; ++i) sp.taps[i] = 0.0f;
        // kap0 offsets [-R, R+1] -> centred (2kr+1)^2 with offset index P + kr
        for (int P = -R; P <= R + 1; ++P)
            for (int Q = -R; Q <= R + 1; ++Q) {
                double v = kap0[(size_t)(P + R) * KD + (Q + R)];
                if (v == 0.0) continue;
                sp.taps[(P + kr) * kd + (Q + kr)] = (float)v;
            }
        for (int i = 0; i < MAXBW * MAXBW; ++i) sp.gam[i] = 0.0f;
        for (int dy = 0; dy < c.btv_window; ++dy)
            for (int dx = 0; dx < c.btv_window; ++dx)
                if (dy || dx) sp.gam[dy * MAXBW + dx] = (float)std::pow(c.btv_alpha, dx + dy);
        for (int cl = 0; cl < 4; ++cl) sp.gcls[cl] = std::pow(c.btv_alpha, cl + 1);
        for (int i = 0; i < MAXBW * MAXBW; ++i) sp.lgam[i] = (float)(c.lambda * (double)sp.gam[i]);
        for (int cl = 0; cl < 4; ++cl) sp.lgc[cl] = (float)(c.lambda * (double)(float)std::pow(c.btv_alpha, cl + 1));
        // identity affine correction (tiled kernels compute complete values)
        for (int k = 0; k < NSLOT; ++k) {
            sp.aff_vg[k] = 1.0; sp.aff_vg[NSLOT + k] = 0.0;
            sp.aff_uc[k] = 1.0; sp.aff_uc[NSLOT + k] = 0.0;
        }
        // ---- streaming path (flmisr_stream.cu): separable kappa with KR <= 1, W % 4 == 0 ----
        std::vector<double> K3(9, 0.0);   // kappa as a centred 3x3 (KR <= 1)
        if (kr <= 1) {   // fp64 kappa (offsets [-R, R+1]) -> centred 3x3
            const int KD = 2 * R + 2;
            for (int P = -1; P <= 1; ++P)
                for (int Q = -1; Q <= 1; ++Q)
                    if (P + R >= 0 && P + R < KD && Q + R >= 0 && Q + R < KD)
                        K3[(P + 1) * 3 + (Q + 1)] = kap0[(size_t)(P + R) * KD + (Q + R)];
        }
        int pm = 0;
        for (int i = 1; i < 9; ++i)
            if (std::fabs(K3[i]) > std::fabs(K3[pm])) pm = i;
        const int Pm = pm / 3, Qm = pm % 3;
        double a3[3], b3[3], err = 0.0;
        for (int i = 0; i < 3; ++i) { a3[i] = K3[i * 3 + Qm]; b3[i] = K3[Pm * 3 + i] / K3[pm]; }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) err = std::max(err, std::fabs(K3[i * 3 + j] - a3[i] * b3[j]));
        const bool separable = kr <= 1 && err <= 1e-12 * std::fabs(K3[pm]);
        p->stream_path = (fast && separable && (p->W % 4 == 0) && p->W >= 8 && p->H >= 4 &&
                          std::getenv("FLMISR_FORCE_TILED") == nullptr) || pc;
        if (c.det_rows && !p->stream_path) {
            delete p;
            return fail(FLMISR_ERR_CONFIG, "det_rows needs the streaming path (fast_path 2: polyphase-complete stack, "
                                           "separable composed kernel of radius <= 1, HR width % 4 == 0)");
        }
        if (p->stream_path) {
            for (int i = 0; i < 3; ++i) { sp.ka[i] = (float)a3[i]; sp.kb[i] = (float)b3[i]; }
            sp.wpb = pc ? PC_WPB : SWPB;
            // strips of SCOLS columns stepping by SSTEP (common kappa) or PC_SSTEP (per-phase kernels)
            const int halo = pc ? (SCOLS - PC_SSTEP) / 2 : SHALO, step = SCOLS - 2 * halo;
            sp.nstrips = 1 + (p->W > SCOLS - halo ? (p->W - (SCOLS - halo) + step - 1) / step : 0);
            int nsm = 148;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c.device);
            // virtual bands share one device: each gets 1/world of the SMs (the peer-loop emulation runs
            // all bands in one cooperative launch)
            if (virt) nsm = std::max(1, nsm / world);
            const long long cap = (long long)nsm * (pc ? 1 : SMINB) * sp.wpb;   // one wave of resident warps
            const int rows = p->row_hi - p->row_lo;
            // Work items, one warp each, one wave.  Warps touching an image or band edge run the border
            // instantiation, ~1.4x slower per row (per-warp timing), so border pieces
            // get seg_b ~ seg_rows / 1.4 rows: interior strips are split seg_b | seg_rows ... | seg_b,
            // the two edge strips (column 0 / W-1) into pieces of seg_b.
            // measured border/interior cost ratios (border-piece sweeps, profiles/r02_edge_ratio_sweep.txt):
            // 1.4 for the common-kappa kernels at x2 (C2, C3), 1.6 at x3 (C4), 1.8 for the per-phase
            // kernels (G3: 262 vs 242 proj/s at 1.4)
            double ratio = pc ? 1.8 : (mag == 3 ? 1.6 : 1.4);
            if (const char* ev = std::getenv("FLMISR_EDGE_RATIO")) ratio = std::max(1.0, std::atof(ev));
            sp.ne = sp.nstrips >= 2 ? 2 : 1;
            sp.ni = sp.nstrips - sp.ne;
            // segment lengths: 1 mod 3 for the common-kappa kernels (row loop unrolled by 3; a partial last
            // group -- any length -- measured 2-3% slower on C2/C3, profiles/r02_any_length_segments.txt),
            // multiples of 4 for the per-phase kernels (unrolled by 4; every segment starts on an even row)
            auto to1mod3 = [pc](int v) {
                v = std::max(v, 4);
                return pc ? (v + 3) / 4 * 4 : v + ((1 - v % 3) + 3) % 3;
            };
            auto nseg_int = [&](int Si, int Sb) {   // pieces of one interior strip
                return rows <= 2 * Sb ? (rows + Sb - 1) / Sb : 2 + (rows - 2 * Sb + Si - 1) / Si;
            };
            auto items = [&](int Si, int Sb) {
                return (long long)sp.ni * nseg_int(Si, Sb) + (long long)sp.ne * ((rows + Sb - 1) / Sb);
            };
            // the shortest segments (S = 1 mod 3, >= S0) whose items fit one wave: every resident warp
            // busy, each warp's serial row chain as short as possible (the phase time is ~ rows per
            // warp x ~1.1 us at C3; a band of a g-GPU partition has few rows)
            int S0 = 4;
            if (const char* ev = std::getenv("FLMISR_SEG_MIN")) S0 = std::max(4, std::atoi(ev));
            int S = to1mod3(S0);
            // a piece of S rows streams S + 2 rows (2 warm-up rows); a border piece streams at 1/ratio the
            // speed, so it gets Sb with Sb + 2 = (S + 2) / ratio (measured: C2 452 -> 498 proj/s over
            // Sb = S / ratio; C3 unchanged)
            auto border_rows = [&](int Si) { return to1mod3((int)((Si + 2) / ratio - 2.0)); };
            int Sb = border_rows(S);
            while (S < rows && items(S, Sb) > cap) {
                S += pc ? 4 : 3;
                Sb = border_rows(S);
            }
            if (const char* ev = std::getenv("FLMISR_SEG_ROWS")) {   // tuning override (S = 1 mod 3), never
                const int v = std::atoi(ev);                        // below the one-wave minimum
                if (v >= 4 && to1mod3(v) > S) { S = to1mod3(v); Sb = border_rows(S); }
            }
            S = std::min(S, pc ? to1mod3(rows) : rows + ((1 - rows % 3) + 3) % 3);   // smallest admissible >= rows
            Sb = std::min(Sb, S);
            sp.seg_rows = S;
            sp.seg_b = Sb;
            sp.nseg_i = nseg_int(S, Sb);
            if (rows <= 2 * Sb) sp.seg_rows = Sb;   // short bands: interior strips in seg_b pieces too
            if (c.det_rows) {
                // det mode: the same one-wave search in units of the fixed tiles of T rows (bands are unions
                // of them; flmisr_stream_common.cuh geometry_item), so every segment is a union of whole
                // tiles and each tile's sums are committed exactly inside the row loop
                const int T = c.det_rows, nt = (rows + T - 1) / T;
                auto nseg_t = [&](int m, int mb) {
                    return nt <= 2 * mb ? (nt + mb - 1) / mb : 2 + (nt - 2 * mb + m - 1) / m;
                };
                auto items_t = [&](int m, int mb) {
                    return (long long)sp.ni * nseg_t(m, mb) + (long long)sp.ne * ((nt + mb - 1) / mb);
                };
                auto mb_of = [&](int m) {
                    return std::min(m, std::max(1, (int)std::lround(((double)(m * T + 2) / ratio - 2.0) / T)));
                };
                int m = 1, mb = mb_of(1);
                while (m < nt && items_t(m, mb) > cap) { ++m; mb = mb_of(m); }
                sp.seg_rows = m * T;
                sp.seg_b = mb * T;
                sp.nseg_i = nseg_t(m, mb);
                sp.nseg_b = (nt + mb - 1) / mb;
                sp.det_rows = T;
            } else {
                sp.nseg_b = (rows + Sb - 1) / Sb;
            }
            sp.n_int = sp.ni * sp.nseg_i;
            sp.nitems = sp.n_int + sp.ne * sp.nseg_b;
            sp.nsegs = sp.nseg_i;
            // persistent loop kernels: one warp per item (one wave by construction; in det mode unless a band
            // has more strips x tiles than a wave holds, then a grid-stride loop over the items)
            sp.loop_warps = c.det_rows ? (int)std::min<long long>(sp.nitems, cap) : sp.nitems;
            sp.det = c.det_rows ? 1 : 0;
            // hoisted constants: D = sum q rs - eps N, R = sum gamma q rs - eps sum_d gamma_d n_d,
            // curvature sums carry eps^2 (p = 1) or 2 (p = 2)
            const double eps = c.l1_eps;
            double npairs_g = 0.0;
            for (int dy = 0; dy < c.btv_window; ++dy)
                for (int dx = 0; dx < c.btv_window; ++dx) {
                    if (!dy && !dx) continue;
                    const long long nr = std::max(0, std::min(p->row_hi, p->H - dy) - p->row_lo);
                    npairs_g += std::pow(c.btv_alpha, dx + dy) * (double)nr * (double)(p->W - dx);
                }
            sp.aff_vg[NSLOT + 0] = c.p_norm == 1 ? -eps * (double)rows * p->W : 0.0;
            sp.aff_vg[NSLOT + 1] = -eps * npairs_g;
            sp.aff_uc[0] = c.p_norm == 1 ? eps * eps : 2.0;
            sp.aff_uc[1] = eps * eps;
            // det mode: the offsets of the whole image, applied once to the exact all-band total
            double npairs_all = 0.0;
            for (int dy = 0; dy < c.btv_window; ++dy)
                for (int dx = 0; dx < c.btv_window; ++dx) {
                    if (!dy && !dx) continue;
                    npairs_all += std::pow(c.btv_alpha, dx + dy) * (double)(p->H - dy) * (double)(p->W - dx);
                }
            for (int k = 0; k < NSLOT; ++k) { sp.det_off_vg[k] = 0.0; sp.det_off_uc[k] = sp.aff_uc[NSLOT + k]; }
            sp.det_off_vg[0] = c.p_norm == 1 ? -eps * (double)p->H * p->W : 0.0;
            sp.det_off_vg[1] = -eps * npairs_all;
        }
    }
    IngestParams& ip = p->ip;
    ip.H = p->H; ip.W = p->W; ip.pitch = p->pitch; ip.k = K; ip.lr_h = c.lr_h; ip.lr_w = c.lr_w; ip.mag = mag;
    ip.store_lo = p->store_lo; ip.store_hi = p->store_hi;
    for (int i = 0; i < 16; ++i) { ip.frame_of_phase[i] = 0; ip.sy[i] = 0; ip.sx[i] = 0; }
    if (fast) {
        for (int ph = 0; ph < mag * mag; ++ph) ip.frame_of_phase[ph] = frame_of_phase[ph];
        for (int i = 0; i < K; ++i) { ip.sy[i] = sy[i]; ip.sx[i] = sx[i]; }
    }
    ip.t0y = (float)(mag * c.shifts[0]);
    ip.t0x = (float)(mag * c.shifts[1]);
    ip.perm = sp.perm = p->stream_path;
    ip.complete = p->complete;
    // streaming kernels on one GPU: per-CTA slots are reduced by every CTA of the next kernel instead of
    // by the last CTA of the producing one (no serial last-CTA tail)
    sp.deferred = p->stream_path && !pc && c.world == 1 && std::getenv("FLMISR_NO_DEFER") == nullptr;

    // ---- device memory ----
    auto cleanup_fail = [&](flmisr_status st) { flmisr_destroy(p); return st; };
    cudaError_t e = cudaSetDevice(c.device);
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
    e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(e)));
    p->hr_bytes = (size_t)srows * p->pitch * sizeof(float);
    const int nhr = 7;  // Y, X0, X1, P0, P1, R0, R1
    // + 4 padding rows: interior streaming warps may prefetch one row past the band's storage
    // (values only feed non-output rows), which must stay inside the allocation
    const size_t pad = (size_t)8 * p->pitch * sizeof(float);   // also covers the L2 prefetch distance
    e = cudaMalloc(&p->mem, p->hr_bytes * nhr + pad);
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, std::string("cudaMalloc HR buffers: ") + cudaGetErrorString(e)));
    cudaMemsetAsync(p->mem, 0, p->hr_bytes * nhr + pad, p->stream);
    const size_t fl = p->hr_bytes / sizeof(float);
    Buffers& b = p->b;
    b.Y = p->mem;
    b.X[0] = p->mem + 1 * fl; b.X[1] = p->mem + 2 * fl;
    b.P[0] = p->mem + 3 * fl; b.P[1] = p->mem + 4 * fl;
    b.R[0] = p->mem + 5 * fl; b.R[1] = p->mem + 6 * fl;
    const size_t nsblk = p->stream_path ? ((size_t)sp.nitems + sp.wpb - 1) / sp.wpb : 0;
    const long long nlr_px = (long long)K * c.lr_h * c.lr_w, nhr_px = (long long)p->H * p->W;
    int gcap = 148;
    cudaDeviceGetAttribute(&gcap, cudaDevAttrMultiProcessorCount, c.device);
    gcap *= 8;   // general path: grid-stride CTAs, 8 per SM
    const size_t ngblk = fast ? 0 : std::max<size_t>(std::max<size_t>(gen_blocks_lr(K, c.lr_h, c.lr_w, gcap),
                                                                       gen_blocks_hr(p->W, p->row_hi - p->row_lo, gcap)),
                                                     gen3_blocks(p->W, p->H, gcap));
    const size_t ntiles = std::max<size_t>(std::max<size_t>((size_t)sp.tiles_x * sp.tiles_y, nsblk), ngblk);
    // x2: the persistent loop kernel double-buffers its per-CTA slots by phase parity
    // det mode: FXW 128-bit words (2 doubles each) per CTA slot
    // (and the allgathered rank-sum records: RSW doubles per rank)
    // (and the loop kernels' three grid_sum accumulator sets of 6 NSLOT + 1 words)
    const size_t npart = std::max<size_t>(std::max<size_t>(std::max<size_t>(2 * NSLOT * ntiles, (size_t)RSW * world),
                                                            (size_t)2 * 2 * FXW * nsblk),
                                          (size_t)3 * (6 * NSLOT + 1) + 1);
    const size_t ntrace = (size_t)(c.n_iter + 1) * 6;
    const size_t nd = npart + RSW + ntrace + 1;   // + the grid-barrier counter
    e = cudaMalloc(&p->dmem, nd * sizeof(double));
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, std::string("cudaMalloc partials: ") + cudaGetErrorString(e)));
    cudaMemsetAsync(p->dmem, 0, nd * sizeof(double), p->stream);
    b.part = p->dmem;
    b.rank_sums = p->dmem + npart;   // RSW doubles: 16-byte aligned (npart is even)
    b.trace = p->dmem + npart + RSW;
    b.gbar = reinterpret_cast<unsigned*>(p->dmem + nd - 1);
    b.mem_lo = p->mem;
    b.mem_hi = p->mem + (p->hr_bytes * nhr + pad) / sizeof(float);
    {   // the whole SCG loop as one cooperative kernel (streaming path, one GPU):
        // removes the per-phase kernel boundary and reduction tail.  FLMISR_NO_PERSIST=1 falls back to
        // the per-phase kernels (deferred reduction), which bench.py uses for the per-kernel split.
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c.device);
        p->persist = p->stream_path && world == 1 && !virt && coop &&
                     (c.det_rows || std::getenv("FLMISR_NO_PERSIST") == nullptr);
        if (c.det_rows && world == 1 && !virt && !coop)
            return cleanup_fail(fail(FLMISR_ERR_CONFIG, "det_rows needs cooperative launch (the persistent loop kernel)"));
    }
    e = cudaMalloc(&p->st, sizeof(ScgState));
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, std::string("cudaMalloc state: ") + cudaGetErrorString(e)));
    cudaMemsetAsync(p->st, 0, sizeof(ScgState), p->stream);
    b.st = p->st;
    e = cudaEventCreateWithFlags(&p->done_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, "cudaEventCreate"));
    e = cudaMallocHost(&p->st_host, sizeof(ScgState));
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, "cudaMallocHost state"));
    e = cudaMallocHost(&p->trace_host, ntrace * sizeof(double));
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, "cudaMallocHost trace"));
    b.eta = p->eta;
    b.halo_top = b.halo_bot = nullptr;
    b.send_top = b.send_bot = nullptr;

    // ---- general-geometry path: per-frame taps and phases, LR copy, rho' weights (flmisr_general.cu) ----
    if (!fast) {
        GenParams& gp = p->gp;
        gp.k = K; gp.lr_h = c.lr_h; gp.lr_w = c.lr_w; gp.mag = mag;
        gp.R = R; gp.kd = 2 * R + 2;
        gp.nblk_lr = (int)gen_blocks_lr(K, c.lr_h, c.lr_w, gcap);
        gp.nblk_hr = (int)gen_blocks_hr(p->W, p->row_hi - p->row_lo, gcap);
        gp.fy_lo = 0; gp.fx_lo = 0; gp.fy_hi = p->H - 1; gp.fx_hi = p->W - 1;
        const size_t ntap = (size_t)K * gp.kd * gp.kd;
        std::vector<float> taps(ntap);
        for (int i = 0; i < K; ++i) {
            std::vector<double> kap;
            double fy, fx;
            int syi, sxi;
            composed_taps(c, i, kap, syi, sxi, fy, fx);
            for (size_t j = 0; j < kap.size(); ++j) taps[(size_t)i * gp.kd * gp.kd + j] = (float)kap[j];
            gp.sy[i] = syi; gp.sx[i] = sxi;
            gp.integer_phase[i] = (fy == 0.0 && fx == 0.0);
            gp.fy_lo = std::min(gp.fy_lo, syi - R);
            gp.fx_lo = std::min(gp.fx_lo, sxi - R);
            gp.fy_hi = std::max(gp.fy_hi, mag * (c.lr_h - 1) + syi + R + 1);
            gp.fx_hi = std::max(gp.fx_hi, mag * (c.lr_w - 1) + sxi + R + 1);
        }
        gp.noff = 0;   // BTV offset list: quadrant or Farsiu's set (NEXT-4)
        for (int dy = 0; dy < c.btv_window; ++dy)
            for (int dx = c.btv_offsets ? -(c.btv_window - 1) : 0; dx < c.btv_window; ++dx) {
                if ((dy == 0 && dx == 0) || (c.btv_offsets && dx + dy < 0)) continue;
                gp.offy[gp.noff] = dy;
                gp.offx[gp.noff] = dx;
                gp.ogam[gp.noff] = (float)std::pow(c.btv_alpha, std::abs(dx) + dy);
                ++gp.noff;
            }
        // fused tiled kernels (flmisr_general.cu, k_gen3_*): every integer phase in [-(R+1), mag-1+R] on
        // both axes keeps each tile's LR windows and their clamp folds inside the staged halo
        {
            bool ok = gen3_smem(R, mag, K) <= (size_t)200 * 1024 && std::getenv("FLMISR_GEN2") == nullptr;
            for (int i = 0; i < K; ++i)
                ok = ok && gp.sy[i] >= -(R + 1) && gp.sy[i] <= mag - 1 + R && gp.sx[i] >= -(R + 1) &&
                     gp.sx[i] <= mag - 1 + R;
            gp.fused = ok ? 1 : 0;
            gp.btvq = (c.btv_offsets == 0 && c.btv_window == 3) ? 3 : 0;
            if (gp.fused) {   // hoisted constants of the fused kernels (as on the streaming path)
                const double eps = c.l1_eps;
                double npairs_g = 0.0;   // sum over the offset list of gamma_d (as fp32) x valid pairs
                for (int o = 0; o < gp.noff; ++o)
                    npairs_g += (double)gp.ogam[o] * (double)std::max(0, p->H - gp.offy[o]) *
                                (double)std::max(0, p->W - std::abs(gp.offx[o]));
                sp.aff_vg[NSLOT + 0] = c.p_norm == 1 ? -eps * (double)K * c.lr_h * c.lr_w : 0.0;
                sp.aff_vg[NSLOT + 1] = -eps * npairs_g;
                if (c.curv_mode != 1) {   // the FD mode's update pass is a flmisr_general.cu kernel
                    sp.aff_uc[0] = c.p_norm == 1 ? eps * eps : 2.0;
                    sp.aff_uc[1] = eps * eps;
                }
            }
            gp.nblk3 = (int)gen3_blocks(p->W, p->H, gcap);
        }
        gp.fd = c.curv_mode == 1;
        gp.sigma0 = c.scg_sigma0;
        const size_t gbytes = ntap * sizeof(float) + 2 * (size_t)nlr_px * sizeof(float) +
                              (gp.fd ? (size_t)nlr_px * sizeof(double) + sizeof(double) : 0);
        e = cudaMalloc(&p->gmem, gbytes);
        if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, "cudaMalloc general-path buffers"));
        e = cudaMalloc(&p->gpart, (size_t)NSLOT * ngblk * sizeof(double));
        if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, "cudaMalloc general-path partials"));
        cudaMemcpyAsync(p->gmem, taps.data(), ntap * sizeof(float), cudaMemcpyHostToDevice, p->stream);
        gp.taps = p->gmem;
        gp.lr = p->gmem + ntap;
        gp.w = p->gmem + ntap + nlr_px;
        gp.wd = nullptr;
        if (gp.fd) {   // 8-byte aligned after the fp32 arrays
            const uintptr_t end = reinterpret_cast<uintptr_t>(p->gmem + ntap + 2 * nlr_px);
            gp.wd = reinterpret_cast<double*>((end + 7) / 8 * 8);
        }
        gp.part_a = p->gpart;
    }

    // ---- world > 1: halo buffers (inner-outer border exchange) and the NCCL communicator ----
    if (world > 1) {
        if (!p->stream_path)
            return cleanup_fail(fail(FLMISR_ERR_CONFIG, "row-band partitioning (world > 1) needs the streaming path: "
                                                        "separable PSF up to 3x3 with integer HR phases and W % 4 == 0"));
        const size_t hb = (size_t)p->eta * p->pitch * sizeof(float);
        float* hm = nullptr;
        // + 1 row: the bulk copies of a right-border strip read up to 512 B past a row's end
        e = cudaMalloc(&hm, 4 * hb + (size_t)p->pitch * sizeof(float));
        if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, "cudaMalloc halo buffers"));
        cudaMemsetAsync(hm, 0, 4 * hb + (size_t)p->pitch * sizeof(float), p->stream);
        p->halo_mem = hm;
        const size_t hf = hb / sizeof(float);
        if (rank > 0) { b.send_top = hm; p->recv_top = hm + 2 * hf; b.halo_top = p->recv_top; }
        if (rank < world - 1) { b.send_bot = hm + hf; p->recv_bot = hm + 3 * hf; b.halo_bot = p->recv_bot; }
        if (world > PMAX) return cleanup_fail(fail(FLMISR_ERR_CONFIG, "row bands: world <= 8"));
        e = cudaMalloc(&p->peer_mem, peer_mem_bytes(world));
        if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, "cudaMalloc peer mailbox"));
        cudaMemsetAsync(p->peer_mem, 0, peer_mem_bytes(world), p->stream);
        if (!virt) {
            NcclApi& api = nccl();
            if (!api.ok) return cleanup_fail(fail(FLMISR_ERR_NCCL, "libnccl.so.2 could not be loaded"));
            ncclUniqueId id;
            std::memcpy(&id, cfg->nccl_unique_id, sizeof(id));
            ncclResult_t r = api.CommInitRank(&p->comm, world, id, rank);
            if (r != ncclSuccess)
                return cleanup_fail(fail(FLMISR_ERR_NCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(r)));
        }
    }
    // the plan's own (non-blocking) stream, not a device-wide sync: another host thread may be capturing
    // a graph on its plan's stream meanwhile
    e = cudaStreamSynchronize(p->stream);
    if (e != cudaSuccess) return cleanup_fail(fail(FLMISR_ERR_CUDA, std::string("plan sync: ") + cudaGetErrorString(e)));
    *out = p;
    g_last_error.clear();
    return FLMISR_OK;
}

flmisr_status flmisr_plan(const flmisr_config* cfg, flmisr_plan_t* out) { return make_plan(cfg, out, false); }

flmisr_status flmisr_plan_virtual(const flmisr_config* cfg, flmisr_plan_t* out) { return make_plan(cfg, out, true); }

flmisr_status flmisr_band(int32_t H, int32_t world, int32_t rank, int32_t mag, int32_t* row_lo, int32_t* row_hi) {
    if (H < 1 || world < 1 || rank < 0 || rank >= world || mag < 1 || !row_lo || !row_hi)
        return fail(FLMISR_ERR_CONFIG, "flmisr_band: invalid arguments");
    *row_lo = (int32_t)(((long long)rank * H / world) / mag * mag);
    *row_hi = (rank == world - 1) ? H : (int32_t)(((long long)(rank + 1) * H / world) / mag * mag);
    return FLMISR_OK;
}

flmisr_status flmisr_nccl_unique_id(void* out128) {
    if (!out128) return fail(FLMISR_ERR_SHAPE, "out is NULL");
    NcclApi& api = nccl();
    if (!api.ok || !api.GetUniqueId) return fail(FLMISR_ERR_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    NCCL_TRY(api.GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return FLMISR_OK;
}

flmisr_status flmisr_plan_info(flmisr_plan_t p, int32_t* H, int32_t* W, int32_t* row_lo, int32_t* row_hi,
                               int32_t* fast_path, int32_t* loop_kernel) {
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    if (loop_kernel) *loop_kernel = p->persist;
    if (H) *H = p->H;
    if (W) *W = p->W;
    if (row_lo) *row_lo = p->row_lo;
    if (row_hi) *row_hi = p->row_hi;
    if (fast_path) *fast_path = p->pc ? 4 : p->fast ? (p->stream_path ? 2 : 1) : (p->gp.fused ? 3 : 0);
    return FLMISR_OK;
}

flmisr_status flmisr_destroy(flmisr_plan_t p) {
    if (!p) return FLMISR_OK;
    if (p->pipe) flmisr_pipeline_destroy(p->pipe);   // drains it; the pipeline cannot outlive its plan
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->comm && nccl().ok) nccl().CommDestroy(p->comm);
    for (void* m : p->ipc_open) cudaIpcCloseMemHandle(m);
    if (p->peer_mem) cudaFree(p->peer_mem);
    if (p->halo_mem) cudaFree(p->halo_mem);
    if (p->gmem) cudaFree(p->gmem);
    if (p->gpart) cudaFree(p->gpart);
    if (p->mem) cudaFree(p->mem);
    if (p->dmem) cudaFree(p->dmem);
    if (p->st) cudaFree(p->st);
    if (p->st_host) cudaFreeHost(p->st_host);
    if (p->trace_host) cudaFreeHost(p->trace_host);
    if (p->pin_in) cudaFreeHost(p->pin_in);
    if (p->pin_out) cudaFreeHost(p->pin_out);
    if (p->d_lr) cudaFree(p->d_lr);
    if (p->d_out) cudaFree(p->d_out);
    for (auto e : p->prof.ev) cudaEventDestroy(e);
    if (p->done_ev) cudaEventDestroy(p->done_ev);
    if (p->graph_exec) cudaGraphExecDestroy(p->graph_exec);
    if (p->virt_graph) cudaGraphExecDestroy(p->virt_graph);
    if (p->graph_exec_prof) cudaGraphExecDestroy(p->graph_exec_prof);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
    return FLMISR_OK;
}

}  // extern "C"

namespace {

// Multi-image interpolation fusion (reading 24) into dst (rows [0, H), pitch dpitch, layout dperm)
// for a world == 1 plan: the bilinear frame-0 estimate, then every integer-phase frame's LR pixels on
// their HR sites (first frame in index order wins), staged in the natural-layout scratch buffer.
flmisr_status enqueue_interp(flmisr_plan_s* p, const float* lr, float* dst, int dpitch, int dperm, float* scratch,
                             cudaStream_t s) {
    IngestParams ip0 = p->ip;
    ip0.perm = 0;
    StencilParams sp0 = p->sp;
    sp0.perm = 0;
    GenParams gi{};
    gi.k = p->cfg.k; gi.lr_h = p->cfg.lr_h; gi.lr_w = p->cfg.lr_w; gi.mag = p->cfg.mag;
    gi.lr = lr;
    for (int i = 0; i < p->cfg.k && i < GMAXK; ++i) {
        const double ty = p->cfg.mag * p->cfg.shifts[2 * i], tx = p->cfg.mag * p->cfg.shifts[2 * i + 1];
        gi.sy[i] = (int)std::floor(ty);
        gi.sx[i] = (int)std::floor(tx);
        gi.integer_phase[i] = ty == std::floor(ty) && tx == std::floor(tx);
    }
    CUDA_TRY(launch_init_x0(ip0, lr, scratch, s));
    CUDA_TRY(launch_gen_interp(sp0, gi, scratch, p->pitch, s));
    CUDA_TRY(launch_hr_copy(scratch, p->pitch, 0, dst, dpitch, dperm, p->H, p->W, s));
    return FLMISR_OK;
}

// a1 polyphase ingest, a2 initial estimate (or the caller's x0), p0 = 0, r_old = 0, SCG state.
flmisr_status enqueue_setup(flmisr_plan_s* p, const float* lr_stack, const float* x0, cudaStream_t s) {
    const Buffers& b = p->b;
    const int srows = p->store_hi - p->store_lo;
    if (p->fast) {
        CUDA_TRY(launch_ingest(p->ip, lr_stack, const_cast<float*>(b.Y), s));
    } else {   // general path: the kernels read the frames in their own layout from a plan-owned copy
        CUDA_TRY(cudaMemcpyAsync(const_cast<float*>(p->gp.lr), lr_stack,
                                 (size_t)p->cfg.k * p->cfg.lr_h * p->cfg.lr_w * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
    }
    bool p_zeroed = false;
    if (x0) {
        CUDA_TRY(launch_hr_copy(x0 + (size_t)p->store_lo * p->W, p->W, 0, b.X[0], p->pitch, p->sp.perm, srows, p->W, s));
    } else if (p->cfg.x0_mode == 1 && p->fast && p->all_int && p->complete) {
        // interpolation fusion on a polyphase-complete stack of integer phases is the ingested Y itself
        // (every HR site holds one LR pixel), band + halo rows, in the same buffer layout
        CUDA_TRY(cudaMemcpyAsync(b.X[0], b.Y, p->hr_bytes, cudaMemcpyDeviceToDevice, s));
    } else if (p->cfg.x0_mode == 1) {   // world 1 (plan check): staged through R[1], unused until the first pass
        flmisr_status st = enqueue_interp(p, lr_stack, b.X[0], p->pitch, p->sp.perm, b.R[1], s);
        if (st != FLMISR_OK) return st;
    } else {   // the permuted-layout x0 kernel writes p0 = 0 in the same pass
        CUDA_TRY(launch_init_x0(p->ip, lr_stack, b.X[0], s, b.P[0]));
        p_zeroed = init_x0_zeroes_p(p->ip);
    }
    if (!p_zeroed) CUDA_TRY(cudaMemsetAsync(b.P[0], 0, p->hr_bytes, s));
    // r_old = R[0] only enters the init pass's <r0, r_old>, which the scalar logic ignores; bands still
    // clear it (their halo logic reads rows of it before the first exchange)
    if (p->cfg.world > 1) CUDA_TRY(cudaMemsetAsync(b.R[0], 0, p->hr_bytes, s));
    CUDA_TRY(launch_state_init(b, p->cfg.scg_lambda0, p->cfg.lambda, p->cfg.n_iter, (long long)p->H * p->W,
                               p->cfg.scg_rules, s));
    return FLMISR_OK;
}

// Enqueue one value+gradient pass and, for world > 1, the consensus allgather + scalar kernel and
// the inner-outer border exchange of the r candidate.
cudaError_t launch_vg(flmisr_plan_s* p, int phase, cudaStream_t s) {
    if (!p->fast) return launch_gen_value_grad(p->bw, p->pn, p->sp, p->gp, p->b, phase, s);
    if (p->pc) return launch_pc_vg(p->bw, p->pn, p->sp, p->b, p->pct, phase, s);
    return p->stream_path ? launch_value_grad_stream(p->bw, p->pn, p->sp, p->b, phase, s)
                          : launch_value_grad(p->kr, p->bw, p->pn, p->sp, p->b, phase, s);
}

cudaError_t launch_uc(flmisr_plan_s* p, int phase, cudaStream_t s) {
    if (!p->fast) return launch_gen_update_curv(p->bw, p->pn, p->sp, p->gp, p->b, phase, s);
    if (p->pc) return launch_pc_uc(p->bw, p->pn, p->sp, p->b, p->pct, phase, s);
    return p->stream_path ? launch_update_curv_stream(p->bw, p->pn, p->sp, p->b, phase, s)
                          : launch_update_curv(p->kr, p->bw, p->pn, p->sp, p->b, phase, s);
}

flmisr_status enqueue_value_grad(flmisr_plan_s* p, int phase, cudaStream_t s) {
    CUDA_TRY(launch_vg(p, phase, s));
    if (p->cfg.world > 1 && !p->virt) {
        NcclApi& api = nccl();
        const int rank = p->cfg.rank, world = p->cfg.world;
        const size_t hcount = (size_t)p->eta * p->pitch;
        NCCL_TRY(api.GroupStart());
        NCCL_TRY(api.AllGather(p->b.rank_sums, p->b.part, p->sp.det ? RSW : NSLOT, ncclFloat64, p->comm, s));
        if (rank > 0) {
            NCCL_TRY(api.Send(p->b.send_top, hcount, ncclFloat32, rank - 1, p->comm, s));
            NCCL_TRY(api.Recv(p->recv_top, hcount, ncclFloat32, rank - 1, p->comm, s));
        }
        if (rank < world - 1) {
            NCCL_TRY(api.Send(p->b.send_bot, hcount, ncclFloat32, rank + 1, p->comm, s));
            NCCL_TRY(api.Recv(p->recv_bot, hcount, ncclFloat32, rank + 1, p->comm, s));
        }
        NCCL_TRY(api.GroupEnd());
        CUDA_TRY(launch_scalar_after_value(p->sp, p->b, world, phase, s));
    }
    return FLMISR_OK;
}

flmisr_status enqueue_update_curv(flmisr_plan_s* p, int phase, cudaStream_t s) {
    CUDA_TRY(launch_uc(p, phase, s));
    if (p->cfg.world > 1 && !p->virt) {
        NCCL_TRY(nccl().AllGather(p->b.rank_sums, p->b.part, p->sp.det ? RSW : NSLOT, ncclFloat64, p->comm, s));
        CUDA_TRY(launch_scalar_after_curv(p->sp, p->b, p->cfg.world, s));
    }
    return FLMISR_OK;
}

}  // namespace

extern "C" {

flmisr_status flmisr_reconstruct_async(flmisr_plan_t p, const float* lr_stack, const float* x0, float* hr_out,
                                       void* cuda_stream) {
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    if (!lr_stack) return fail(FLMISR_ERR_SHAPE, "lr_stack is NULL");
    if (!hr_out && (p->cfg.world == 1 || p->cfg.rank == 0)) return fail(FLMISR_ERR_SHAPE, "hr_out is NULL");
    if (p->cfg.world > 1 && !hr_out) return fail(FLMISR_ERR_SHAPE, "hr_out is required on every rank for the band gather");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : p->stream;
    p->last_stream = s;
    const Buffers& b = p->b;
    const size_t srows = (size_t)(p->store_hi - p->store_lo);
    Prof& pr = p->prof;
    const bool prof = pr.enabled;
    int ev = 0;
    auto mark = [&]() -> cudaError_t { return prof ? cudaEventRecord(pr.ev[ev++], s) : cudaSuccess; };

    // a1: polyphase ingest; a2: initial estimate, p0 = 0, r_old = 0, state
    CUDA_TRY(mark());
    {
        flmisr_status st0 = enqueue_setup(p, lr_stack, x0, s);
        if (st0 != FLMISR_OK) return st0;
    }
    (void)srows;
    (void)b;
    CUDA_TRY(mark());  // ev1: end of setup

    // init: f0 = J(x0), r0 = -grad J(x0) (Moller step 1), then n_iter SCG passes (Alg. 1 while-loop).
    // Single GPU without per-kernel profiling: the whole loop (plan-owned buffers only, all control on
    // the device) is one CUDA graph, captured on the first call and replayed into the caller's stream.
    flmisr_status st = FLMISR_OK;
    // the loop body; with profiling, event records between the kernels (captured as graph nodes)
    auto loop = [&](cudaStream_t ls, int ev0, bool captured) -> flmisr_status {
        int e = ev0;
        // external event nodes: inside a captured graph a plain record is only an internal dependency
        auto m = [&]() -> cudaError_t {
            if (!prof) return cudaSuccess;
            return captured ? cudaEventRecordWithFlags(pr.ev[e++], ls, cudaEventRecordExternal)
                            : cudaEventRecord(pr.ev[e++], ls);
        };
        flmisr_status r = enqueue_value_grad(p, PH_INIT, ls);
        if (r != FLMISR_OK) return r;
        CUDA_TRY(m());  // ev2
        for (int it = 0; it < p->cfg.n_iter; ++it) {
            if ((r = enqueue_update_curv(p, PH_ITER, ls)) != FLMISR_OK) return r;
            CUDA_TRY(m());
            if ((r = enqueue_value_grad(p, PH_ITER, ls)) != FLMISR_OK) return r;
            CUDA_TRY(m());
        }
        return FLMISR_OK;
    };
    bool looped = false;
    if (p->peer) {   // row bands over peer memory: the whole loop of this band as one cooperative kernel
        CUDA_TRY(launch_scg_peer_loop(p->bw, p->pn, p->sp, p->b_peer, p->pl, nullptr, s));
        looped = true;
        CUDA_TRY(mark());
        p->prof_mode = 1;
    }
    if (p->persist && !looped) {   // one cooperative kernel for the init pass and all n_iter passes
        cudaError_t le = p->pc ? launch_pc_loop(p->bw, p->pn, p->sp, p->b, p->pct, s)
                               : launch_scg_loop_stream(p->bw, p->pn, p->sp, p->b, s);
        if (le == cudaSuccess) {
            looped = true;
            CUDA_TRY(mark());   // ev2: end of the loop kernel
            p->prof_mode = 1;
        } else if ((le == cudaErrorCooperativeLaunchTooLarge || le == cudaErrorNotSupported) && !p->sp.det) {
            cudaGetLastError();   // not co-resident on this device / context: per-kernel launches instead
            p->persist = 0;
        } else {
            return fail(FLMISR_ERR_CUDA, std::string("persistent SCG loop launch: ") + cudaGetErrorString(le));
        }
    }
    if (!looped && p->sp.det && p->cfg.world == 1)   // det mode at world 1 is the persistent loop kernel
        return fail(FLMISR_ERR_CONFIG, "det_rows needs the persistent loop kernel (cooperative launch)");
    // world > 1 over NCCL: the per-phase kernels, the halo send/recv, the consensus allgather and the
    // scalar kernels are captured into the same graph (NCCL operations are graph-capturable; SURVEY
    // 8(e)); every rank captures the same operation sequence, so graph and eager ranks still match.
    const bool nccl_graph = p->cfg.world > 1 && !p->virt && std::getenv("FLMISR_NO_NCCL_GRAPH") == nullptr;
    const bool use_graph = !looped && !p->no_graph && (p->cfg.world == 1 || nccl_graph);
    bool graphed = false;
    if (looped) {
    } else if (use_graph) {
        cudaGraphExec_t& ge = prof ? p->graph_exec_prof : p->graph_exec;
        if (!ge) {
            cudaStream_t cs = p->stream;   // capture needs a non-legacy stream
            CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            st = loop(cs, ev, true);
            cudaGraph_t graph = nullptr;
            cudaError_t ce = cudaStreamEndCapture(cs, &graph);
            if (st == FLMISR_OK && ce == cudaSuccess) {
                ce = cudaGraphInstantiate(&ge, graph, 0);
                if (ce != cudaSuccess) ge = nullptr;
            }
            if (graph) cudaGraphDestroy(graph);
            if (p->cfg.world > 1 && (st != FLMISR_OK || ce != cudaSuccess)) {
                cudaGetLastError();   // the NCCL path could not be captured here: launch eagerly from now on
                p->no_graph = 1;
                st = FLMISR_OK;
            } else {
                if (st != FLMISR_OK) return st;
                if (ce != cudaSuccess) return fail(FLMISR_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
            }
        }
        if (ge) {
            CUDA_TRY(cudaGraphLaunch(ge, s));
            graphed = true;
        }
    }
    if (looped || graphed) {
    } else {
        st = loop(s, ev, false);
        if (st != FLMISR_OK) return st;
    }
    if (!looped) {
        p->prof_mode = 0;
        if (prof) ev += 1 + 2 * p->cfg.n_iter;
    }
    // deferred reduction: the last value+gradient kernel's scalar step is still pending
    if (p->sp.deferred && !looped) CUDA_TRY(launch_settle(p->sp, b, s));
    // a12: fuse (owned rows; rank 0 gathers the bands for world > 1)
    if (hr_out) CUDA_TRY(launch_finalize(p->sp, b, hr_out, p->W, p->row_lo, p->row_hi, s));
    if (p->cfg.world > 1) {
        NcclApi& api = nccl();
        const int rank = p->cfg.rank, world = p->cfg.world;
        if (rank == 0) {
            NCCL_TRY(api.GroupStart());
            for (int h = 1; h < world; ++h) {
                int lo = (int)(((long long)h * p->H / world) / p->cfg.mag * p->cfg.mag);
                int hi = (h == world - 1) ? p->H : (int)(((long long)(h + 1) * p->H / world) / p->cfg.mag * p->cfg.mag);
                NCCL_TRY(api.Recv(hr_out + (size_t)lo * p->W, (size_t)(hi - lo) * p->W, ncclFloat32, h, p->comm, s));
            }
            NCCL_TRY(api.GroupEnd());
        } else {
            NCCL_TRY(api.Send(hr_out + (size_t)p->row_lo * p->W, (size_t)(p->row_hi - p->row_lo) * p->W, ncclFloat32,
                              0, p->comm, s));
        }
    }
    CUDA_TRY(mark());  // last
    const size_t ntrace = (size_t)(p->cfg.n_iter + 1) * 6;
    CUDA_TRY(cudaMemcpyAsync(p->st_host, p->st, sizeof(ScgState), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(p->trace_host, p->b.trace, ntrace * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaEventRecord(p->done_ev, s));
    p->pending = 1;
    p->prof_marks = ev;
    return FLMISR_OK;
}

flmisr_status flmisr_finish(flmisr_plan_t p, flmisr_report* rep) {
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    if (!p->pending) return fail(FLMISR_ERR_SHAPE, "no reconstruction in flight");
    p->pending = 0;
    CUDA_TRY(cudaEventSynchronize(p->done_ev));
    const size_t ntrace = (size_t)(p->cfg.n_iter + 1) * 6;
    const ScgState& h = *p->st_host;
    if (rep) {
        rep->iters_run = h.k;
        rep->accepted = h.accepted;
        rep->converged_at = h.converged_at;
        rep->failed_stage = h.failed_stage;
        rep->failed_iter = h.failed_iter;
        if (rep->f_trace) std::memcpy(rep->f_trace, p->trace_host, ntrace * sizeof(double));
    }
    Prof& pr = p->prof;
    if (pr.enabled && p->prof_mode == 1 && p->prof_marks >= 4) {
        // marks: 0 start, 1 setup end, 2 loop kernel end, 3 last
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.ev[0], pr.ev[1]); pr.ms[2] += ms;
        cudaEventElapsedTime(&ms, pr.ev[1], pr.ev[2]); pr.ms[0] += ms; pr.n[0] += 1;
        cudaEventElapsedTime(&ms, pr.ev[2], pr.ev[3]); pr.ms[2] += ms;
        cudaEventElapsedTime(&ms, pr.ev[0], pr.ev[3]); pr.ms[3] += ms; pr.n[3] += 1;
        pr.n[2] += 1;
        cudaError_t pe = cudaGetLastError();
        if (pe != cudaSuccess) return fail(FLMISR_ERR_CUDA, std::string("profiling events: ") + cudaGetErrorString(pe));
    } else if (pr.enabled && p->prof_marks >= 4) {
        // marks: 0 start, 1 setup end, 2 init value/grad end, then (curv end, value end) per pass, last
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.ev[0], pr.ev[1]); pr.ms[2] += ms;
        cudaEventElapsedTime(&ms, pr.ev[1], pr.ev[2]); pr.ms[0] += ms; pr.n[0] += 1;
        int m = 2;
        for (int it = 0; it < p->cfg.n_iter; ++it) {
            cudaEventElapsedTime(&ms, pr.ev[m], pr.ev[m + 1]); pr.ms[1] += ms; pr.n[1] += 1;
            cudaEventElapsedTime(&ms, pr.ev[m + 1], pr.ev[m + 2]); pr.ms[0] += ms; pr.n[0] += 1;
            m += 2;
        }
        cudaEventElapsedTime(&ms, pr.ev[m], pr.ev[m + 1]); pr.ms[2] += ms;
        cudaEventElapsedTime(&ms, pr.ev[0], pr.ev[m + 1]); pr.ms[3] += ms; pr.n[3] += 1;
        pr.n[2] += 1;
        cudaError_t pe = cudaGetLastError();   // do not leave a timing error sticky for the next launch
        if (pe != cudaSuccess) return fail(FLMISR_ERR_CUDA, std::string("profiling events: ") + cudaGetErrorString(pe));
    }
    if (h.failed_stage) return failed_status(h, "reconstruct");
    return FLMISR_OK;
}

flmisr_status flmisr_reconstruct(flmisr_plan_t p, const float* lr_stack, const float* x0, float* hr_out,
                                 void* cuda_stream, flmisr_report* report) {
    flmisr_status st = flmisr_reconstruct_async(p, lr_stack, x0, hr_out, cuda_stream);
    if (st != FLMISR_OK) return st;
    return flmisr_finish(p, report);
}

flmisr_status flmisr_profile(flmisr_plan_t p, int32_t enable, double* out8) {
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    Prof& pr = p->prof;
    if (out8) {
        for (int i = 0; i < 4; ++i) { out8[2 * i] = (double)pr.n[i]; out8[2 * i + 1] = pr.ms[i]; }
    }
    if (enable >= 0) {
        for (int i = 0; i < 4; ++i) { pr.n[i] = 0; pr.ms[i] = 0.0; }
        if (enable && pr.ev.empty()) {
            pr.ev.resize((size_t)2 * p->cfg.n_iter + 8);
            for (auto& e : pr.ev) CUDA_TRY(cudaEventCreate(&e));
        }
        pr.enabled = enable != 0;
    }
    return FLMISR_OK;
}

// In-process virtual group: the g row bands of one reconstruction, each with its own plan (own
// buffers, halos, state), run on ONE device and stream in Algorithm 1's order; the NCCL collectives
// are replaced by device-to-device copies (allgather of the rank sums, halo rows to the neighbours).
// Exercises every band-mode kernel path on a single GPU (the multi-GPU run differs only in transport).
flmisr_status flmisr_reconstruct_virtual(flmisr_plan_t* plans, int32_t g, const float* lr_stack, const float* x0,
                                         float* hr_out, flmisr_report* report) {
    if (!plans || g < 2) return fail(FLMISR_ERR_SHAPE, "virtual group needs g >= 2 plans");
    if (!lr_stack || !hr_out) return fail(FLMISR_ERR_SHAPE, "lr_stack and hr_out are required");
    for (int h = 0; h < g; ++h) {
        flmisr_plan_s* q = plans[h];
        if (!q || !q->virt || q->cfg.world != g || q->cfg.rank != h || q->H != plans[0]->H || q->W != plans[0]->W ||
            q->cfg.n_iter != plans[0]->cfg.n_iter || q->cfg.device != plans[0]->cfg.device)
            return fail(FLMISR_ERR_SHAPE, "plans must be flmisr_plan_virtual bands 0..g-1 of one configuration");
        if (q->cfg.det_rows != plans[0]->cfg.det_rows)
            return fail(FLMISR_ERR_SHAPE, "plans must be flmisr_plan_virtual bands 0..g-1 of one configuration");
    }
    CUDA_TRY(cudaSetDevice(plans[0]->cfg.device));
    cudaStream_t s = plans[0]->stream;
    const size_t hb = (size_t)plans[0]->eta * plans[0]->pitch * sizeof(float);
    const size_t rec = plans[0]->sp.det ? RSW : NSLOT;   // doubles per rank-sum record
    auto gather = [&]() -> flmisr_status {
        for (int h = 0; h < g; ++h)
            for (int r = 0; r < g; ++r)
                CUDA_TRY(cudaMemcpyAsync(plans[h]->b.part + (size_t)r * rec, plans[r]->b.rank_sums,
                                         rec * sizeof(double), cudaMemcpyDeviceToDevice, s));
        return FLMISR_OK;
    };
    auto exchange = [&]() -> flmisr_status {
        for (int h = 0; h < g; ++h) {
            if (h > 0)
                CUDA_TRY(cudaMemcpyAsync(plans[h]->recv_top, plans[h - 1]->b.send_bot, hb, cudaMemcpyDeviceToDevice, s));
            if (h < g - 1)
                CUDA_TRY(cudaMemcpyAsync(plans[h]->recv_bot, plans[h + 1]->b.send_top, hb, cudaMemcpyDeviceToDevice, s));
        }
        return FLMISR_OK;
    };
    flmisr_status st;
    for (int h = 0; h < g; ++h)
        if ((st = enqueue_setup(plans[h], lr_stack, x0, s)) != FLMISR_OK) return st;
    auto value_grad = [&](int phase) -> flmisr_status {
        flmisr_status r;
        for (int h = 0; h < g; ++h)
            if ((r = enqueue_value_grad(plans[h], phase, s)) != FLMISR_OK) return r;
        if ((r = gather()) != FLMISR_OK || (r = exchange()) != FLMISR_OK) return r;
        for (int h = 0; h < g; ++h) CUDA_TRY(launch_scalar_after_value(plans[h]->sp, plans[h]->b, g, phase, s));
        return FLMISR_OK;
    };
    auto update_curv = [&]() -> flmisr_status {
        flmisr_status r;
        for (int h = 0; h < g; ++h)
            if ((r = enqueue_update_curv(plans[h], PH_ITER, s)) != FLMISR_OK) return r;
        if ((r = gather()) != FLMISR_OK) return r;
        for (int h = 0; h < g; ++h) CUDA_TRY(launch_scalar_after_curv(plans[h]->sp, plans[h]->b, g, s));
        return FLMISR_OK;
    };
    auto body = [&]() -> flmisr_status {
        flmisr_status r;
        if ((r = value_grad(PH_INIT)) != FLMISR_OK) return r;
        for (int it = 0; it < plans[0]->cfg.n_iter; ++it) {
            if ((r = update_curv()) != FLMISR_OK) return r;
            if ((r = value_grad(PH_ITER)) != FLMISR_OK) return r;
        }
        return FLMISR_OK;
    };
    // the loop of all bands (kernels, the copies standing in for the NCCL allgather and halo
    // send/recv, the scalar kernels) as one CUDA graph, captured once per band set (as on one GPU)
    flmisr_plan_s* p0 = plans[0];
    std::vector<const void*> key;
    for (int h = 0; h < g; ++h) { key.push_back(plans[h]); key.push_back(plans[h]->mem); }
    if (p0->no_graph) {
        if ((st = body()) != FLMISR_OK) return st;
    } else {
        if (!p0->virt_graph || p0->virt_key != key) {
            if (p0->virt_graph) cudaGraphExecDestroy(p0->virt_graph);
            p0->virt_graph = nullptr;
            CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            st = body();
            cudaGraph_t graph = nullptr;
            cudaError_t ce = cudaStreamEndCapture(s, &graph);
            if (st == FLMISR_OK && ce == cudaSuccess) ce = cudaGraphInstantiate(&p0->virt_graph, graph, 0);
            if (graph) cudaGraphDestroy(graph);
            if (st != FLMISR_OK) return st;
            if (ce != cudaSuccess) return fail(FLMISR_ERR_CUDA, std::string("virtual group graph: ") + cudaGetErrorString(ce));
            p0->virt_key = key;
        }
        CUDA_TRY(cudaGraphLaunch(p0->virt_graph, s));
    }
    for (int h = 0; h < g; ++h)
        CUDA_TRY(launch_finalize(plans[h]->sp, plans[h]->b, hr_out, plans[h]->W, plans[h]->row_lo, plans[h]->row_hi, s));
    // every band holds the same consensus scalars; report band 0 and check the others agree
    const size_t ntrace = (size_t)(plans[0]->cfg.n_iter + 1) * 6;
    for (int h = 0; h < g; ++h) {
        CUDA_TRY(cudaMemcpyAsync(plans[h]->st_host, plans[h]->st, sizeof(ScgState), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(plans[h]->trace_host, plans[h]->b.trace, ntrace * sizeof(double), cudaMemcpyDeviceToHost,
                                 s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int h = 1; h < g; ++h)
        if (std::memcmp(plans[h]->trace_host, plans[0]->trace_host, ntrace * sizeof(double)) != 0 ||
            plans[h]->st_host->k != plans[0]->st_host->k)
            return fail(FLMISR_ERR_NUMERIC, "virtual group: bands disagree on the consensus trace");
    const ScgState& hs = *plans[0]->st_host;
    if (report) {
        report->iters_run = hs.k;
        report->accepted = hs.accepted;
        report->converged_at = hs.converged_at;
        report->failed_stage = hs.failed_stage;
        report->failed_iter = hs.failed_iter;
        if (report->f_trace) std::memcpy(report->f_trace, plans[0]->trace_host, ntrace * sizeof(double));
    }
    if (hs.failed_stage) return failed_status(hs, "virtual group");
    return FLMISR_OK;
}

// PeerLoop of one band (g = 1) or of all bands of a virtual group (g = world, one device); mbox /
// flags of rank q at the given (local or peer-mapped) peer_mem base
static void peer_fill(PeerLoop& pl, int world, unsigned char* const* mem_of_rank) {
    for (int q = 0; q < world; ++q) {
        pl.mbox[q] = peer_mbox(mem_of_rank[q]);
        pl.cnt[q] = peer_cnt(mem_of_rank[q]);
    }
    // a phase takes well under a millisecond: 20 s without every arrival means a lost rank or CTA
    // (FLMISR_PEER_TIMEOUT_MS overrides; tests use a short one)
    pl.timeout_ns = 20000000000ull;
    if (const char* ev = std::getenv("FLMISR_PEER_TIMEOUT_MS")) pl.timeout_ns = (unsigned long long)std::atoll(ev) * 1000000ull;
    pl.drop_band = -1;
    if (const char* ev = std::getenv("FLMISR_PEER_TEST_DROP")) pl.drop_band = std::atoi(ev);
}
static int peer_ctas(const flmisr_plan_s* p) { return (p->sp.loop_warps + SWPB - 1) / SWPB; }

// The g row bands of one reconstruction on ONE device, synchronised through the peer-loop protocol
// (mailboxes, flags, halo rows stored into the neighbours' buffers) in one cooperative launch of
// g x ctas CTAs -- the multi-GPU kernel with local pointers in place of the peer mappings.
flmisr_status flmisr_reconstruct_virtual_peer(flmisr_plan_t* plans, int32_t g, const float* lr_stack,
                                              const float* x0, float* hr_out, flmisr_report* report) {
    if (!plans || g < 2 || g > PMAX) return fail(FLMISR_ERR_SHAPE, "virtual peer group needs 2 <= g <= 8 plans");
    if (!lr_stack || !hr_out) return fail(FLMISR_ERR_SHAPE, "lr_stack and hr_out are required");
    int ctas = 0;
    for (int h = 0; h < g; ++h) {
        flmisr_plan_s* q = plans[h];
        if (!q || !q->virt || q->cfg.world != g || q->cfg.rank != h || q->H != plans[0]->H || q->W != plans[0]->W ||
            q->cfg.n_iter != plans[0]->cfg.n_iter || q->cfg.device != plans[0]->cfg.device || !q->stream_path ||
            q->cfg.det_rows != plans[0]->cfg.det_rows)
            return fail(FLMISR_ERR_SHAPE, "plans must be flmisr_plan_virtual streaming bands 0..g-1 of one configuration");
        ctas = std::max(ctas, peer_ctas(q));
    }
    CUDA_TRY(cudaSetDevice(plans[0]->cfg.device));
    int nsm = 0, coop = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, plans[0]->cfg.device));
    CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, plans[0]->cfg.device));
    if (!coop || g * ctas > nsm || ctas > PEER_MAXCTAS)
        return fail(FLMISR_ERR_CONFIG, "virtual peer group does not fit one cooperative wave");
    cudaStream_t s = plans[0]->stream;
    flmisr_status st;
    for (int h = 0; h < g; ++h)
        if ((st = enqueue_setup(plans[h], lr_stack, x0, s)) != FLMISR_OK) return st;
    auto* pb = new PeerBands();   // ~6 KB: kernel-parameter space, not the host stack
    std::vector<unsigned char*> mems(g);
    PeerLoop pl{};
    pl.g = g; pl.rank0 = 0; pl.world = g; pl.ctas = ctas;
    for (int h = 0; h < g; ++h) {
        pb->sp[h] = plans[h]->sp;
        pb->b[h] = plans[h]->b;
        pb->b[h].send_top = h > 0 ? plans[h - 1]->recv_bot : nullptr;       // straight into the neighbours' halos
        pb->b[h].send_bot = h < g - 1 ? plans[h + 1]->recv_top : nullptr;
        mems[h] = plans[h]->peer_mem;
        pl.epoch_word[h] = peer_epoch(mems[h]);
    }
    peer_fill(pl, g, mems.data());
    cudaError_t le = launch_scg_peer_loop(plans[0]->bw, plans[0]->pn, plans[0]->sp, plans[0]->b, pl, pb, s);
    delete pb;
    if (le != cudaSuccess) return fail(FLMISR_ERR_CUDA, std::string("peer loop launch: ") + cudaGetErrorString(le));
    for (int h = 0; h < g; ++h)
        CUDA_TRY(launch_finalize(plans[h]->sp, plans[h]->b, hr_out, plans[h]->W, plans[h]->row_lo, plans[h]->row_hi, s));
    const size_t ntrace = (size_t)(plans[0]->cfg.n_iter + 1) * 6;
    for (int h = 0; h < g; ++h) {
        CUDA_TRY(cudaMemcpyAsync(plans[h]->st_host, plans[h]->st, sizeof(ScgState), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(plans[h]->trace_host, plans[h]->b.trace, ntrace * sizeof(double), cudaMemcpyDeviceToHost,
                                 s));
    }
    cudaError_t se = cudaStreamSynchronize(s);
    if (se != cudaSuccess) return fail(FLMISR_ERR_CUDA, std::string("virtual peer group: ") + cudaGetErrorString(se));
    for (int h = 0; h < g; ++h)   // a band that abandoned the loop (barrier timeout) reports first
        if (plans[h]->st_host->failed_stage == FAIL_PEER_TIMEOUT) return failed_status(*plans[h]->st_host, "virtual peer group");
    for (int h = 1; h < g; ++h)
        if (std::memcmp(plans[h]->trace_host, plans[0]->trace_host, ntrace * sizeof(double)) != 0 ||
            plans[h]->st_host->k != plans[0]->st_host->k)
            return fail(FLMISR_ERR_NUMERIC, "virtual peer group: bands disagree on the consensus trace");
    const ScgState& hs = *plans[0]->st_host;
    if (report) {
        report->iters_run = hs.k;
        report->accepted = hs.accepted;
        report->converged_at = hs.converged_at;
        report->failed_stage = hs.failed_stage;
        report->failed_iter = hs.failed_iter;
        if (report->f_trace) std::memcpy(report->f_trace, plans[0]->trace_host, ntrace * sizeof(double));
    }
    if (hs.failed_stage) return failed_status(hs, "virtual group");
    return FLMISR_OK;
}

// What a rank publishes for its peers: IPC handles of its halo buffers and of its mailbox block, and
// where its receive rows sit in the halo allocation.
// The geometry fields and the configuration digest let every rank reject a peer that planned a
// different problem (it would wait on barrier epochs that never come); the PCI bus id lets it check
// that the peer device supports native peer atomics (the system-scope arrival counters).
struct PeerBlob {
    uint32_t magic, rank, world, ctas;
    cudaIpcMemHandle_t halo, mbox;
    uint64_t recv_top_off, recv_bot_off;
    uint32_t H, W, n_iter, eta, pitch, pad;
    uint64_t cfg_digest;
    char pci[32];
};
static_assert(sizeof(PeerBlob) <= FLMISR_PEER_BLOB_BYTES, "peer blob size");

// FNV-1a over every numeric configuration field that shapes the SCG trajectory
static uint64_t cfg_digest(const flmisr_config& c) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* d, size_t n) {
        for (size_t i = 0; i < n; ++i) { h ^= ((const unsigned char*)d)[i]; h *= 1099511628211ull; }
    };
    const int32_t iv[] = {c.k, c.lr_h, c.lr_w, c.psf_h, c.psf_w, c.mag, c.p_norm, c.btv_window, c.n_iter,
                          c.btv_offsets, c.curv_mode, c.scg_rules, c.x0_mode, c.det_rows};
    const double dv[] = {c.l1_eps, c.lambda, c.btv_alpha, c.scg_sigma0, c.scg_lambda0};
    mix(iv, sizeof(iv));
    mix(dv, sizeof(dv));
    mix(c.shifts, sizeof(double) * 2 * (size_t)c.k);
    mix(c.psf, sizeof(double) * (size_t)c.psf_h * c.psf_w);
    return h;
}

flmisr_status flmisr_peer_export(flmisr_plan_t p, void* out) {
    if (!p || !out) return fail(FLMISR_ERR_SHAPE, "plan and out are required");
    if (p->cfg.world < 2 || p->virt || !p->peer_mem) return fail(FLMISR_ERR_CONFIG, "peer export needs a band plan (world > 1)");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    PeerBlob bl{};
    bl.magic = 0x464c4d50u;   // "FLMP"
    bl.rank = (uint32_t)p->cfg.rank;
    bl.world = (uint32_t)p->cfg.world;
    bl.ctas = (uint32_t)peer_ctas(p);
    CUDA_TRY(cudaIpcGetMemHandle(&bl.halo, p->halo_mem));
    CUDA_TRY(cudaIpcGetMemHandle(&bl.mbox, p->peer_mem));
    bl.recv_top_off = p->recv_top ? (uint64_t)((char*)p->recv_top - (char*)p->halo_mem) : 0;
    bl.recv_bot_off = p->recv_bot ? (uint64_t)((char*)p->recv_bot - (char*)p->halo_mem) : 0;
    bl.H = (uint32_t)p->H; bl.W = (uint32_t)p->W; bl.n_iter = (uint32_t)p->cfg.n_iter;
    bl.eta = (uint32_t)p->eta; bl.pitch = (uint32_t)p->pitch;
    bl.cfg_digest = cfg_digest(p->cfg);
    CUDA_TRY(cudaDeviceGetPCIBusId(bl.pci, (int)sizeof(bl.pci), p->cfg.device));
    std::memset(out, 0, FLMISR_PEER_BLOB_BYTES);
    std::memcpy(out, &bl, sizeof(bl));
    return FLMISR_OK;
}

flmisr_status flmisr_peer_connect(flmisr_plan_t p, const void* blobs) {
    if (!p || !blobs) return fail(FLMISR_ERR_SHAPE, "plan and blobs are required");
    const int world = p->cfg.world, rank = p->cfg.rank;
    if (world < 2 || p->virt || !p->peer_mem || !p->stream_path) return fail(FLMISR_ERR_CONFIG, "peer connect needs a streaming band plan (world > 1)");
    if (p->peer) return fail(FLMISR_ERR_CONFIG, "plan already connected");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    std::vector<unsigned char*> mems(world, nullptr);
    std::vector<char*> halos(world, nullptr);
    std::vector<PeerBlob> bl(world);
    for (int q = 0; q < world; ++q) {
        std::memcpy(&bl[q], (const char*)blobs + (size_t)q * FLMISR_PEER_BLOB_BYTES, sizeof(PeerBlob));
        if (bl[q].magic != 0x464c4d50u || (int)bl[q].rank != q || (int)bl[q].world != world)
            return fail(FLMISR_ERR_CONFIG, "peer blobs must be the world ranks' flmisr_peer_export outputs in rank order");
        if ((int)bl[q].H != p->H || (int)bl[q].W != p->W || (int)bl[q].n_iter != p->cfg.n_iter ||
            (int)bl[q].eta != p->eta || (int)bl[q].pitch != p->pitch || bl[q].cfg_digest != cfg_digest(p->cfg))
            return fail(FLMISR_ERR_CONFIG, "peer rank " + std::to_string(q) +
                                               " planned a different problem (geometry, n_iter or parameters differ)");
    }
    // the arrival counters are system-scope atomics on peer memory: every peer device must be
    // reachable with native peer atomics (NVLink); a peer whose PCI id this process cannot resolve
    // (not visible here) is accepted on the IPC mapping alone
    for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        int pd = -1;
        bl[q].pci[sizeof(bl[q].pci) - 1] = 0;
        if (cudaDeviceGetByPCIBusId(&pd, bl[q].pci) != cudaSuccess) { cudaGetLastError(); continue; }
        if (pd == p->cfg.device) return fail(FLMISR_ERR_CONFIG, "two ranks share one device");
        int acc = 0, atom = 0;
        CUDA_TRY(cudaDeviceGetP2PAttribute(&acc, cudaDevP2PAttrAccessSupported, p->cfg.device, pd));
        CUDA_TRY(cudaDeviceGetP2PAttribute(&atom, cudaDevP2PAttrNativeAtomicSupported, p->cfg.device, pd));
        if (!acc || !atom)
            return fail(FLMISR_ERR_CONFIG, "peer device " + std::string(bl[q].pci) +
                                               " lacks peer access or native peer atomics; use the NCCL transport");
    }
    for (int q = 0; q < world; ++q) {
        if (q == rank) {
            mems[q] = p->peer_mem;
            halos[q] = (char*)p->halo_mem;
            continue;
        }
        void* m = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&m, bl[q].mbox, cudaIpcMemLazyEnablePeerAccess));
        p->ipc_open.push_back(m);
        mems[q] = (unsigned char*)m;
        if (q == rank - 1 || q == rank + 1) {   // the neighbours' halo buffers receive our boundary rows
            void* hmap = nullptr;
            CUDA_TRY(cudaIpcOpenMemHandle(&hmap, bl[q].halo, cudaIpcMemLazyEnablePeerAccess));
            p->ipc_open.push_back(hmap);
            halos[q] = (char*)hmap;
        }
    }
    PeerLoop& pl = p->pl;
    pl = PeerLoop{};
    pl.g = 1; pl.rank0 = rank; pl.world = world;
    pl.ctas = 0;   // the same on every rank: the largest band's (smaller bands idle their extra CTAs)
    for (int q = 0; q < world; ++q) pl.ctas = std::max(pl.ctas, (int)bl[q].ctas);
    peer_fill(pl, world, mems.data());
    pl.epoch_word[0] = peer_epoch(p->peer_mem);
    p->b_peer = p->b;
    p->b_peer.send_top = rank > 0 ? (float*)(halos[rank - 1] + bl[rank - 1].recv_bot_off) : nullptr;
    p->b_peer.send_bot = rank < world - 1 ? (float*)(halos[rank + 1] + bl[rank + 1].recv_top_off) : nullptr;
    int coop = 0, nsm = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, p->cfg.device));
    CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->cfg.device));
    if (!coop || pl.ctas > nsm || pl.ctas > PEER_MAXCTAS)
        return fail(FLMISR_ERR_CONFIG, "peer loop needs a cooperative launch of one wave");
    p->peer = 1;
    return FLMISR_OK;
}

flmisr_status flmisr_reconstruct_host(flmisr_plan_t p, const float* lr_host, float* hr_host, flmisr_report* report) {
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    if (!lr_host) return fail(FLMISR_ERR_SHAPE, "lr_stack_host is NULL");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    const size_t nlr = (size_t)p->cfg.k * p->cfg.lr_h * p->cfg.lr_w;
    const size_t nhr = (size_t)p->H * p->W;
    if (!p->d_lr) {
        CUDA_TRY(cudaMalloc(&p->d_lr, nlr * sizeof(float)));
        CUDA_TRY(cudaMalloc(&p->d_out, nhr * sizeof(float)));
    }
    // page-locked caller buffers are DMA'd directly; pageable ones are staged through pinned memory
    auto pinned = [](const void* ptr) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) { cudaGetLastError(); return false; }
        return a.type == cudaMemoryTypeHost;
    };
    const float* src = lr_host;
    if (!pinned(lr_host)) {
        if (!p->pin_in) CUDA_TRY(cudaMallocHost(&p->pin_in, nlr * sizeof(float)));
        std::memcpy(p->pin_in, lr_host, nlr * sizeof(float));
        src = p->pin_in;
    }
    CUDA_TRY(cudaMemcpyAsync(p->d_lr, src, nlr * sizeof(float), cudaMemcpyHostToDevice, p->stream));
    flmisr_status st = flmisr_reconstruct_async(p, p->d_lr, nullptr, p->d_out, p->stream);
    if (st != FLMISR_OK) return st;
    const bool root = p->cfg.world == 1 || p->cfg.rank == 0;
    float* dst = hr_host;
    const bool direct = hr_host && pinned(hr_host);
    if (hr_host && root) {
        if (!direct && !p->pin_out) CUDA_TRY(cudaMallocHost(&p->pin_out, nhr * sizeof(float)));
        dst = direct ? hr_host : p->pin_out;
        CUDA_TRY(cudaMemcpyAsync(dst, p->d_out, nhr * sizeof(float), cudaMemcpyDeviceToHost, p->stream));
        CUDA_TRY(cudaEventRecord(p->done_ev, p->stream));
    }
    st = flmisr_finish(p, report);
    if (hr_host && root && !direct) std::memcpy(hr_host, p->pin_out, nhr * sizeof(float));
    return st;
}

flmisr_status flmisr_interp_fuse(flmisr_plan_t p, const float* lr, float* out, void* cuda_stream) {
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    if (!lr || !out) return fail(FLMISR_ERR_SHAPE, "lr_stack and hr_out are required");
    if (p->cfg.world != 1) return fail(FLMISR_ERR_CONFIG, "flmisr_interp_fuse needs a world == 1 plan");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : p->stream;
    const Buffers& b = p->b;
    IngestParams ip0 = p->ip;
    ip0.perm = 0;
    if (p->fast && p->all_int && p->complete) {   // polyphase-complete, integer phases: one LR pixel per HR site
        CUDA_TRY(launch_ingest(ip0, lr, b.R[0], s));
        CUDA_TRY(launch_hr_copy(b.R[0], p->pitch, 0, out, p->W, 0, p->H, p->W, s));
        return FLMISR_OK;
    }
    return enqueue_interp(p, lr, out, p->W, 0, b.R[0], s);
}

flmisr_status flmisr_debug_apply(flmisr_plan_t p, int32_t op, const float* lr, const float* in0, const float* in1,
                                 float* out, double* sc) {
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    if (p->cfg.world != 1) return fail(FLMISR_ERR_CONFIG, "debug entries need world == 1");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    cudaStream_t s = p->stream;
    Buffers& b = p->b;
    const int H = p->H, perm = p->sp.perm;
    // HR copies between the caller's natural layout and the plan's buffer layout (perm: streaming path)
    auto put_hr = [&](float* dst, const float* src) {
        return launch_hr_copy(src, p->W, 0, dst, p->pitch, perm, H, p->W, s);
    };
    auto get_hr = [&](float* dst, const float* src) {
        return launch_hr_copy(src, p->pitch, perm, dst, p->W, 0, H, p->W, s);
    };
    // FORWARD / ADJOINT run the tap-by-tap debug stencils on natural-layout scratch
    IngestParams ip0 = p->ip;
    ip0.perm = 0;
    StencilParams sp0 = p->sp;
    sp0.perm = 0;
    CUDA_TRY(launch_state_init(b, p->cfg.scg_lambda0, p->cfg.lambda, p->cfg.n_iter, (long long)p->H * p->W,
                               p->cfg.scg_rules, s));
    const bool gen = !p->fast;
    const size_t lr_bytes = (size_t)p->cfg.k * p->cfg.lr_h * p->cfg.lr_w * sizeof(float);
    // the LR stack in the layout the data-term kernels read (polyphase Y, or the general path's copy)
    auto put_lr = [&](const float* src) -> cudaError_t {
        return gen ? cudaMemcpyAsync(const_cast<float*>(p->gp.lr), src, lr_bytes, cudaMemcpyDeviceToDevice, s)
                   : launch_ingest(p->ip, src, const_cast<float*>(b.Y), s);
    };
    switch (op) {
        case FLMISR_OP_FORWARD:
            if (!in0 || !out) return fail(FLMISR_ERR_SHAPE, "FORWARD needs in0 and out");
            CUDA_TRY(launch_hr_copy(in0, p->W, 0, b.X[0], p->pitch, 0, H, p->W, s));
            if (gen) {
                CUDA_TRY(launch_gen_forward(sp0, p->gp, b.X[0], out, s));
            } else if (p->pc) {
                CUDA_TRY(launch_pc_forward_debug(sp0, p->pct, b.X[0], b.R[0], s));
                CUDA_TRY(launch_egest(ip0, b.R[0], out, s));
            } else {
                CUDA_TRY(launch_forward_debug(p->kr, sp0, b.X[0], b.R[0], s));
                CUDA_TRY(launch_egest(ip0, b.R[0], out, s));
            }
            break;
        case FLMISR_OP_ADJOINT:
            if (!in0 || !out) return fail(FLMISR_ERR_SHAPE, "ADJOINT needs in0 and out");
            if (gen) {
                CUDA_TRY(cudaMemcpyAsync(p->gp.w, in0, lr_bytes, cudaMemcpyDeviceToDevice, s));
                CUDA_TRY(launch_gen_adjoint(sp0, p->gp, p->gp.w, b.R[1], s));
            } else if (p->pc) {
                CUDA_TRY(launch_ingest(ip0, in0, b.R[0], s));
                CUDA_TRY(launch_pc_adjoint_debug(sp0, p->pct, b.R[0], b.R[1], s));
            } else {
                CUDA_TRY(launch_ingest(ip0, in0, b.R[0], s));
                CUDA_TRY(launch_adjoint_debug(p->kr, sp0, b.R[0], b.R[1], s));
            }
            CUDA_TRY(launch_hr_copy(b.R[1], p->pitch, 0, out, p->W, 0, H, p->W, s));
            break;
        case FLMISR_OP_GRAD:
        case FLMISR_OP_VALUE:
            if (!lr || !in0) return fail(FLMISR_ERR_SHAPE, "GRAD/VALUE need lr and in0");
            CUDA_TRY(put_lr(lr));
            CUDA_TRY(put_hr(b.X[0], in0));
            CUDA_TRY(cudaMemsetAsync(b.P[0], 0, p->hr_bytes, s));
            CUDA_TRY(cudaMemsetAsync(b.R[0], 0, p->hr_bytes, s));
            CUDA_TRY(launch_vg(p, PH_DEBUG, s));
            if (op == FLMISR_OP_GRAD && out) CUDA_TRY(get_hr(out, b.R[1]));
            break;
        case FLMISR_OP_CURV:
            if (!lr || !in0 || !in1) return fail(FLMISR_ERR_SHAPE, "CURV needs lr, in0 and in1");
            CUDA_TRY(put_lr(lr));
            CUDA_TRY(put_hr(b.X[0], in0));
            CUDA_TRY(cudaMemsetAsync(b.P[0], 0, p->hr_bytes, s));
            CUDA_TRY(put_hr(b.R[0], in1));
            CUDA_TRY(launch_uc(p, PH_DEBUG, s));
            break;
        case FLMISR_OP_INTERP:
            if (!lr || !out) return fail(FLMISR_ERR_SHAPE, "INTERP needs lr and out");
            if (p->fast && p->all_int && p->complete) {   // polyphase-complete, integer phases
                CUDA_TRY(launch_ingest(ip0, lr, b.R[0], s));
                CUDA_TRY(launch_hr_copy(b.R[0], p->pitch, 0, out, p->W, 0, H, p->W, s));
            } else {   // bilinear estimate everywhere, then the integer-phase frames' pixels on their sites
                flmisr_status ist = enqueue_interp(p, lr, out, p->W, 0, b.R[0], s);
                if (ist != FLMISR_OK) return ist;
            }
            break;
        case FLMISR_OP_X0:
            if (!lr || !out) return fail(FLMISR_ERR_SHAPE, "X0 needs lr and out");
            CUDA_TRY(launch_init_x0(p->ip, lr, b.X[0], s));
            CUDA_TRY(get_hr(out, b.X[0]));
            break;
        default:
            return fail(FLMISR_ERR_CONFIG, "unknown debug op");
    }
    CUDA_TRY(cudaMemcpyAsync(p->st_host, p->st, sizeof(ScgState), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (sc) {
        const double* d = p->st_host->dbg;
        if (op == FLMISR_OP_GRAD || op == FLMISR_OP_VALUE) { sc[0] = d[0]; sc[1] = d[1]; sc[2] = d[2]; }
        if (op == FLMISR_OP_CURV) { sc[0] = d[0] + p->cfg.lambda * d[1]; sc[1] = d[2]; sc[2] = d[3]; }
    }
    return FLMISR_OK;
}

}  // extern "C"

// ---- streaming capture-reconstruct pipeline ----
struct flmisr_pipeline_s {
    flmisr_plan_s* p = nullptr;
    int depth = 0, u16 = 0;
    float scale = 1.0f;
    size_t nlr = 0, nhr = 0, in_bytes = 0, out_bytes = 0;
    bool root = true;
    cudaStream_t up = nullptr, dn = nullptr;   // copy streams; compute runs on the plan's stream
    std::vector<void*> d_in, pin_in;
    std::vector<float*> d_out, pin_out, user_out;
    float* d_lr = nullptr;                     // fp32 frames converted from uint16 (compute stream)
    std::vector<cudaEvent_t> ev_up, ev_dn;
    ScgState* slot_state = nullptr;            // pinned, one per slot: the view's final SCG state
    std::vector<int> busy;
    long long submitted = 0, done = 0;
    flmisr_status first_err = FLMISR_OK;
    std::string err_msg;
    ScgState last{};
};

namespace {

bool host_pinned(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeHost;
}

// wait for slot `i`'s view (its download, hence its compute), record its status, copy staged output
flmisr_status pipe_complete(flmisr_pipeline_s* q, int i) {
    if (!q->busy[i]) return FLMISR_OK;
    q->busy[i] = 0;
    CUDA_TRY(cudaEventSynchronize(q->ev_dn[i]));
    if (q->user_out[i]) std::memcpy(q->user_out[i], q->pin_out[i], q->out_bytes);
    q->user_out[i] = nullptr;
    q->last = q->slot_state[i];
    q->done += 1;
    if (q->last.failed_stage && q->first_err == FLMISR_OK) {
        q->first_err = FLMISR_ERR_NUMERIC;
        q->err_msg = "pipeline view " + std::to_string(q->done - 1) + ": non-finite consensus scalar at SCG pass " +
                     std::to_string(q->last.failed_iter);
    }
    return FLMISR_OK;
}

}  // namespace

extern "C" {

flmisr_status flmisr_pipeline_destroy(flmisr_pipeline_t q) {
    if (!q) return FLMISR_OK;
    if (q->p && q->p->pipe == q) q->p->pipe = nullptr;
    for (int i = 0; i < q->depth; ++i)
        if (q->busy[i]) cudaEventSynchronize(q->ev_dn[i]);
    if (q->p && q->p->stream) cudaStreamSynchronize(q->p->stream);
    for (auto v : q->d_in) if (v) cudaFree(v);
    for (auto v : q->d_out) if (v) cudaFree(v);
    for (auto v : q->pin_in) if (v) cudaFreeHost(v);
    for (auto v : q->pin_out) if (v) cudaFreeHost(v);
    for (auto e : q->ev_up) if (e) cudaEventDestroy(e);
    for (auto e : q->ev_dn) if (e) cudaEventDestroy(e);
    if (q->d_lr) cudaFree(q->d_lr);
    if (q->slot_state) cudaFreeHost(q->slot_state);
    if (q->up) cudaStreamDestroy(q->up);
    if (q->dn) cudaStreamDestroy(q->dn);
    delete q;
    return FLMISR_OK;
}

flmisr_status flmisr_pipeline_create(flmisr_plan_t p, int32_t depth, int32_t input_u16, float u16_scale,
                                     flmisr_pipeline_t* out) {
    if (!out) return fail(FLMISR_ERR_SHAPE, "out is NULL");
    *out = nullptr;
    if (!p) return fail(FLMISR_ERR_SHAPE, "plan is NULL");
    if (depth < 2 || depth > 64) return fail(FLMISR_ERR_SHAPE, "pipeline depth must be in [2, 64]");
    if (input_u16 != 0 && input_u16 != 1) return fail(FLMISR_ERR_SHAPE, "input_u16 must be 0 or 1");
    if (input_u16 && !(u16_scale > 0.0f) ) return fail(FLMISR_ERR_SHAPE, "u16_scale must be > 0");
    if (p->virt) return fail(FLMISR_ERR_SHAPE, "virtual band plans cannot drive a pipeline");
    if (p->pipe) return fail(FLMISR_ERR_SHAPE, "the plan already drives a pipeline");
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    auto* q = new flmisr_pipeline_s();
    q->p = p;
    q->depth = depth;
    q->u16 = input_u16;
    q->scale = u16_scale;
    q->nlr = (size_t)p->cfg.k * p->cfg.lr_h * p->cfg.lr_w;
    q->nhr = (size_t)p->H * p->W;
    q->in_bytes = q->nlr * (input_u16 ? sizeof(uint16_t) : sizeof(float));
    q->out_bytes = q->nhr * sizeof(float);
    q->root = p->cfg.world == 1 || p->cfg.rank == 0;
    q->d_in.assign(depth, nullptr); q->pin_in.assign(depth, nullptr);
    q->d_out.assign(depth, nullptr); q->pin_out.assign(depth, nullptr); q->user_out.assign(depth, nullptr);
    q->ev_up.assign(depth, nullptr); q->ev_dn.assign(depth, nullptr);
    q->busy.assign(depth, 0);
    auto bad = [&](const char* what, cudaError_t e) {
        flmisr_pipeline_destroy(q);
        return fail(FLMISR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&q->up, cudaStreamNonBlocking)) != cudaSuccess) return bad("upload stream", e);
    if ((e = cudaStreamCreateWithFlags(&q->dn, cudaStreamNonBlocking)) != cudaSuccess) return bad("download stream", e);
    for (int i = 0; i < depth; ++i) {
        // input slots padded to 16 B (the uint16 conversion reads 8 codes per thread)
        if ((e = cudaMalloc(&q->d_in[i], (q->in_bytes + 15) / 16 * 16)) != cudaSuccess) return bad("cudaMalloc input slot", e);
        if ((e = cudaMalloc(&q->d_out[i], q->out_bytes)) != cudaSuccess) return bad("cudaMalloc output slot", e);
        if ((e = cudaEventCreateWithFlags(&q->ev_up[i], cudaEventDisableTiming)) != cudaSuccess) return bad("event", e);
        if ((e = cudaEventCreateWithFlags(&q->ev_dn[i], cudaEventDisableTiming)) != cudaSuccess) return bad("event", e);
    }
    if (input_u16 && (e = cudaMalloc(&q->d_lr, q->nlr * sizeof(float))) != cudaSuccess) return bad("cudaMalloc frames", e);
    if ((e = cudaMallocHost(&q->slot_state, (size_t)depth * sizeof(ScgState))) != cudaSuccess) return bad("pinned state", e);
    p->pipe = q;
    *out = q;
    return FLMISR_OK;
}

flmisr_status flmisr_pipeline_submit(flmisr_pipeline_t q, const void* lr_host, float* hr_host) {
    if (!q) return fail(FLMISR_ERR_SHAPE, "pipeline is NULL");
    if (!lr_host) return fail(FLMISR_ERR_SHAPE, "lr_host is NULL");
    if (q->root && !hr_host) return fail(FLMISR_ERR_SHAPE, "hr_host is NULL (world 1 / rank 0)");
    flmisr_plan_s* p = q->p;
    CUDA_TRY(cudaSetDevice(p->cfg.device));
    const int i = (int)(q->submitted % q->depth);
    flmisr_status st = pipe_complete(q, i);   // the slot's previous view must be out of the device buffers
    if (st != FLMISR_OK) return st;
    cudaStream_t cs = p->stream;
    // 1. upload (pageable sources are staged through the slot's pinned buffer)
    const void* src = lr_host;
    if (!host_pinned(lr_host)) {
        if (!q->pin_in[i]) CUDA_TRY(cudaMallocHost(&q->pin_in[i], q->in_bytes));
        std::memcpy(q->pin_in[i], lr_host, q->in_bytes);
        src = q->pin_in[i];
    }
    CUDA_TRY(cudaMemcpyAsync(q->d_in[i], src, q->in_bytes, cudaMemcpyHostToDevice, q->up));
    CUDA_TRY(cudaEventRecord(q->ev_up[i], q->up));
    // 2. reconstruct on the compute stream once the frames are in
    CUDA_TRY(cudaStreamWaitEvent(cs, q->ev_up[i], 0));
    const float* lr_dev = (const float*)q->d_in[i];
    if (q->u16) {
        CUDA_TRY(launch_u16_to_f32((const uint16_t*)q->d_in[i], q->d_lr, (long long)q->nlr, q->scale, cs));
        lr_dev = q->d_lr;
    }
    st = flmisr_reconstruct_async(p, lr_dev, nullptr, q->d_out[i], cs);
    p->pending = 0;   // the pipeline tracks completion per slot
    if (st != FLMISR_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(&q->slot_state[i], p->st, sizeof(ScgState), cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaEventRecord(p->done_ev, cs));
    // 3. download after the reconstruction (ev_dn marks the whole view complete on every rank)
    CUDA_TRY(cudaStreamWaitEvent(q->dn, p->done_ev, 0));
    if (q->root && hr_host) {
        float* dst = hr_host;
        if (!host_pinned(hr_host)) {
            if (!q->pin_out[i]) CUDA_TRY(cudaMallocHost(&q->pin_out[i], q->out_bytes));
            dst = q->pin_out[i];
            q->user_out[i] = hr_host;
        }
        CUDA_TRY(cudaMemcpyAsync(dst, q->d_out[i], q->out_bytes, cudaMemcpyDeviceToHost, q->dn));
    }
    CUDA_TRY(cudaEventRecord(q->ev_dn[i], q->dn));
    q->busy[i] = 1;
    q->submitted += 1;
    return FLMISR_OK;
}

flmisr_status flmisr_pipeline_wait(flmisr_pipeline_t q, int64_t* n_done, flmisr_report* rep) {
    if (!q) return fail(FLMISR_ERR_SHAPE, "pipeline is NULL");
    CUDA_TRY(cudaSetDevice(q->p->cfg.device));
    for (long long v = std::max(0LL, q->submitted - q->depth); v < q->submitted; ++v) {
        flmisr_status st = pipe_complete(q, (int)(v % q->depth));
        if (st != FLMISR_OK) return st;
    }
    if (n_done) *n_done = q->done;
    if (rep) {
        rep->iters_run = q->last.k;
        rep->accepted = q->last.accepted;
        rep->converged_at = q->last.converged_at;
        rep->failed_stage = q->last.failed_stage;
        rep->failed_iter = q->last.failed_iter;
    }
    const flmisr_status e = q->first_err;
    q->first_err = FLMISR_OK;
    if (e != FLMISR_OK) return fail(e, q->err_msg);
    return FLMISR_OK;
}

}  // extern "C"
