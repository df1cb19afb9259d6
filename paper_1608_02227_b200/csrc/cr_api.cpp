// libcr: C ABI (include/cr.h) and host orchestration of the P-APG hot path.
//
// Per iteration (Fig. 2) the host enqueues on the context stream:
//   prologue  (Step 1 closed form from the sums of Theta^{k-1}, Theta^{k-2})
//   [world > 1: ncclAllGather of y']
//   fused pass (Steps 2 + 4 for every owned pair, sums of Theta^k)
//   reduce    (fixed-order fp64 sums -> S^k; Step 3 momentum update on device)
//   [world > 1: ncclReduceScatter of the column sums]
// cr_solve replays the iteration as a CUDA graph (one graph per (Theta^{k-1}, Theta^{k-2})
// buffer assignment).  With CR_FLAG_ADAPTIVE a third Theta buffer (and sums slot) receives the
// trial Theta^k of the adaptive step rule, so a rejected trial leaves both state
// matrices intact; the host accepts or retries from two device scalars per trial.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>
#include <limits>

#include "../../include/cr.h"
#include "comm.h"
#include "cr_internal.h"

namespace cr {
double sigma_max_sq_lanczos(int64_t N, int n, const double *X, double tol, int max_iter);
}

using namespace cr;

namespace cr {
bool pdl_enabled() {
    static const bool on = !std::getenv("CR_NO_PDL");
    return on;
}
}  // namespace cr

namespace {

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
    int64_t N = 0, S = 0, Ns = 0, row0 = 0, Rp = 0, ldT = 0;
    int n = 0, NB = 0, NBP = 0, nRB = 0, world = 1, fp64 = 0;
    int nbuf = 2;                  // Theta buffers / sums slots (3 with CR_FLAG_ADAPTIVE)
    int64_t nbar = 1;              // partition block size (Assumption 1; 1: K = N, all pairs dualized)
    int64_t ipm_blocks = 0;        // blocks per shard (nbar > 1)
    size_t ipm_pb = 0, ipm = 0, ipm_it = 0, ipm_prof = 0, ipm_work = 0;   // per-block scratch (doubles), scratch and iteration offsets
    int ipm_smem = 0, ipm_G = 0;
    bool resident = false;         // small-N SMEM-resident solver eligible (row-major, n <= 32, world 1)
    size_t es = 4;
    // tensor-core pass
    bool tc = false;
    int NK = 0, NP2 = 0, nCBtc = 0, nRBtc = 0;
    // byte offsets
    size_t yg = 0, cpart = 0;      // resident solver: y of all rows, per-CTA column partials
    size_t th[3] = {0, 0, 0}, XT, Xh, X64, ybar, r[3] = {0, 0, 0}, c[3] = {0, 0, 0}, P[3] = {0, 0, 0}, dsq = 0, y64, yv, bv, XiT, Xi64, a64, colpart, rowpart,
        slot0, rb_ptr, rb_slots, cfull, ts, statpro, statres, g1h, g1l, g2h, g2l, XiR, slot0_tc, rb_ptr_tc, rb_slots_tc,
        XT64, XiT64, total;
    int nP = 0;                    // n rounded up to 8: rows of the k-major fp64 operands of the residual pass
};

// Kernel the library uses for this shape: the tcgen05 pass for fp32 with n >= 16 (where the
// two rank-n contractions make the CUDA-core pass FFMA-bound), else the SIMT pass.
bool use_tc(int n, cr_precision prec, cr_kernel kernel) {
    if (prec != CR_FP32) return false;
    if (kernel == CR_KERNEL_TC) return true;
    if (kernel == CR_KERNEL_SIMT) return false;
    return n >= 16;
}

bool make_layout(int64_t N, int n, cr_precision prec, cr_kernel kernel, int rank, int world, int flags,
                 int64_t nbar, Layout *L) {
    if (N < 2 || n < 1 || world < 1 || rank < 0 || rank >= world) return false;
    if (flags & ~(CR_FLAG_ADAPTIVE | CR_FLAG_P2P)) return false;
    if (nbar < 0) return false;
    L->nbar = std::max<int64_t>(nbar, 1);
    if (L->nbar > 1) {
        // Assumption 1: N = K nbar; blocks may not straddle shards; the adaptive check's
        // quadratic form (R15) holds only for the unconstrained Step 1 (K = N)
        if (N % L->nbar || L->nbar > kIpmMaxNbar || (flags & CR_FLAG_ADAPTIVE)) return false;
        if (world > 1 && ((N + world - 1) / world) % L->nbar) return false;
        L->ipm_G = block_ipm_group((int)L->nbar, n, kIpmMaxSmem);
        if (L->ipm_G < 1) return false;
        L->ipm_smem = (int)block_ipm_smem((int)L->nbar, n, L->ipm_G);
    }
    L->nbuf = (flags & CR_FLAG_ADAPTIVE) ? 3 : 2;
    if (kernel == CR_KERNEL_TC && prec != CR_FP32) return false;
    L->tc = use_tc(n, prec, kernel);
    L->N = N;
    L->n = n;
    L->world = world;
    L->fp64 = prec == CR_FP64;
    L->es = L->fp64 ? 8 : 4;
    L->NB = simt_bucket(n);
    if (L->NB == 0 || (L->fp64 && L->NB > 24)) return false;
    L->NBP = L->NB + 4;
    L->S = shard_rows(N, world, L->nbar);
    L->row0 = std::min<int64_t>(N, (int64_t)rank * L->S);
    L->Ns = std::min<int64_t>(N, L->row0 + L->S) - L->row0;
    L->Rp = (int64_t)align_up((size_t)std::max<int64_t>(L->S, 1), kRowAlign);
    L->ldT = (int64_t)align_up((size_t)N, kColAlign);
    L->nRB = (int)(L->Rp / kBM);
    const size_t es = L->es, A = 256;
    const int64_t WS = (int64_t)world * L->S;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + std::max<size_t>(bytes, 1), A); return r; };
    for (int b = 0; b < L->nbuf; ++b) L->th[b] = take((size_t)L->Rp * L->ldT * es);
    L->XT = take((size_t)L->NB * L->ldT * es);
    L->Xh = take((size_t)L->ldT * L->NBP * es);
    L->X64 = take((size_t)N * n * 8);
    L->nP = (n + 7) / 8 * 8;
    L->XT64 = take((size_t)L->nP * L->ldT * 8);
    L->XiT64 = take((size_t)L->nP * L->Rp * 8);
    L->ybar = take((size_t)N * 8);
    for (int s = 0; s < L->nbuf; ++s) {
        L->r[s] = take((size_t)L->Rp * 8);
        L->c[s] = take((size_t)L->Rp * 8);
        L->P[s] = take((size_t)L->Rp * n * 8);
    }
    L->dsq = take((size_t)L->Rp * 8);
    L->y64 = take((size_t)std::max(WS, N) * 8);
    L->yv = take((size_t)std::max(WS, L->ldT) * es);
    L->bv = take((size_t)L->Rp * es);
    L->XiT = take((size_t)L->NB * L->Rp * es);
    L->Xi64 = take((size_t)L->Rp * n * 8);
    L->a64 = take((size_t)L->Rp * 8);
    L->colpart = take((size_t)L->nRB * L->ldT * es);
    size_t rp_simt = (size_t)(L->nRB + kGMax) * kBM * L->NBP * 8;
    if (L->tc) {
        L->NK = (n + 7) / 8 * 8;
        L->NP2 = (n + 15) / 16 * 16;
        L->nCBtc = (int)((N + kTcBN - 1) / kTcBN);
        L->nRBtc = (int)(L->Rp / kTcBM);
        if (192 + L->NP2 + 2 * L->NK > 512) return false;     // TMEM columns
        rp_simt = std::max(rp_simt, (size_t)(L->nRBtc + kGMax) * kTcBM * (L->NP2 + 4) * 8);
    }
    L->rowpart = take(rp_simt);
    L->resident = !L->tc && n <= 32 && world == 1 && N <= kResidentMaxN && L->nbar == 1;
    if (L->resident) {
        L->yg = take((size_t)N * 8);
        L->cpart = take((size_t)kResidentMaxCTAs * N * 8);
    }
    L->slot0 = take((size_t)kGMax * 4);
    L->rb_ptr = take((size_t)(L->nRB + 1) * 4);
    L->rb_slots = take((size_t)(L->nRB + kGMax) * 4);
    L->cfull = take((size_t)WS * 8);
    L->ts = take(sizeof(DevScalars));
    L->statpro = take((size_t)kStatBlocks * 8 * 8);
    L->statres = take((size_t)kStatBlocks * 8 * 8);
    if (L->nbar > 1) {
        L->ipm_blocks = L->S / L->nbar;
        L->ipm_pb = block_ipm_scratch_per_block((int)L->nbar, n);
        L->ipm = take((size_t)L->ipm_blocks * L->ipm_pb * 8);
        L->ipm_it = take((size_t)L->ipm_blocks * 32);
        L->ipm_prof = take((size_t)L->ipm_blocks * 64);
        L->ipm_work = take((size_t)L->ipm_blocks * 24);
    }
    if (L->tc) {
        L->g1h = take((size_t)L->nCBtc * L->NK * 128);
        L->g1l = take((size_t)L->nCBtc * L->NK * 128);
        L->g2h = take((size_t)L->nCBtc * L->NP2 * 128);
        L->g2l = take((size_t)L->nCBtc * L->NP2 * 128);
        L->XiR = take((size_t)L->Rp * L->NK * 4);
        L->slot0_tc = take((size_t)kGMax * 4);
        L->rb_ptr_tc = take((size_t)(L->nRBtc + 1) * 4);
        L->rb_slots_tc = take((size_t)(L->nRBtc + kGMax) * 4);
    }
    L->total = o;
    return true;
}

// Slot tables for a persistent pass with G CTAs over T = nRB x nCB tiles (row-major),
// CTA g owning [g T / G, (g+1) T / G): slot0[g] = first row-partial slot of g; per row
// block, the slots of the CTA runs that cover it, in CTA order.
void slot_tables(int G, int64_t T, int nRB, int nCB, std::vector<int> &slot0, std::vector<int> &rb_ptr,
                 std::vector<int> &slots) {
    slot0.assign(G, 0);
    rb_ptr.assign(nRB + 1, 0);
    std::vector<std::vector<int>> per(nRB);
    int cur = 0;
    for (int g = 0; g < G; ++g) {
        const int64_t t0 = (int64_t)g * T / G, t1 = (int64_t)(g + 1) * T / G;
        slot0[g] = cur;
        if (t0 >= t1) continue;
        for (int64_t rb = t0 / nCB; rb <= (t1 - 1) / nCB; ++rb) per[rb].push_back(cur++);
    }
    slots.clear();
    for (int rb = 0; rb < nRB; ++rb) {
        rb_ptr[rb] = (int)slots.size();
        slots.insert(slots.end(), per[rb].begin(), per[rb].end());
    }
    rb_ptr[nRB] = (int)slots.size();
    if (slots.empty()) slots.push_back(0);
}

}  // namespace

struct cr_ctx {
    Layout lay;
    cr_precision prec = CR_FP32;
    cr_kernel kernel = CR_KERNEL_SIMT;
    double gamma = 0, L = 0;
    double sigma2 = 0;   // sigma_max(C)^2 = L gamma (Eq. (lischitz)), for cr_set_gamma
    int rank = 0, world = 1, device = 0;
    cudaStream_t stream = nullptr;
    char *ws = nullptr;
    // device views
    void *th[3] = {nullptr, nullptr, nullptr};
    double *r[3], *c[3], *P[3];      // sums slot b holds the sums of Theta buffer b
    int bA = 0;          // buffer holding Theta^k (= Theta^{k-1} of the next iteration)
    int bB = 1;          // buffer holding Theta^{k-1} (= Theta^{k-2} of the next iteration)
    // step rule: constant 1/L, or adaptive 1/s_k
    cr_step_rule rule = CR_STEP_CONSTANT;
    double ups = 2.0;    // growth factor upsilon > 1
    int max_trials = 64;  // (s_{k-1}, trial counters: device-resident, DevScalars::ad)
    bool backtrack = false;  // CR_STEP_BACKTRACK (monotone variant of the adaptive rule)
    cudaGraphExec_t graph_ad[9] = {};   // adaptive iteration (WHILE loop over trials) per (bA, bB)
    int64_t k = 0;
    int G = 0, nCB = 0;
    int64_t T = 0;
    int64_t launches = 0;
    bool poisoned = false;
    int64_t multi_launches = 0;   // kernels in one kMultiIters-iteration graph
    int g1passes = 3;             // tcgen05 pass: tf32 passes of GEMM1
    int g1f16 = 1, xexp = 0;      // tcgen05 pass: GEMM1 in kind::f16 (X scaled by 2^xexp)
    int g1_runahead = 0;          // tcgen05 pass: GEMM1 runs ahead of the Theta stream (CR_TC_G1_RUNAHEAD)
    unsigned long long *tc_check = nullptr;   // CR_TC_CHECK=1: ring-protocol violation word
    std::string err;
    // pass timing
    bool timing = false;
    std::vector<cudaEvent_t> ev;
    size_t ev_used = 0;
    std::vector<cudaEvent_t> bp_ev;   // block-projection launches (partition K < N), same switch
    size_t bp_ev_used = 0;
    double bp_ms = 0.0;               // their summed time, collected by cr_pass_timing
    int64_t bp_launches = 0;
    int64_t ev_iters = 0;    // iterations covered by the recorded event pairs
    // small-N SMEM-resident solver (kernels/resident.cu): CTAs, rows per CTA (0: not usable)
    int res_G = 0, res_R = 0, res_ldS = 0;
    // constant-step graphs per (bA, bB) assignment
    cudaGraphExec_t graph[9] = {};
    cudaGraphExec_t graph_multi[9] = {};   // kMultiIters constant-step iterations per replay
    cudaStream_t cap_stream = nullptr;   // private stream used only to record graphs
    // tensor-core pass
    int G_tc = 0, stages = 0, g1stages = 0, g2stages = 0, window = 64, smem_tc = 0;
    int64_t T_tc = 0;
    unsigned long long *trace = nullptr;   // debug timeline buffer (CR_TC_TRACE=<file>)
    Comm comm;           // NCCL communicator or in-process local group (world > 1)
    // CR_FLAG_P2P: peer-memory reduce-scatter of the column sums (receive slab + flags + epoch
    // in p2p_buf, IPC-mapped by the other ranks; p2p_tab = device table of every rank's slab
    // and flag array)
    bool p2p = false;
    double *p2p_buf = nullptr;       // [W S] c slab | c flags [W] | c epoch | y flags [W] | y epoch | (256-B) y' receive [W S]
    void **p2p_tab = nullptr;        // [4][kP2PTab]: every rank's c slab, c flags, y' receive, y flags
    size_t p2p_yf = 0, p2p_yr = 0;   // byte offsets of the y flags and the y' receive array in p2p_buf
    std::vector<void *> p2p_opened;
    bool coll = false;   // collectives active: world > 1, or a 1-rank NCCL comm (CR_FORCE_NCCL test mode)

    template <typename P> P *at(size_t off) { return reinterpret_cast<P *>(ws + off); }
};

namespace {

cr_status fail(cr_ctx *c, cr_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        if (s == CR_ERR_CUDA || s == CR_ERR_NCCL || s == CR_ERR_OOM) c->poisoned = true;
    }
    return s;
}

#define CK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return fail(ctx, CR_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,           \
                        cudaGetErrorString(e_));                                               \
    } while (0)
#define CM(call)                                                                               \
    do {                                                                                       \
        const char *m_ = (call);                                                               \
        if (m_) return fail(ctx, CR_ERR_NCCL, "%s:%d %s", __FILE__, __LINE__, m_);             \
    } while (0)

PassParams pass_params(cr_ctx *ctx, int b_read, int b_read2, int b_out = -1, bool adapt = false) {
    const Layout &Ly = ctx->lay;
    PassParams p{};
    p.B1 = ctx->th[b_read];
    p.B2 = ctx->th[b_read2];
    p.Bout = ctx->th[b_out < 0 ? b_read2 : b_out];
    p.adapt = adapt ? 1 : 0;
    p.dcol = Ly.n + 1;
    p.tiled = Ly.tc ? 1 : 0;
    p.nCBt = Ly.nCBtc;
    p.ldT = Ly.ldT;
    p.N = Ly.N;
    p.Ns = Ly.Ns;
    p.row0 = Ly.row0;
    p.nbar = Ly.nbar;
    p.nRB = Ly.nRB;
    p.nCB = ctx->nCB;
    p.T = ctx->T;
    p.G = ctx->G;
    p.XT = ctx->ws + Ly.XT;
    p.Xh = ctx->ws + Ly.Xh;
    p.XiT = ctx->ws + Ly.XiT;
    p.bv = ctx->ws + Ly.bv;
    p.yv = ctx->ws + Ly.yv;
    p.Rp = Ly.Rp;
    p.colpart = ctx->ws + Ly.colpart;
    p.rowpart = ctx->at<double>(Ly.rowpart);
    p.cta_slot0 = ctx->at<int>(Ly.slot0);
    p.ts = ctx->at<double>(Ly.ts);
    return p;
}

ReduceParams reduce_params(cr_ctx *ctx, int slot, int advance, bool tc = false, bool adapt = false) {
    const Layout &Ly = ctx->lay;
    ReduceParams q{};
    q.N = Ly.N;
    q.Ns = Ly.Ns;
    q.Rp = Ly.Rp;
    q.ldT = Ly.ldT;
    q.n = Ly.n;
    q.NBP = tc ? Ly.NP2 + 4 : Ly.NBP;
    q.rcol0 = tc ? Ly.NP2 : Ly.n;
    q.rcol1 = tc ? Ly.NP2 + 1 : -1;
    q.dcol0 = adapt ? (tc ? Ly.NP2 + 2 : Ly.n + 1) : -1;
    q.dcol1 = (adapt && tc) ? Ly.NP2 + 3 : -1;
    q.dsq = ctx->at<double>(Ly.dsq);
    q.nRB = tc ? Ly.nRBtc : Ly.nRB;
    q.rbm = tc ? kTcBM : kBM;
    q.colpart = ctx->ws + Ly.colpart;
    q.rowpart = ctx->at<double>(Ly.rowpart);
    q.rb_ptr = ctx->at<int>(tc ? Ly.rb_ptr_tc : Ly.rb_ptr);
    q.rb_slots = ctx->at<int>(tc ? Ly.rb_slots_tc : Ly.rb_slots);
    q.r = ctx->r[slot];
    q.P = ctx->P[slot];
    q.c_out = ctx->coll ? ctx->at<double>(Ly.cfull) : ctx->c[slot];
    if (ctx->p2p) {
        q.p2p_recv = reinterpret_cast<double *const *>(ctx->p2p_tab);
        q.p2p_flag = reinterpret_cast<unsigned long long *const *>(ctx->p2p_tab + kP2PTab);
        q.p2p_rank = ctx->rank;
        q.p2p_S = Ly.S;
    }
    q.ts = ctx->at<DevScalars>(Ly.ts);
    q.advance_t = advance;
    return q;
}

SmallParams small_params(cr_ctx *ctx, int sa, int sb, int use_beta, double scale, bool stats) {
    const Layout &Ly = ctx->lay;
    SmallParams p{};
    p.N = Ly.N;
    p.Ns = Ly.Ns;
    p.row0 = Ly.row0;
    p.Rp = Ly.Rp;
    p.ldT = Ly.ldT;
    p.n = Ly.n;
    p.NB = Ly.NB;
    p.NBP = Ly.NBP;
    p.gamma = ctx->gamma;
    p.scale = scale;
    p.X64 = ctx->at<double>(Ly.X64);
    p.ybar = ctx->at<double>(Ly.ybar);
    p.r1 = ctx->r[sa]; p.c1 = ctx->c[sa]; p.P1 = ctx->P[sa];
    p.r2 = ctx->r[sb]; p.c2 = ctx->c[sb]; p.P2 = ctx->P[sb];
    p.y64 = ctx->at<double>(Ly.y64);
    p.Xi64 = ctx->at<double>(Ly.Xi64);
    p.a64 = ctx->at<double>(Ly.a64);
    p.yv = ctx->ws + Ly.yv;
    p.bv = ctx->ws + Ly.bv;
    p.XiT = Ly.tc ? nullptr : ctx->ws + Ly.XiT;          // the SIMT pass operand only
    p.statpart = stats ? ctx->at<double>(Ly.statpro) : nullptr;
    p.ts = ctx->at<DevScalars>(Ly.ts);
    p.use_beta = use_beta;
    p.XiR = Ly.tc ? ctx->at<float>(Ly.XiR) : nullptr;
    p.NK = Ly.NK;
    if (ctx->p2p) {
        p.p2p_yrecv = ctx->p2p_tab + 2 * kP2PTab;
        p.p2p_yflag = reinterpret_cast<unsigned long long *const *>(ctx->p2p_tab + 3 * kP2PTab);
        p.p2p_rank = ctx->rank;
        p.p2p_W = ctx->world;
    }
    return p;
}

TcParams tc_params(cr_ctx *ctx, int b1, int b2, int bo, bool adapt = false) {
    const Layout &Ly = ctx->lay;
    TcParams p{};
    p.B1 = static_cast<const float *>(ctx->th[b1]);
    p.B2 = static_cast<const float *>(ctx->th[b2]);
    p.Bout = static_cast<float *>(ctx->th[bo]);
    p.N = Ly.N;
    p.Ns = Ly.Ns;
    p.row0 = Ly.row0;
    p.nbar = Ly.nbar;
    p.ldT = Ly.ldT;
    p.T = ctx->T_tc;
    p.G = ctx->G_tc;
    p.nCB = Ly.nCBtc;
    p.NK = Ly.NK;
    p.NP2 = Ly.NP2;
    p.stages = ctx->stages;
    p.window = ctx->window;
    p.g1stages = ctx->g1stages;
    p.g1passes = ctx->g1passes;
    p.g1f16 = ctx->g1f16;
    p.xexp = ctx->xexp;
    p.n = Ly.n;
    p.g2stages = ctx->g2stages;
    p.adapt = adapt ? 1 : 0;
    p.poll_ns = std::getenv("CR_TC_POLL_NS") ? std::atoi(std::getenv("CR_TC_POLL_NS")) : 64;
    // L2 policy of the Theta stream: evict-normal for loads and stores measured +1.6% at C4
    // (0.878 -> 0.892), but -1.5% at C5 where the 84 MB of X images (evict-last) need the L2,
    // and -1% at C3 (state ~ L2): used when the images are small and the state far exceeds L2
    {
        const double img = 2.0 * (double)Ly.nCBtc * (Ly.NK + Ly.NP2) * 128.0;
        p.theta_l2 = (img <= 32e6 && Ly.N >= 8192) ? 3 : 0;
        if (const char *e = std::getenv("CR_TC_THETA_L2")) p.theta_l2 = std::atoi(e);
    }
    p.smem_bytes = ctx->smem_tc;
    p.g1_hi = ctx->at<float>(Ly.g1h);
    p.g1_lo = ctx->at<float>(Ly.g1l);
    p.g2_hi = ctx->at<float>(Ly.g2h);
    p.g2_lo = ctx->at<float>(Ly.g2l);
    p.yv = ctx->at<float>(Ly.yv);
    p.XiR = ctx->at<float>(Ly.XiR);
    p.bv = ctx->at<float>(Ly.bv);
    p.colpart = ctx->at<float>(Ly.colpart);
    p.rowpart = ctx->at<double>(Ly.rowpart);
    p.cta_slot0 = ctx->at<int>(Ly.slot0_tc);
    p.trace = ctx->trace;
    p.ts = ctx->at<double>(Ly.ts);
    p.g1_runahead = ctx->g1_runahead;
    p.check = ctx->tc_check;
    return p;
}

cudaEvent_t next_bp_event(cr_ctx *ctx) {
    if (ctx->bp_ev_used == ctx->bp_ev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        ctx->bp_ev.push_back(e);
    }
    return ctx->bp_ev[ctx->bp_ev_used++];
}

cudaEvent_t next_event(cr_ctx *ctx) {
    if (ctx->ev_used == ctx->ev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        ctx->ev.push_back(e);
    }
    return ctx->ev[ctx->ev_used++];
}

// The column sums of slot s for this rank's rows from every rank's partials: NCCL / local
// reduce-scatter of cfull, or (CR_FLAG_P2P) the owner-side gather of the peer-memory slabs the
// reduce kernels of all ranks stored into.
cr_status reduce_scatter_c(cr_ctx *ctx, int s) {
    const Layout &Ly = ctx->lay;
    if (ctx->p2p) {
        P2PGather g{};
        g.W = ctx->world;
        g.S = Ly.S;
        g.Ns = Ly.Ns;
        g.slab = ctx->p2p_buf;
        g.flag = reinterpret_cast<unsigned long long *>(ctx->p2p_buf + (size_t)ctx->world * Ly.S);
        g.epoch = g.flag + ctx->world;
        const int cbw = reduce_col_block(Ly.fp64);
        g.nblk = (Ly.Ns + cbw - 1) / cbw;
        g.c_out = ctx->c[s];
        CK(launch_p2p_gather(g, ctx->stream));
        ctx->launches += 1;
        return CR_OK;
    }
    CM(comm_reduce_scatter_f64(ctx->comm, ctx->at<double>(Ly.cfull), ctx->c[s], (size_t)Ly.S, ctx->stream));
    return CR_OK;
}

// Sums (r, c, Theta X) of buffer b into slot s, read-only pass.
cr_status enqueue_sums(cr_ctx *ctx, int b, int s) {
    const Layout &Ly = ctx->lay;
    PassParams p = pass_params(ctx, b, b);
    CK(launch_pass_simt(p, Ly.fp64, Ly.NB, MODE_SUMS, ctx->stream));
    ReduceParams q = reduce_params(ctx, s, 0);
    CK(launch_reduce(q, Ly.fp64, ctx->stream));
    ctx->launches += 2;
    if (ctx->coll) {
        cr_status st = reduce_scatter_c(ctx, s);
        if (st != CR_OK) return st;
    }
    return CR_OK;
}

// Partition K < N (Assumption 1): Step 1 = the closed-form point just written by the prologue
// projected per block onto the intra-block constraints (block_ipm), then the prologue again in
// from_eta mode to refresh a, the pass operands and (stats) the objective partials.
cr_status project_blocks(cr_ctx *ctx, SmallParams sp, int *nb_pro, bool allow_timing = false, bool push = false) {
    const Layout &Ly = ctx->lay;
    BlockIpmParams bp{};
    bp.nbar = (int)Ly.nbar;
    bp.n = Ly.n;
    bp.max_iter = kIpmMaxIter;
    bp.nblocks = Ly.Ns / Ly.nbar;
    bp.row0 = Ly.row0;
    bp.gamma = ctx->gamma;
    bp.tol = kIpmTol;
    bp.X64 = ctx->at<double>(Ly.X64);
    bp.y64 = ctx->at<double>(Ly.y64);
    bp.Xi64 = ctx->at<double>(Ly.Xi64);
    bp.scratch = ctx->at<double>(Ly.ipm);
    bp.scratch_per_block = Ly.ipm_pb;
    bp.iters = ctx->at<int>(Ly.ipm_it);
    bp.smem = Ly.ipm_smem;
    bp.lgroup = Ly.ipm_G;
    bp.warm = std::getenv("CR_IPM_COLD") ? 0 : 1;
    bp.work = ctx->at<unsigned long long>(Ly.ipm_work);
    bp.prof = std::getenv("CR_IPM_PROF") ? ctx->at<unsigned long long>(Ly.ipm_prof) : nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (allow_timing && ctx->timing) {
        e0 = next_bp_event(ctx);
        e1 = next_bp_event(ctx);
        if (!e0 || !e1) return fail(ctx, CR_ERR_CUDA, "cudaEventCreate failed");
        CK(cudaEventRecord(e0, ctx->stream));
    }
    CK(launch_block_ipm(bp, ctx->stream));
    if (e1) CK(cudaEventRecord(e1, ctx->stream));
    sp.from_eta = 1;
    sp.p2p_push = push ? 1 : 0;                 // the step's final y' (partition): sent to the peers
    CK(launch_prologue(sp, Ly.fp64, ctx->stream, nb_pro));
    ctx->launches += 2;
    return CR_OK;
}

// One P-APG iteration (no host sync): Step 1 at theta~^k from the sums of Theta^{k-1} (bA) and
// Theta^{k-2} (bB) with step 1/s (scale), then the fused pass writing Theta^k into buffer bo
// (bB in place for the constant step; the spare buffer for an adaptive trial) and its sums
// into slot bo.  advance_t: Step 3 on the device (constant step); adapt: also ||D||^2 per row.
// fuse (constant step inside a multi-iteration graph, can_fuse): FUSE_NONE = prologue, pass,
// reduce; FUSE_FIRST = prologue, pass (reduce deferred); FUSE_MID = reduce of the previous
// iteration fused with this prologue (reduce_prologue_kernel), pass; FUSE_LAST = fused, pass, reduce.
enum FuseMode { FUSE_NONE = 0, FUSE_FIRST = 1, FUSE_MID = 2, FUSE_LAST = 3 };

bool can_fuse(const cr_ctx *ctx) {
    const Layout &Ly = ctx->lay;
    return !Ly.fp64 && !ctx->coll && !ctx->p2p && Ly.nbar == 1 && !std::getenv("CR_NO_FUSE");
}

cr_status enqueue_step(cr_ctx *ctx, bool allow_timing, int bo, double scale, bool advance_t, bool adapt,
                       const double *s_dev = nullptr, int fuse = FUSE_NONE) {
    const Layout &Ly = ctx->lay;
    const int bA = ctx->bA, bB = ctx->bB;
    SmallParams sp = small_params(ctx, bA, bB, 1, scale, false);
    sp.s_dev = s_dev;
    sp.p2p_push = (ctx->p2p && Ly.nbar == 1) ? 1 : 0;
    if (fuse == FUSE_MID || fuse == FUSE_LAST) {
        // the previous iteration's Theta^k is buffer bA now: its reduce + this Step 1
        ReduceParams q = reduce_params(ctx, bA, 1, Ly.tc, false);
        CK(launch_reduce_prologue(q, sp, ctx->stream));
    } else {
        CK(launch_prologue(sp, Ly.fp64, ctx->stream, nullptr));
    }
    if (Ly.nbar > 1) {
        sp.p2p_push = 0;
        cr_status st = project_blocks(ctx, sp, nullptr, allow_timing, ctx->p2p);
        if (st != CR_OK) return st;
    }
    // CR_FLAG_P2P with the tensor-core pass (all pairs): the y' acquire is fused into the pass
    // (TcParams::yflag, own columns first); otherwise a one-CTA acquire + copy kernel
    const bool p2p_fused = ctx->p2p && Ly.tc && Ly.nbar == 1 && !std::getenv("CR_P2P_YGATHER");
    if (ctx->p2p && !p2p_fused) {
        // y' all-gather over peer memory: every rank's prologue pushed its rows; acquire + copy
        P2PYGather g{};
        g.yrecv = reinterpret_cast<char *>(ctx->p2p_buf) + ctx->p2p_yr;
        g.flag = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(ctx->p2p_buf) + ctx->p2p_yf);
        g.epoch = g.flag + ctx->world;
        g.W = ctx->world;
        g.N = Ly.N;
        g.S = Ly.S;
        g.yv = ctx->ws + Ly.yv;
        CK(launch_p2p_ygather(g, Ly.fp64, ctx->stream));
        ctx->launches += 1;
    } else if (ctx->coll) {
        CM(comm_allgather(ctx->comm, ctx->ws + Ly.yv, (size_t)Ly.S, (int)Ly.es, ctx->stream));
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (allow_timing && ctx->timing) {
        e0 = next_event(ctx);
        e1 = next_event(ctx);
        if (!e0 || !e1) return fail(ctx, CR_ERR_CUDA, "cudaEventCreate failed");
        CK(cudaEventRecord(e0, ctx->stream));
    }
    if (Ly.tc) {
        TcParams tp = tc_params(ctx, bA, bB, bo, adapt);
        if (p2p_fused) {
            char *pb = reinterpret_cast<char *>(ctx->p2p_buf);
            tp.yv = reinterpret_cast<const float *>(pb + ctx->p2p_yr);
            tp.yflag = reinterpret_cast<const unsigned long long *>(pb + ctx->p2p_yf);
            tp.yepoch = tp.yflag + ctx->world;
            tp.W = ctx->world;
            tp.S = Ly.S;
            tp.rot = (int)((Ly.row0 / kTcBN) % Ly.nCBtc);
        }
        CK(launch_pass_tc(tp, ctx->stream));
    } else {
        PassParams p = pass_params(ctx, bA, bB, bo, adapt);
        CK(launch_pass_simt(p, Ly.fp64, Ly.NB, MODE_STEP, ctx->stream));
    }
    if (e1) {
        CK(cudaEventRecord(e1, ctx->stream));
        ctx->ev_iters += 1;
    }
    if (fuse == FUSE_FIRST || fuse == FUSE_MID) {      // reduce deferred into the next prologue
        ctx->launches += 2;
        return CR_OK;
    }
    ReduceParams q = reduce_params(ctx, bo, advance_t ? 1 : 0, Ly.tc, adapt);
    if (p2p_fused)                                     // the pass consumed this epoch's peer y'
        q.yepoch = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(ctx->p2p_buf) + ctx->p2p_yf) +
                   ctx->world;
    CK(launch_reduce(q, Ly.fp64, ctx->stream));
    if (ctx->coll) {
        cr_status st = reduce_scatter_c(ctx, bo);
        if (st != CR_OK) return st;
    }
    ctx->launches += 3;
    return CR_OK;
}

// Theta^k now in buffer bo: it becomes Theta^{k-1} of the next iteration, the old Theta^{k-1}
// becomes Theta^{k-2}.
void advance_host(cr_ctx *ctx, int bo) {
    ctx->bB = ctx->bA;
    ctx->bA = bo;
    ctx->k += 1;
}

// One adaptive trial, all on the device: Step 1 with 1/s of the trial (ts->ad),
// the fused pass writing the trial Theta^k into the spare buffer (+ ||D||^2), the reduce, the
// check (Eq. (adaptive-check) in quadratic form, R15) and the accept/retry kernel
// (which drives the WHILE node `cond` when the trial runs inside a CUDA graph).
cr_status enqueue_adaptive_trial(cr_ctx *ctx, unsigned long long cond, int has_cond, bool allow_timing) {
    const Layout &Ly = ctx->lay;
    const int bo = 3 - ctx->bA - ctx->bB;
    DevScalars *ts = ctx->at<DevScalars>(Ly.ts);
    cr_status st = enqueue_step(ctx, allow_timing, bo, 0.0, false, true, &ts->ad[AD_STRY]);
    if (st != CR_OK) return st;
    AdaptParams ap{};
    ap.Ns = Ly.Ns;
    ap.row0 = Ly.row0;
    ap.n = Ly.n;
    ap.gamma = ctx->gamma;
    ap.X64 = ctx->at<double>(Ly.X64);
    ap.rA = ctx->r[ctx->bA]; ap.cA = ctx->c[ctx->bA]; ap.PA = ctx->P[ctx->bA];
    ap.rB = ctx->r[ctx->bB]; ap.cB = ctx->c[ctx->bB]; ap.PB = ctx->P[ctx->bB];
    ap.rO = ctx->r[bo]; ap.cO = ctx->c[bo]; ap.PO = ctx->P[bo];
    ap.dsq = ctx->at<double>(Ly.dsq);
    ap.statpart = ctx->at<double>(Ly.statres);
    ap.ts = ts;
    CK(launch_adapt_check(ap, ctx->stream));
    if (ctx->coll) CM(comm_allreduce_f64(ctx->comm, ts->stats + 8, 2, COLL_SUM, ctx->stream));
    CK(launch_adapt_decide(ts, cond, has_cond, ctx->stream));
    ctx->launches += 3;
    return CR_OK;
}

// An adaptive iteration whose trials l = 0 .. max_trials-1 all failed Eq. (adaptive-check): the
// device did not advance t_k and holds a rejected trial in the spare buffer, so there is no valid
// iterate to continue from -- the context is poisoned (include/cr.h, cr_set_step_rule).
cr_status adaptive_exhausted(cr_ctx *ctx) {
    ctx->poisoned = true;
    return fail(ctx, CR_ERR_STATE, "adaptive step: no l < %d passed Eq. (adaptive-check); context poisoned",
                ctx->max_trials);
}

// true if the device recorded an exhausted adaptive iteration (synchronizes)
cr_status adaptive_error_flag(cr_ctx *ctx, bool *failed) {
    double err = 0.0;
    CK(cudaMemcpyAsync(&err, &ctx->at<DevScalars>(ctx->lay.ts)->ad[AD_ERR], sizeof err, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *failed = err != 0.0;
    return CR_OK;
}

// One adaptive iteration driven from the host (local groups, per-pass timing): one trial per
// round trip; the accept/retry state lives on the device exactly as in the graph path.
cr_status adaptive_step(cr_ctx *ctx) {
    const Layout &Ly = ctx->lay;
    const int bo = 3 - ctx->bA - ctx->bB;
    DevScalars *ts = ctx->at<DevScalars>(Ly.ts);
    for (;;) {
        cr_status st = enqueue_adaptive_trial(ctx, 0, 0, true);
        if (st != CR_OK) return st;
        double ad[8];
        CK(cudaMemcpyAsync(ad, ts->ad, sizeof ad, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (ad[AD_ERR] != 0.0) return adaptive_exhausted(ctx);
        if (ad[AD_L] == 0.0) break;                       // accepted
    }
    advance_host(ctx, bo);
    return CR_OK;
}

// CUDA graph of one adaptive iteration: a WHILE node whose body is one trial; the decide kernel
// leaves the loop on acceptance.  One graph per (bA, bB) assignment (the spare buffer differs).
cr_status build_adaptive_graph(cr_ctx *ctx, int key) {
    const int bA = ctx->bA, bB = ctx->bB;
    const int64_t k = ctx->k, launches = ctx->launches;
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        return fail(ctx, CR_ERR_CUDA, "adaptive graph: %s", cudaGetErrorString(e));
    }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->cap_stream;
    e = cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    cr_status st = e == cudaSuccess ? enqueue_adaptive_trial(ctx, h, 1, false) : CR_ERR_CUDA;
    cudaGraph_t out = nullptr;
    const cudaError_t e2 = e == cudaSuccess ? cudaStreamEndCapture(ctx->stream, &out) : e;
    ctx->stream = user;
    ctx->bA = bA; ctx->bB = bB; ctx->k = k; ctx->launches = launches;
    if (st != CR_OK || e2 != cudaSuccess) {
        cudaGraphDestroy(g);
        return st != CR_OK ? st : fail(ctx, CR_ERR_CUDA, "adaptive graph capture: %s", cudaGetErrorString(e2));
    }
    e = cudaGraphInstantiate(&ctx->graph_ad[key], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(ctx, CR_ERR_CUDA, "adaptive graph instantiate: %s", cudaGetErrorString(e));
    return CR_OK;
}

bool use_adaptive_graph(const cr_ctx *ctx) {
    return !ctx->coll && !ctx->timing && ctx->world == 1 && !std::getenv("CR_NO_ADAPTIVE_GRAPH");
}

// eta(Theta^k) and diagnostics (Theorem 1 semantics); synchronizes once.  With y_host / xi_host
// (cr_primal) the D2H copies of eta join the same synchronization.
cr_status eval_stats(cr_ctx *ctx, cr_step_stats *out, double *y_host = nullptr, double *xi_host = nullptr) {
    const Layout &Ly = ctx->lay;
    const int s = ctx->bA, b = ctx->bA;
    int nb_pro = 0, nb_res = 0;
    SmallParams sp = small_params(ctx, s, s, 0, 1.0, true);
    CK(launch_prologue(sp, Ly.fp64, ctx->stream, &nb_pro));
    if (Ly.nbar > 1) {
        cr_status st = project_blocks(ctx, sp, &nb_pro);
        if (st != CR_OK) return st;
    }
    double *y64 = ctx->at<double>(Ly.y64);
    if (ctx->coll) CM(comm_allgather(ctx->comm, y64, (size_t)Ly.S, 8, ctx->stream));
    ResidualParams rp{};
    rp.Theta = ctx->th[b];
    rp.ldT = Ly.ldT;
    rp.tiled = Ly.tc ? 1 : 0;
    rp.nCBt = Ly.nCBtc;
    rp.N = Ly.N;
    rp.Ns = Ly.Ns;
    rp.row0 = Ly.row0;
    rp.Rp = Ly.Rp;
    rp.n = Ly.n;
    rp.X64 = ctx->at<double>(Ly.X64);
    rp.y64 = y64;
    rp.Xi64 = ctx->at<double>(Ly.Xi64);
    rp.a64 = ctx->at<double>(Ly.a64);
    rp.statpart = ctx->at<double>(Ly.statres);
    rp.nP = Ly.nP;
    rp.XT = ctx->at<double>(Ly.XT64);
    rp.ldX = Ly.ldT;
    rp.XiT = ctx->at<double>(Ly.XiT64);
    CK(launch_residual(rp, Ly.fp64, ctx->stream, &nb_res));
    DevScalars *ts = ctx->at<DevScalars>(Ly.ts);
    CK(launch_stats_finalize(ctx->at<double>(Ly.statpro), nb_pro, ctx->at<double>(Ly.statres), nb_res, ts,
                             ctx->stream));
    ctx->launches += 4;
    if (ctx->coll) {
        // stats[0..5] and [7] are sums; [6] is a max
        CM(comm_allreduce_f64(ctx->comm, ts->stats, 6, COLL_SUM, ctx->stream));
        CM(comm_allreduce_f64(ctx->comm, ts->stats + 6, 1, COLL_MAX, ctx->stream));
        CM(comm_allreduce_f64(ctx->comm, ts->stats + 7, 1, COLL_SUM, ctx->stream));
    }
    DevScalars h{};
    CK(cudaMemcpyAsync(&h, ts, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    if (y_host) CK(cudaMemcpyAsync(y_host, y64, (size_t)Ly.N * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (xi_host && Ly.Ns > 0)
        CK(cudaMemcpyAsync(xi_host, ctx->ws + Ly.Xi64, (size_t)Ly.Ns * Ly.n * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (out) {
        const double u2 = h.stats[0], uy = h.stats[1], xi2 = h.stats[2];
        const double Nd = (double)Ly.N;
        out->k = ctx->k;
        out->t_k = h.t_cur;
        out->r_gamma = 0.5 * u2 + 0.5 * ctx->gamma * xi2;                 // Eq. (regularize)
        out->gap = h.stats[4];                                            // <theta, C eta>
        // g at eta(theta): the Lagrangian at its minimizer, r_gamma - <theta, C eta>; at
        // K = N its closed form (no cancellation between r_gamma and gap)
        out->g = Ly.nbar > 1 ? out->r_gamma - out->gap : -0.5 * u2 - 0.5 * ctx->gamma * xi2 - uy;
        out->max_violation = h.stats[6];
        out->infeas_norm = std::sqrt(h.stats[5]) / std::sqrt(Nd * Nd - Nd);
        out->nonfinite = (h.stats[3] + h.stats[7]) > 0 ||
                         !std::isfinite(out->g) || !std::isfinite(out->gap);
    }
    return CR_OK;
}

// eta(Theta^k) (Step-1 formulas at Theta^k, Theorem 1) into y64 (all rows), Xi64, a64.
cr_status compute_eta(cr_ctx *ctx) {
    const Layout &Ly = ctx->lay;
    SmallParams sp = small_params(ctx, ctx->bA, ctx->bA, 0, 1.0, false);
    CK(launch_prologue(sp, Ly.fp64, ctx->stream, nullptr));
    ctx->launches += 1;
    if (Ly.nbar > 1) {
        cr_status st = project_blocks(ctx, sp, nullptr);
        if (st != CR_OK) return st;
    }
    if (ctx->coll) CM(comm_allgather(ctx->comm, ctx->at<double>(Ly.y64), (size_t)Ly.S, 8, ctx->stream));
    return CR_OK;
}

cr_status check_ctx(cr_ctx *ctx) {
    if (!ctx) return CR_ERR_INVALID_ARG;
    if (ctx->poisoned) return CR_ERR_STATE;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return fail(ctx, CR_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    return CR_OK;
}

void drop_graphs(cr_ctx *ctx) {
    for (auto &g : ctx->graph)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    for (auto &g : ctx->graph_multi)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    for (auto &g : ctx->graph_ad)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
}

// kMultiIters (even: the buffer roles repeat with period 2, so the graph starts and ends in the
// same assignment) constant-step iterations in one graph: the PDL chain then also spans the
// iteration boundaries and the host launches one graph per kMultiIters iterations.
constexpr int kMultiIters = 8;

cr_status build_graph_multi(cr_ctx *ctx, int key) {
    cudaGraph_t g = nullptr;
    const int bA = ctx->bA, bB = ctx->bB;
    const int64_t k = ctx->k, launches = ctx->launches;
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->cap_stream;
    cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        ctx->stream = user;
        return fail(ctx, CR_ERR_CUDA, "cudaStreamBeginCapture: %s", cudaGetErrorString(e));
    }
    cr_status st = CR_OK;
    const bool fuse = can_fuse(ctx);
    for (int i = 0; i < kMultiIters && st == CR_OK; ++i) {
        const int bo = ctx->bB;
        const int mode = !fuse ? FUSE_NONE : i == 0 ? FUSE_FIRST : i == kMultiIters - 1 ? FUSE_LAST : FUSE_MID;
        st = enqueue_step(ctx, false, bo, 1.0 / ctx->L, true, false, nullptr, mode);
        advance_host(ctx, bo);
    }
    e = cudaStreamEndCapture(ctx->stream, &g);
    ctx->stream = user;
    ctx->multi_launches = ctx->launches - launches;
    ctx->bA = bA; ctx->bB = bB; ctx->k = k; ctx->launches = launches;
    if (st != CR_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (e != cudaSuccess) return fail(ctx, CR_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&ctx->graph_multi[key], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(ctx, CR_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
    return CR_OK;
}

cr_status build_graph(cr_ctx *ctx, int key) {
    // key = 3 bA + bB at capture time; capture one constant-step iteration, restore host state
    cudaGraph_t g = nullptr;
    const int bA = ctx->bA, bB = ctx->bB;
    const int64_t k = ctx->k, launches = ctx->launches;
    // The caller's stream may be the legacy default stream, which cannot be captured: record
    // on a private stream, replay on the caller's stream (cudaGraphLaunch(..., ctx->stream)).
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->cap_stream;
    cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        ctx->stream = user;
        return fail(ctx, CR_ERR_CUDA, "cudaStreamBeginCapture: %s", cudaGetErrorString(e));
    }
    cr_status st = enqueue_step(ctx, false, bB, 1.0 / ctx->L, true, false);
    e = cudaStreamEndCapture(ctx->stream, &g);
    ctx->stream = user;
    ctx->bA = bA; ctx->bB = bB; ctx->k = k; ctx->launches = launches;
    if (st != CR_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (e != cudaSuccess) return fail(ctx, CR_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&ctx->graph[key], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(ctx, CR_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
    return CR_OK;
}

// Instantiate every constant-step graph cr_solve may replay -- the 8-iteration and the
// 1-iteration graph of both buffer-role assignments -- on first use, so no later cr_solve call
// (e.g. a timed one after a short warm-up) pays a capture.
cr_status prebuild_graphs(cr_ctx *ctx) {
    const int bA = ctx->bA, bB = ctx->bB;
    for (int swap = 0; swap < 2; ++swap) {
        ctx->bA = swap ? bB : bA;
        ctx->bB = swap ? bA : bB;
        const int key = 3 * ctx->bA + ctx->bB;
        cr_status st = CR_OK;
        if (!ctx->graph_multi[key]) st = build_graph_multi(ctx, key);
        if (st == CR_OK && !ctx->graph[key]) st = build_graph(ctx, key);
        ctx->bA = bA;
        ctx->bB = bB;
        if (st != CR_OK) return st;
    }
    return CR_OK;
}

// K constant-step iterations with the SMEM-resident solver (small N, world 1); the state is
// left exactly as K graph replays of the streaming path would leave it.
cr_status enqueue_resident(cr_ctx *ctx, int64_t K) {
    const Layout &Ly = ctx->lay;
    ResidentParams p{};
    p.N = Ly.N;
    p.ldT = Ly.ldT;
    p.K = K;
    p.n = Ly.n;
    p.R = ctx->res_R;
    p.ldS = ctx->res_ldS;
    p.G = ctx->res_G;
    p.TA = ctx->th[ctx->bA];
    p.TB = ctx->th[ctx->bB];
    p.rA = ctx->r[ctx->bA]; p.cA = ctx->c[ctx->bA]; p.PA = ctx->P[ctx->bA];
    p.rB = ctx->r[ctx->bB]; p.cB = ctx->c[ctx->bB]; p.PB = ctx->P[ctx->bB];
    p.X64 = ctx->at<double>(Ly.X64);
    p.ybar = ctx->at<double>(Ly.ybar);
    p.gamma = ctx->gamma;
    p.L = ctx->L;
    p.ts = ctx->at<DevScalars>(Ly.ts);
    p.yg = ctx->at<double>(Ly.yg);
    p.y64 = ctx->at<double>(Ly.y64);
    p.a64 = ctx->at<double>(Ly.a64);
    p.Xi64 = ctx->at<double>(Ly.Xi64);
    p.cpart = ctx->at<double>(Ly.cpart);
    p.trace = ctx->trace;                 // CR_TC_TRACE debug buffer (also sized for this)
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->timing) {
        e0 = next_event(ctx);
        e1 = next_event(ctx);
        if (!e0 || !e1) return fail(ctx, CR_ERR_CUDA, "cudaEventCreate failed");
        CK(cudaEventRecord(e0, ctx->stream));
    }
    CK(launch_resident(p, Ly.fp64, ctx->stream));
    ctx->launches += 1;
    if (ctx->trace) {   // debug: dump the phase timeline of CTA 0
        std::vector<unsigned long long> h(16 * 8);
        CK(cudaMemcpyAsync(h.data(), ctx->trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (FILE *f = std::fopen(std::getenv("CR_TC_TRACE"), "wb")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    if (e1) {
        CK(cudaEventRecord(e1, ctx->stream));
        ctx->ev_iters += K;
    }
    for (int64_t i = 0; i < K; ++i) advance_host(ctx, ctx->bB);
    return CR_OK;
}

bool use_resident(const cr_ctx *ctx) {
    return ctx->res_G > 0 && ctx->rule == CR_STEP_CONSTANT && !ctx->coll && ctx->world == 1 &&
           !std::getenv("CR_NO_RESIDENT");
}

}  // namespace

// =============================================================================== ABI
extern "C" {

const char *cr_status_string(cr_status s) {
    switch (s) {
        case CR_OK: return "CR_OK";
        case CR_ERR_INVALID_ARG: return "CR_ERR_INVALID_ARG";
        case CR_ERR_CUDA: return "CR_ERR_CUDA";
        case CR_ERR_NCCL: return "CR_ERR_NCCL";
        case CR_ERR_OOM: return "CR_ERR_OOM";
        case CR_ERR_STATE: return "CR_ERR_STATE";
        case CR_ERR_UNSUPPORTED: return "CR_ERR_UNSUPPORTED";
    }
    return "CR_ERR_UNKNOWN";
}

const char *cr_last_error(const cr_ctx *ctx) { return ctx ? ctx->err.c_str() : ""; }

int32_t cr_max_dim(void) { return 80; }

cr_status cr_local_group_create(int32_t world, cr_group **out) {
    if (!out) return CR_ERR_INVALID_ARG;
    *out = reinterpret_cast<cr_group *>(local_group_create(world));
    return *out ? CR_OK : CR_ERR_INVALID_ARG;
}

void cr_local_group_destroy(cr_group *g) { local_group_destroy(reinterpret_cast<LocalGroup *>(g)); }

cr_status cr_nccl_get_unique_id(void *out) {
    if (!out) return CR_ERR_INVALID_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return CR_ERR_NCCL;
    std::memcpy(out, &id, sizeof id);
    return CR_OK;
}

uint64_t cr_tc_check_word(cr_ctx *ctx) {
    if (!ctx || !ctx->tc_check) return 0;
    unsigned long long w = 0;
    if (cudaMemcpyAsync(&w, ctx->tc_check, sizeof w, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return ~0ULL;
    return w;
}

int64_t cr_shard_rows(int64_t N, int32_t world, int64_t nbar) {
    if (N < 1 || world < 1) return 0;
    return shard_rows(N, world, std::max<int64_t>(nbar, 1));
}

size_t cr_workspace_size(int64_t N, int32_t n, cr_precision prec, cr_kernel kernel, int32_t rank,
                         int32_t world, int32_t flags) {
    return cr_workspace_size_ex(N, n, prec, kernel, rank, world, flags, 1);
}

size_t cr_workspace_size_ex(int64_t N, int32_t n, cr_precision prec, cr_kernel kernel, int32_t rank,
                            int32_t world, int32_t flags, int64_t nbar) {
    Layout L;
    if (!make_layout(N, n, prec, kernel, rank, world, flags, nbar, &L)) return 0;
    return L.total;
}

cr_status cr_lipschitz_host(int64_t N, int32_t n, const double *X, double gamma, double *L_out) {
    if (N < 2 || n < 1 || !X || !L_out || !(gamma > 0.0) || !std::isfinite(gamma)) return CR_ERR_INVALID_ARG;
    const double s2 = sigma_max_sq_lanczos(N, n, X, 1e-13, 2000);
    if (!(s2 > 0.0) || !std::isfinite(s2)) return CR_ERR_INVALID_ARG;
    *L_out = s2 / gamma;
    return CR_OK;
}

static cr_status p2p_setup(cr_ctx *ctx);   // CR_FLAG_P2P (below)

cr_status cr_init(const cr_config *cfg, cr_ctx **out) {
    if (!out) return CR_ERR_INVALID_ARG;
    *out = nullptr;
    if (!cfg || !cfg->X || !cfg->ybar || cfg->N < 2 || cfg->n < 1) return CR_ERR_INVALID_ARG;
    if (!(cfg->gamma > 0.0) || !std::isfinite(cfg->gamma) || !(cfg->L >= 0.0) || !std::isfinite(cfg->L))
        return CR_ERR_INVALID_ARG;
    if (cfg->L == 0.0 && cfg->gamma > 1.0) return CR_ERR_INVALID_ARG;  // sigma^2/gamma bounds only for gamma<=1
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return CR_ERR_INVALID_ARG;
    if (cfg->world > 1 && !cfg->nccl_unique_id && !cfg->local_group) return CR_ERR_INVALID_ARG;
    if (cfg->local_group && local_group_world(reinterpret_cast<const LocalGroup *>(cfg->local_group)) != cfg->world)
        return CR_ERR_INVALID_ARG;
    if (cfg->prec != CR_FP32 && cfg->prec != CR_FP64) return CR_ERR_INVALID_ARG;
    if (cfg->prec == CR_FP64 && cfg->kernel == CR_KERNEL_TC) return CR_ERR_UNSUPPORTED;
    if (cfg->n > cr_max_dim()) return CR_ERR_UNSUPPORTED;
    const int64_t N = cfg->N;
    const int n = cfg->n;
    for (int64_t i = 0; i < N * n; ++i)
        if (!std::isfinite(cfg->X[i])) return CR_ERR_INVALID_ARG;
    for (int64_t i = 0; i < N; ++i)
        if (!std::isfinite(cfg->ybar[i])) return CR_ERR_INVALID_ARG;

    cr_ctx *ctx = new (std::nothrow) cr_ctx();
    if (!ctx) return CR_ERR_OOM;
    ctx->prec = cfg->prec;
    ctx->kernel = use_tc(cfg->n, cfg->prec, cfg->kernel) ? CR_KERNEL_TC : CR_KERNEL_SIMT;
    ctx->gamma = cfg->gamma;
    ctx->rank = cfg->rank;
    ctx->world = cfg->world;
    ctx->device = cfg->device;
    ctx->stream = static_cast<cudaStream_t>(cfg->stream);
    if (!make_layout(N, n, cfg->prec, cfg->kernel, cfg->rank, cfg->world, cfg->flags, cfg->nbar, &ctx->lay)) {
        delete ctx;
        return CR_ERR_UNSUPPORTED;
    }
    const Layout &Ly = ctx->lay;
    auto bail = [&](cr_status s) { cr_destroy(ctx); return s; };
    if (!cfg->workspace || cfg->workspace_bytes < Ly.total || (reinterpret_cast<uintptr_t>(cfg->workspace) & 255))
        return bail(CR_ERR_INVALID_ARG);
    ctx->ws = static_cast<char *>(cfg->workspace);
    if (cudaSetDevice(ctx->device) != cudaSuccess) return bail(CR_ERR_CUDA);

    // step constant (Eq. (lischitz))
    if (cfg->L > 0.0) ctx->L = cfg->L;      // else: device Lanczos once X is on the device (below)

    for (int b = 0; b < Ly.nbuf; ++b) ctx->th[b] = ctx->ws + Ly.th[b];
    for (int s = 0; s < Ly.nbuf; ++s) {
        ctx->r[s] = ctx->at<double>(Ly.r[s]);
        ctx->c[s] = ctx->at<double>(Ly.c[s]);
        ctx->P[s] = ctx->at<double>(Ly.P[s]);
    }
    cudaError_t e;
#define IK(call)                                                                                   \
    do {                                                                                           \
        e = (call);                                                                                \
        if (e != cudaSuccess) {                                                                    \
            fail(ctx, CR_ERR_CUDA, "cr_init %s: %s", #call, cudaGetErrorString(e));              \
            std::fprintf(stderr, "libcr: %s\n", ctx->err.c_str());                                 \
            return bail(CR_ERR_CUDA);                                                              \
        }                                                                                          \
    } while (0)
    // CR_INIT_PROF=1: host-synchronous phase timings of cr_init on stderr (diagnostics)
    const bool iprof = std::getenv("CR_INIT_PROF") != nullptr;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto t_prev = tnow();
    auto mark = [&](const char *what) {
        if (!iprof) return;
        cudaStreamSynchronize(ctx->stream);
        const auto t = tnow();
        std::fprintf(stderr, "cr_init %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_prev).count());
        t_prev = t;
    };
    mark("enter");
    IK(cudaMemsetAsync(ctx->ws, 0, Ly.total, ctx->stream));
    mark("memset");
    if (Ly.nbar > 1) IK(block_ipm_prepare(Ly.ipm_smem));
    IK(cudaMemcpyAsync(ctx->ws + Ly.X64, cfg->X, (size_t)N * n * 8, cudaMemcpyHostToDevice, ctx->stream));
    IK(cudaMemcpyAsync(ctx->ws + Ly.ybar, cfg->ybar, (size_t)N * 8, cudaMemcpyHostToDevice, ctx->stream));
    mark("h2d");
    if (!(cfg->L > 0.0)) {
        // L = sigma_max(C)^2 / gamma by the device Lanczos (the host cr_lipschitz_host computes
        // the same iteration; fixed-order reductions, so every rank gets the same L)
        // Small problems (C1-sized) take the host iteration: ~50 Lanczos steps of O(N n^2) host
        // work beat ~100 device round trips; deterministic either way.
        cudaError_t le = cudaSuccess;
        const bool host = (int64_t)N * (n + 1) <= kLanczosHostMax;
        // device scratch: the Theta buffers (contiguous, not used yet; re-zeroed below)
        const size_t th_bytes = (size_t)Ly.nbuf * Ly.Rp * Ly.ldT * Ly.es;
        const double s2 = host ? sigma_max_sq_lanczos(N, n, cfg->X, 1e-13, 2000)
                               : sigma_max_sq_lanczos_device(N, n, ctx->at<double>(Ly.X64), 1e-13, 2000, ctx->stream, &le,
                                                             ctx->ws + Ly.th[0], th_bytes);
        if (!host) IK(cudaMemsetAsync(ctx->ws + Ly.th[0], 0, th_bytes, ctx->stream));
        if (le != cudaSuccess) {
            fail(ctx, CR_ERR_CUDA, "cr_init Lanczos: %s", cudaGetErrorString(le));
            return bail(CR_ERR_CUDA);
        }
        if (!(s2 > 0.0) || !std::isfinite(s2)) return bail(CR_ERR_INVALID_ARG);
        ctx->L = s2 / cfg->gamma;
    }
    ctx->sigma2 = ctx->L * cfg->gamma;
    mark("lanczos");
    IK(launch_fill_inputs(ctx->at<double>(Ly.X64), N, n, Ly.NB, Ly.NBP, Ly.ldT, Ly.fp64, ctx->ws + Ly.XT,
                          ctx->ws + Ly.Xh, ctx->stream));
    IK(launch_transpose_pad(ctx->at<double>(Ly.X64), N, n, Ly.nP, Ly.ldT, ctx->at<double>(Ly.XT64), ctx->stream));
    ctx->launches += 2;
    DevScalars h{};
    h.t_prev = 1.0;   // beta_0 = 0: theta~^1 = theta^0
    h.t_cur = 1.0;    // t_1 = 1
    IK(cudaMemcpyAsync(ctx->ws + Ly.ts, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));

    // SIMT fused-pass grid (also used for the read-only sums pass of cr_set_theta): one full
    // wave of resident CTAs, contiguous tile ranges
    int smem = 0, bps = 0, nsm = 0;
    IK(pass_simt_config(Ly.fp64, Ly.NB, &smem, &bps));
    IK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
    ctx->nCB = (int)((N + kBN - 1) / kBN);
    ctx->T = (int64_t)Ly.nRB * ctx->nCB;
    ctx->G = (int)std::min<int64_t>({ctx->T, (int64_t)std::max(bps, 1) * nsm, (int64_t)kGMax});
    std::vector<int> slot0, rb_ptr, slots, slot0t, rb_ptrt, slotst;
    slot_tables(ctx->G, ctx->T, Ly.nRB, ctx->nCB, slot0, rb_ptr, slots);
    IK(cudaMemcpyAsync(ctx->ws + Ly.slot0, slot0.data(), slot0.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    IK(cudaMemcpyAsync(ctx->ws + Ly.rb_ptr, rb_ptr.data(), rb_ptr.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    IK(cudaMemcpyAsync(ctx->ws + Ly.rb_slots, slots.data(), slots.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    if (Ly.tc) {
        // tcgen05 pass: one persistent CTA per SM (512 TMEM columns, ~200 KB smem each)
        ctx->T_tc = (int64_t)Ly.nRBtc * Ly.nCBtc;
        ctx->G_tc = (int)std::min<int64_t>({ctx->T_tc, (int64_t)nsm, (int64_t)kGMax});
        // Theta ring: 32 KB slots (B1, B2 tiles, 1024-B aligned for the 128-B swizzle); X_J and
        // X_J^T image rings (hi + lo per slot).  Defaults: 5 Theta slots and 3 + 3 image slots,
        // reduced (images first, not below 2, then Theta slots) until they fit: C4 5/3/2, C5 4/2/2.
        // CR_TC_STAGES / CR_TC_G1STAGES / CR_TC_G2STAGES override.
        // GEMM1 passes (TcParams::g1passes): 3 by default; CR_TC_G1PASSES=2 drops Xi_hi X_lo
        ctx->g1passes = 3;
        if (const char *e = std::getenv("CR_TC_G1PASSES")) ctx->g1passes = std::atoi(e) == 2 ? 2 : 3;
        // GEMM1 in kind::f16 (TcParams::g1f16) for n > 56: there the X_J images' shared memory
        // limits the Theta ring (fp16 halves them: 5 slots instead of 4 at n = 80) and the tensor
        // work drives the power cap; measured C5 0.70 -> 0.78 of the copy peak, C4 (n = 40) 0.90 ->
        // 0.88, C3 0.64 -> 0.60 -- so kind::tf32 below.  CR_TC_G1_F16 / CR_TC_G1_TF32 override.  X
        // is scaled by 2^xexp so its largest |x| sits just below 2^14 (fp16 range, exact scaling)
        ctx->g1f16 = Ly.NK > 56 ? 1 : 0;
        if (std::getenv("CR_TC_G1_F16")) ctx->g1f16 = 1;
        if (std::getenv("CR_TC_G1_TF32")) ctx->g1f16 = 0;
        {
            double mx = 0.0;
            for (int64_t e = 0; e < N * (int64_t)n; ++e) mx = std::max(mx, std::fabs(cfg->X[e]));
            int E = 0;
            if (mx > 0.0) std::frexp(mx, &E);
            ctx->xexp = mx > 0.0 ? 14 - E : 0;
        }
        const int NK16 = Ly.NP2;
        if (const char *e = std::getenv("CR_TC_G1_RUNAHEAD")) ctx->g1_runahead = std::atoi(e) != 0;
        if (std::getenv("CR_TC_CHECK")) {
            IK(cudaMalloc(&ctx->tc_check, sizeof(unsigned long long)));
            IK(cudaMemsetAsync(ctx->tc_check, 0, sizeof(unsigned long long), ctx->stream));
        }
        const size_t tb = 2 * (size_t)kTcBM * kTcBN * 4, b2 = 2 * (size_t)Ly.NP2 * 128;
        const size_t b1 = (ctx->g1passes == 3 ? 2 : 1) * (ctx->g1f16 ? (size_t)NK16 * 64 : (size_t)Ly.NK * 128);
        const size_t fixed = tc_barrier_bytes() + 1024 + 64;
        const size_t budget = 227 * 1024 - fixed;
        auto env_int = [](const char *k, int d, int lo) {
            const char *e = std::getenv(k);
            return e ? std::max(lo, std::min(kTcMaxStages, std::atoi(e))) : d;
        };
        int st = env_int("CR_TC_STAGES", 5, 2), s1 = env_int("CR_TC_G1STAGES", 3, 1),
            s2 = env_int("CR_TC_G2STAGES", 3, 1);
        auto bytes = [&]() { return st * tb + s1 * b1 + s2 * b2; };
        while (bytes() > budget && (s1 > 2 || s2 > 2)) {
            if (s1 * b1 >= s2 * b2 && s1 > 2) --s1;
            else if (s2 > 2) --s2;
            else --s1;
        }
        while (bytes() > budget && st > 2) --st;
        // GEMM1 run-ahead drops the in-order guard GEMM1's own Theta wait gives the epilogue: an
        // epilogue warpgroup at tile u then relies on its parity wait on slot u % S alone, and with
        // an odd S the slot's previous tile u - S belongs to the OTHER warpgroup, which may still be
        // pending -- the wait would match the phase of tile u - 2S and read a slot being refilled
        // (the round-1 fault with 3 slots).  With S even the previous tile is the warpgroup's own.
        if (ctx->g1_runahead && (st & 1)) --st;
        if (bytes() > budget) {
            fail(ctx, CR_ERR_UNSUPPORTED, "tc pass: smem");
            return bail(CR_ERR_UNSUPPORTED);
        }
        ctx->stages = st;
        ctx->g1stages = s1;
        ctx->g2stages = s2;
        ctx->smem_tc = (int)(bytes() + fixed);
        IK(pass_tc_prepare(Ly.NK, ctx->smem_tc));
        slot_tables(ctx->G_tc, ctx->T_tc, Ly.nRBtc, Ly.nCBtc, slot0t, rb_ptrt, slotst);
        IK(cudaMemcpyAsync(ctx->ws + Ly.slot0_tc, slot0t.data(), slot0t.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
        IK(cudaMemcpyAsync(ctx->ws + Ly.rb_ptr_tc, rb_ptrt.data(), rb_ptrt.size() * 4, cudaMemcpyHostToDevice,
                           ctx->stream));
        IK(cudaMemcpyAsync(ctx->ws + Ly.rb_slots_tc, slotst.data(), slotst.size() * 4, cudaMemcpyHostToDevice,
                           ctx->stream));
        IK(launch_tc_images(ctx->at<double>(Ly.X64), N, n, Ly.NK, Ly.NP2, Ly.nCBtc, ctx->at<float>(Ly.g1h),
                            ctx->at<float>(Ly.g1l), ctx->at<float>(Ly.g2h), ctx->at<float>(Ly.g2l), ctx->g1f16,
                            ctx->xexp, ctx->stream));
        ctx->launches += 1;
    }
    if (std::getenv("CR_TC_TRACE")) {     // debug timelines (tcgen05 pass / resident solver)
        IK(cudaMalloc(&ctx->trace, kTraceWords * 8));
        IK(cudaMemsetAsync(ctx->trace, 0, kTraceWords * 8, ctx->stream));
    }
    if (Ly.resident) {
        // SMEM-resident solver geometry: enough CTAs that one iteration's N^2 n work is spread
        // (~64K pair-features per CTA), at most one per SM (cooperative launch: co-resident),
        // more if the rows do not fit in shared memory; unusable if even nsm CTAs do not fit
        int coop = 0;
        IK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device));
        const int64_t work = N * N * (int64_t)n;
        int G = (int)std::min<int64_t>({(int64_t)nsm, (int64_t)kResidentMaxCTAs, std::max<int64_t>(1, (work + 65535) / 65536)});
        for (; coop && G <= std::min(nsm, kResidentMaxCTAs); ++G) {
            ResidentParams rp{};
            rp.N = N;
            rp.n = n;
            rp.R = (int)((N + G - 1) / G);
            rp.ldS = (int)((N + 3) / 4 * 4);
            if (resident_smem_bytes(rp, Ly.fp64) <= (size_t)(226 * 1024)) {
                ctx->res_R = rp.R;
                ctx->res_G = (int)((N + rp.R - 1) / rp.R);
                ctx->res_ldS = rp.ldS;
                break;
            }
        }
    }
    IK(cudaStreamSynchronize(ctx->stream));   // host vectors go out of scope
    mark("setup");
#undef IK
    ctx->comm.rank = ctx->rank;
    ctx->comm.world = ctx->world;
    // CR_FORCE_NCCL (tests): a single rank still runs every collective through a 1-rank NCCL
    // communicator -- exercises the NCCL calls, their in-place conventions and graph capture
    const bool force = ctx->world == 1 && std::getenv("CR_FORCE_NCCL") && !cfg->local_group;
    ctx->coll = ctx->world > 1 || force;
    if (ctx->world > 1 && cfg->local_group) {
        ctx->comm.local = reinterpret_cast<LocalGroup *>(cfg->local_group);
    } else if (ctx->coll) {
        ncclUniqueId id;
        if (force) {
            if (ncclGetUniqueId(&id) != ncclSuccess) return bail(CR_ERR_NCCL);
        } else {
            std::memcpy(&id, cfg->nccl_unique_id, sizeof id);
        }
        ncclResult_t r = ncclCommInitRank(&ctx->comm.nccl, ctx->world, id, ctx->rank);
        if (r != ncclSuccess) {
            fail(ctx, CR_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
            return bail(CR_ERR_NCCL);
        }
    }
    if (cfg->flags & CR_FLAG_P2P) {
        cr_status st = p2p_setup(ctx);
        if (st != CR_OK) return bail(st);
    }
    *out = ctx;
    return CR_OK;
}

// CR_FLAG_P2P: this rank's receive slab [W][S] + arrival flags [W] + epoch in one cudaMalloc
// (IPC-exportable), the handles exchanged once over the NCCL communicator and the peers' slabs
// mapped (cudaIpcOpenMemHandle, NVLink peer access); the device table lists every rank's slab
// and flags.  NCCL mode only; S must be a multiple of the column-sum block.
static cr_status p2p_setup(cr_ctx *ctx) {
    const Layout &Ly = ctx->lay;
    const int W = ctx->world;
    if (!ctx->coll || ctx->comm.local || !ctx->comm.nccl)
        return fail(ctx, CR_ERR_UNSUPPORTED, "CR_FLAG_P2P needs the NCCL path (world > 1, or CR_FORCE_NCCL)");
    if (W > kP2PTab || Ly.S % reduce_col_block(Ly.fp64))
        return fail(ctx, CR_ERR_UNSUPPORTED, "CR_FLAG_P2P: world <= %d and shard rows %% %d == 0 required", kP2PTab,
                    reduce_col_block(Ly.fp64));
    const size_t cbytes = ((size_t)W * Ly.S + W + 1) * 8;          // c slab, c flags, c epoch
    ctx->p2p_yf = cbytes;                                            // y flags [W], y epoch
    ctx->p2p_yr = (cbytes + ((size_t)W + 1) * 8 + 255) / 256 * 256;  // y' receive [W S]
    const size_t bytes = ctx->p2p_yr + (size_t)W * Ly.S * Ly.es;
    CK(cudaMalloc(&ctx->p2p_buf, bytes));
    CK(cudaMemsetAsync(ctx->p2p_buf, 0, bytes, ctx->stream));      // ordered before the exchange below
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMalloc(&ctx->p2p_tab, 4 * kP2PTab * sizeof(void *)));
    std::vector<void *> base(W, nullptr);
    base[ctx->rank] = ctx->p2p_buf;
    if (W > 1) {
        cudaIpcMemHandle_t h{};
        CK(cudaIpcGetMemHandle(&h, ctx->p2p_buf));
        char *dev = nullptr;
        CK(cudaMalloc(&dev, (size_t)W * sizeof h));
        CK(cudaMemcpy(dev + (size_t)ctx->rank * sizeof h, &h, sizeof h, cudaMemcpyHostToDevice));
        ncclResult_t r = ncclAllGather(dev + (size_t)ctx->rank * sizeof h, dev, sizeof h, ncclChar, ctx->comm.nccl,
                                       ctx->stream);
        if (r != ncclSuccess) {
            cudaFree(dev);
            return fail(ctx, CR_ERR_NCCL, "CR_FLAG_P2P handle exchange: %s", ncclGetErrorString(r));
        }
        std::vector<cudaIpcMemHandle_t> all(W);
        CK(cudaMemcpyAsync(all.data(), dev, (size_t)W * sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        cudaFree(dev);
        for (int q = 0; q < W; ++q) {
            if (q == ctx->rank) continue;
            void *ptr = nullptr;
            CK(cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess));
            ctx->p2p_opened.push_back(ptr);
            base[q] = ptr;
        }
    }
    void *tab[4 * kP2PTab] = {};
    for (int q = 0; q < W; ++q) {
        char *b = static_cast<char *>(base[q]);
        tab[q] = b;                                                  // c slab
        tab[kP2PTab + q] = b + (size_t)W * Ly.S * 8;                 // c flags
        tab[2 * kP2PTab + q] = b + ctx->p2p_yr;                      // y' receive
        tab[3 * kP2PTab + q] = b + ctx->p2p_yf;                      // y flags
    }
    CK(cudaMemcpy(ctx->p2p_tab, tab, sizeof tab, cudaMemcpyHostToDevice));
    ctx->p2p = true;
    return CR_OK;
}

cr_status cr_set_theta(cr_ctx *ctx, const double *tk1, const double *tk2, double t_km1, double t_k) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    const Layout &Ly = ctx->lay;
    if (!(t_km1 >= 1.0) || !(t_k >= 1.0) || !std::isfinite(t_km1) || !std::isfinite(t_k))
        return fail(ctx, CR_ERR_INVALID_ARG, "t_{k-1}, t_k must be finite and >= 1");
    const double *src[2] = {tk1, tk2};
    for (int b = 0; b < 2; ++b) {
        if (!src[b]) continue;
        int bad_sign = 0, bad_diag = 0;      // host validation, rows in parallel (full-size C5: 2 x 4.3e9)
#pragma omp parallel for schedule(static) reduction(| : bad_sign, bad_diag)
        for (int64_t i = 0; i < Ly.Ns; ++i) {
            const double *row = src[b] + i * Ly.N;
            const int64_t blk = (Ly.row0 + i) / Ly.nbar;
            for (int64_t j = 0; j < Ly.N; ++j) {
                const double v = row[j];
                if (!(v >= 0.0) || !std::isfinite(v)) bad_sign = 1;
                if (j / Ly.nbar == blk && v != 0.0) bad_diag = 1;
            }
        }
        if (bad_sign) return fail(ctx, CR_ERR_INVALID_ARG, "Theta entries must be finite and >= 0");
        if (bad_diag) return fail(ctx, CR_ERR_INVALID_ARG, "Theta must be 0 on the diagonal / intra-block pairs");
    }
    drop_graphs(ctx);
    for (int b = 0; b < 2; ++b) {
        CK(cudaMemsetAsync(ctx->th[b], 0, (size_t)Ly.Rp * Ly.ldT * Ly.es, ctx->stream));
        if (src[b] && Ly.Ns > 0 && Ly.tc) {
            // tile-major fp32 image of this rank's rows (theta_off), zero padding, one copy
            const size_t tiles = (size_t)Ly.nRBtc * Ly.nCBtc;
            std::vector<float> tmp(tiles * (size_t)kTcBM * kTcBN, 0.f);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < Ly.Ns; ++i)
                for (int64_t j = 0; j < Ly.N; ++j)
                    tmp[(size_t)theta_off(i, j, Ly.ldT, 1, Ly.nCBtc)] = (float)src[b][i * Ly.N + j];
            CK(cudaMemcpyAsync(ctx->th[b], tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
        } else if (src[b] && Ly.Ns > 0) {
            if (Ly.fp64) {
                CK(cudaMemcpy2DAsync(ctx->th[b], Ly.ldT * 8, src[b], Ly.N * 8, Ly.N * 8, Ly.Ns,
                                     cudaMemcpyHostToDevice, ctx->stream));
            } else {
                std::vector<float> tmp((size_t)Ly.Ns * Ly.N);
#pragma omp parallel for schedule(static)
                for (int64_t e = 0; e < (int64_t)tmp.size(); ++e) tmp[e] = (float)src[b][e];
                CK(cudaMemcpy2DAsync(ctx->th[b], Ly.ldT * 4, tmp.data(), Ly.N * 4, Ly.N * 4, Ly.Ns,
                                     cudaMemcpyHostToDevice, ctx->stream));
                CK(cudaStreamSynchronize(ctx->stream));
            }
        }
    }
    ctx->bA = 0;
    ctx->bB = 1;
    st = enqueue_sums(ctx, 0, 0);
    if (st != CR_OK) return st;
    st = enqueue_sums(ctx, 1, 1);
    if (st != CR_OK) return st;
    DevScalars h{};
    h.t_prev = t_km1;
    h.t_cur = t_k;
    CK(cudaMemcpyAsync(ctx->ws + Ly.ts, &h, 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CR_OK;
}

static cr_status read_buffer(cr_ctx *ctx, int b, int64_t row0, int64_t nrows, double *out) {
    const Layout &Ly = ctx->lay;
    if (nrows <= 0) return CR_OK;
    if (Ly.tc) {
        // tile-major: the row blocks covering the rows are contiguous (row-block-major tiles)
        const int64_t rb0 = row0 / kTcBM, rb1 = (row0 + nrows - 1) / kTcBM;
        const size_t per_rb = (size_t)Ly.nCBtc * kTcBM * kTcBN;
        std::vector<float> tmp((size_t)(rb1 - rb0 + 1) * per_rb);
        CK(cudaMemcpyAsync(tmp.data(), static_cast<const float *>(ctx->th[b]) + rb0 * per_rb, tmp.size() * 4,
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < nrows; ++i)
            for (int64_t j = 0; j < Ly.N; ++j)
                out[i * Ly.N + j] = tmp[(size_t)theta_off(row0 + i - rb0 * kTcBM, j, Ly.ldT, 1, Ly.nCBtc)];
        return CR_OK;
    }
    const char *src = static_cast<const char *>(ctx->th[b]) + (size_t)row0 * Ly.ldT * Ly.es;
    if (Ly.fp64) {
        CK(cudaMemcpy2DAsync(out, Ly.N * 8, src, Ly.ldT * 8, Ly.N * 8, nrows, cudaMemcpyDeviceToHost,
                             ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    } else {
        std::vector<float> tmp((size_t)nrows * Ly.N);
        CK(cudaMemcpy2DAsync(tmp.data(), Ly.N * 4, src, Ly.ldT * 4, Ly.N * 4, nrows, cudaMemcpyDeviceToHost,
                             ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (size_t e = 0; e < tmp.size(); ++e) out[e] = tmp[e];
    }
    return CR_OK;
}

cr_status cr_get_theta(cr_ctx *ctx, double *theta_k, double *theta_km1, double *t_k, double *t_kp1) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    const Layout &Ly = ctx->lay;
    if (theta_k && (st = read_buffer(ctx, ctx->bA, 0, Ly.Ns, theta_k)) != CR_OK) return st;
    if (theta_km1 && (st = read_buffer(ctx, ctx->bB, 0, Ly.Ns, theta_km1)) != CR_OK) return st;
    double t[2];
    CK(cudaMemcpyAsync(t, ctx->ws + Ly.ts, sizeof t, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (t_k) *t_k = t[0];
    if (t_kp1) *t_kp1 = t[1];
    return CR_OK;
}

cr_status cr_get_theta_rows(cr_ctx *ctx, int32_t which, int64_t row0, int64_t nrows, double *out) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    const Layout &Ly = ctx->lay;
    if ((which != 0 && which != 1) || row0 < 0 || nrows < 0 || row0 + nrows > Ly.Ns || (!out && nrows))
        return fail(ctx, CR_ERR_INVALID_ARG, "cr_get_theta_rows: bad range");
    return read_buffer(ctx, which == 0 ? ctx->bA : ctx->bB, row0, nrows, out);
}

cr_status cr_dual_step(cr_ctx *ctx, cr_step_stats *out) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (ctx->rule == CR_STEP_ADAPTIVE) {
        if ((st = adaptive_step(ctx)) != CR_OK) return st;
        if (out) return eval_stats(ctx, out);
        return CR_OK;
    }
    const int bo = ctx->bB;
    if ((st = enqueue_step(ctx, true, bo, 1.0 / ctx->L, true, false)) != CR_OK) return st;
    if (ctx->trace) {   // debug: dump the tensor-core pass timeline of CTA 0
        std::vector<unsigned long long> h(kTraceWords);
        CK(cudaMemcpyAsync(h.data(), ctx->trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (FILE *f = std::fopen(std::getenv("CR_TC_TRACE"), "wb")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    advance_host(ctx, bo);
    if (out) return eval_stats(ctx, out);
    return CR_OK;
}

cr_status cr_solve(cr_ctx *ctx, int64_t max_iters, const cr_stop *stop, cr_report *out) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (max_iters < 0 || (stop && stop->report_every < 1))
        return fail(ctx, CR_ERR_INVALID_ARG, "cr_solve: bad arguments");
    if (out) std::memset(out, 0, sizeof *out);
    // no graphs with the in-process local group: its collectives are host rendezvous
    const bool use_graph = !ctx->timing && !ctx->comm.local;
    int64_t ttot0 = 0;                      // adaptive trials so far (launch accounting of the graph path)
    if (ctx->rule == CR_STEP_ADAPTIVE && use_adaptive_graph(ctx)) {
        double v = 0.0;
        CK(cudaMemcpyAsync(&v, &ctx->at<DevScalars>(ctx->lay.ts)->ad[AD_TTOT], sizeof v, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ttot0 = (int64_t)v;
    }
    const double Nd = (double)ctx->lay.N;
    if (use_graph && max_iters > 0 && ctx->rule == CR_STEP_CONSTANT && !use_resident(ctx) &&
        (st = prebuild_graphs(ctx)) != CR_OK)
        return st;
    int64_t it = 0;
    while (it < max_iters) {
        if (use_resident(ctx)) {
            // one cooperative launch for the whole chunk (to the next stop test, or the end)
            int64_t chunk = max_iters - it;
            if (stop) chunk = std::min<int64_t>(chunk, stop->report_every - it % stop->report_every);
            if ((st = enqueue_resident(ctx, chunk)) != CR_OK) return st;
            it += chunk - 1;
        } else if (ctx->rule == CR_STEP_ADAPTIVE && use_adaptive_graph(ctx)) {
            const int key = 3 * ctx->bA + ctx->bB;
            if (!ctx->graph_ad[key] && (st = build_adaptive_graph(ctx, key)) != CR_OK) return st;
            CK(cudaGraphLaunch(ctx->graph_ad[key], ctx->stream));
            advance_host(ctx, 3 - ctx->bA - ctx->bB);
        } else if (ctx->rule == CR_STEP_ADAPTIVE) {
            if ((st = adaptive_step(ctx)) != CR_OK) return st;
        } else {
            const int bo = ctx->bB;
            const int per_iter = ctx->lay.nbar > 1 ? 5 : 3;     // (+ block projections, prologue refresh)
            int64_t room = max_iters - it;                      // iterations before the end / next stop test
            if (stop) room = std::min<int64_t>(room, stop->report_every - it % stop->report_every);
            if (use_graph && room >= kMultiIters) {
                const int key = 3 * ctx->bA + ctx->bB;
                if (!ctx->graph_multi[key] && (st = build_graph_multi(ctx, key)) != CR_OK) return st;
                CK(cudaGraphLaunch(ctx->graph_multi[key], ctx->stream));
                ctx->launches += ctx->multi_launches;
                for (int i = 0; i < kMultiIters; ++i) advance_host(ctx, ctx->bB);
                it += kMultiIters - 1;
            } else if (use_graph) {
                const int key = 3 * ctx->bA + ctx->bB;
                if (!ctx->graph[key] && (st = build_graph(ctx, key)) != CR_OK) return st;
                CK(cudaGraphLaunch(ctx->graph[key], ctx->stream));
                ctx->launches += per_iter;
                advance_host(ctx, bo);
            } else {
                if ((st = enqueue_step(ctx, true, bo, 1.0 / ctx->L, true, false)) != CR_OK) return st;
                advance_host(ctx, bo);
            }
        }
        ++it;
        if (stop && (it % stop->report_every == 0 || it == max_iters)) {
            if (ctx->rule == CR_STEP_ADAPTIVE) {          // never report stats of a rejected trial
                bool failed = false;
                if ((st = adaptive_error_flag(ctx, &failed)) != CR_OK) return st;
                if (failed) return adaptive_exhausted(ctx);
            }
            cr_step_stats s{};
            if ((st = eval_stats(ctx, &s)) != CR_OK) return st;
            if (out) out->last = s;
            if (s.infeas_norm <= stop->infeas_tol && std::fabs(s.gap) / (Nd * Nd - Nd) <= stop->gap_tol) {
                if (out) out->converged = 1;
                break;
            }
        }
    }
    if (out) out->iters = it;
    if (ctx->rule == CR_STEP_ADAPTIVE && use_adaptive_graph(ctx)) {     // trials ran on the device
        double ad[8];
        CK(cudaMemcpyAsync(ad, ctx->at<DevScalars>(ctx->lay.ts)->ad, sizeof ad, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->launches += 6 * ((int64_t)ad[AD_TTOT] - ttot0);     // prologue, pass, reduce, check x2, decide
        if (ad[AD_ERR] != 0.0) return adaptive_exhausted(ctx);
    }
    return CR_OK;
}

cr_status cr_primal(cr_ctx *ctx, double *y, double *xi, cr_step_stats *out) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    cr_step_stats s{};
    // eta(Theta^k) into y64 / Xi64 (all ranks' y gathered), the diagnostics, and the D2H of y, xi:
    // one synchronization
    if ((st = eval_stats(ctx, &s, y, xi)) != CR_OK) return st;
    if (out) *out = s;
    return CR_OK;
}

cr_status cr_get_eta(cr_ctx *ctx, double *y, double *xi) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    const Layout &Ly = ctx->lay;
    double *y64 = ctx->at<double>(Ly.y64);
    if (y && ctx->coll) {
        // make sure all ranks' rows are present (eta of a plain step is only local until gathered)
        CM(comm_allgather(ctx->comm, y64, (size_t)Ly.S, 8, ctx->stream));
    }
    if (y) CK(cudaMemcpyAsync(y, y64, (size_t)Ly.N * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (xi && Ly.Ns > 0)
        CK(cudaMemcpyAsync(xi, ctx->ws + Ly.Xi64, (size_t)Ly.Ns * Ly.n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CR_OK;
}

cr_status cr_get_sums(cr_ctx *ctx, int32_t which, double *r, double *c, double *P) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (which != 0 && which != 1) return fail(ctx, CR_ERR_INVALID_ARG, "cr_get_sums: which");
    const Layout &Ly = ctx->lay;
    const int s = which == 0 ? ctx->bA : ctx->bB;
    if (Ly.Ns > 0) {
        if (r) CK(cudaMemcpyAsync(r, ctx->r[s], (size_t)Ly.Ns * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (c) CK(cudaMemcpyAsync(c, ctx->c[s], (size_t)Ly.Ns * 8, cudaMemcpyDeviceToHost, ctx->stream));
        if (P) CK(cudaMemcpyAsync(P, ctx->P[s], (size_t)Ly.Ns * Ly.n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return CR_OK;
}

cr_status cr_set_step_rule(cr_ctx *ctx, cr_step_rule rule, double upsilon, double s_prev) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (rule != CR_STEP_CONSTANT && rule != CR_STEP_ADAPTIVE && rule != CR_STEP_BACKTRACK)
        return fail(ctx, CR_ERR_INVALID_ARG, "cr_set_step_rule: unknown rule");
    if (rule != CR_STEP_CONSTANT) {
        if (ctx->lay.nbuf < 3)
            return fail(ctx, CR_ERR_STATE, "adaptive step needs the third Theta buffer (cr_config.flags CR_FLAG_ADAPTIVE)");
        if (!(upsilon > 1.0) || !std::isfinite(upsilon))
            return fail(ctx, CR_ERR_INVALID_ARG, "upsilon must be finite and > 1");
        if (s_prev < 0.0 || !std::isfinite(s_prev)) return fail(ctx, CR_ERR_INVALID_ARG, "s_prev must be >= 0");
        ctx->ups = upsilon;
        const double s0 = s_prev > 0.0 ? s_prev : ctx->L;     // s_0 = L_gamma
        const bool mono = rule == CR_STEP_BACKTRACK;
        const double ad[10] = {s0, mono ? s0 : s0 * std::pow(upsilon, -1.0), upsilon, 0.0, 0.0, 0.0,
                               (double)ctx->max_trials, 0.0, mono ? 1.0 : 0.0, 0.0};
        CK(cudaMemcpyAsync(ctx->at<DevScalars>(ctx->lay.ts)->ad, ad, sizeof ad, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    ctx->rule = rule == CR_STEP_CONSTANT ? CR_STEP_CONSTANT : CR_STEP_ADAPTIVE;   // one trial machinery
    ctx->backtrack = rule == CR_STEP_BACKTRACK;
    return CR_OK;
}

cr_status cr_step_info(cr_ctx *ctx, double *s_k, int64_t *trials_last, int64_t *trials_total) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    double ad[8];
    CK(cudaMemcpyAsync(ad, ctx->at<DevScalars>(ctx->lay.ts)->ad, sizeof ad, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const bool a = ctx->rule == CR_STEP_ADAPTIVE;
    if (s_k) *s_k = a ? ad[AD_S] : ctx->L;
    if (trials_last) *trials_last = a ? (int64_t)ad[AD_TLAST] : 1;
    if (trials_total) *trials_total = (int64_t)ad[AD_TTOT];
    if (a && ad[AD_ERR] != 0.0)
        return fail(ctx, CR_ERR_STATE, "adaptive step: no l < %d passed Eq. (adaptive-check)", ctx->max_trials);
    return CR_OK;
}

cr_status cr_partition_info(cr_ctx *ctx, cr_partition_stats *out) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (!out) return fail(ctx, CR_ERR_INVALID_ARG, "cr_partition_info: out is NULL");
    const Layout &Ly = ctx->lay;
    *out = cr_partition_stats{};
    out->nbar = Ly.nbar;
    out->timed_ms = ctx->bp_ms;
    out->timed_launches = ctx->bp_launches;
    if (Ly.nbar > 1 && Ly.Ns > 0) {
        const int64_t nb = Ly.Ns / Ly.nbar;
        std::vector<int32_t> it((size_t)(8 * nb));
        CK(cudaMemcpyAsync(it.data(), ctx->at<int>(Ly.ipm_it), it.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        out->blocks = nb;
        std::vector<unsigned long long> wk((size_t)(3 * nb));
        CK(cudaMemcpyAsync(wk.data(), ctx->at<unsigned long long>(Ly.ipm_work), wk.size() * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (int64_t b = 0; b < nb; ++b) {
            out->factorizations += (int64_t)wk[3 * b];
            out->solves += (int64_t)wk[3 * b + 1];
            out->products += (int64_t)wk[3 * b + 2];
        }
        for (int64_t b = 0; b < nb; ++b) {
            out->ipm_iters_max = std::max(out->ipm_iters_max, it[8 * b]);
            out->polish_rounds_max = std::max(out->polish_rounds_max, it[8 * b + 1]);
            out->multiplier_iters_max = std::max(out->multiplier_iters_max, it[8 * b + 2]);
            out->failed_blocks += it[8 * b + 3] == 1;
            out->unpolished_blocks += it[8 * b + 3] == 2;
            out->warm_blocks += it[8 * b + 4] == 1;
        }
    }
    if (std::getenv("CR_IPM_PROF") && Ly.nbar > 1 && Ly.Ns > 0) {
        unsigned long long pf[8];
        CK(cudaMemcpy(pf, ctx->at<unsigned long long>(Ly.ipm_prof), sizeof pf, cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "block_ipm block 0 cycles: factor %llu solve %llu A %llu AT %llu total %llu\n", pf[0], pf[1],
                     pf[2], pf[3], pf[4]);
    }
    if (out->failed_blocks)
        return fail(ctx, CR_ERR_STATE, "block projection failed in %lld of %lld blocks", (long long)out->failed_blocks,
                    (long long)out->blocks);
    return CR_OK;
}

cr_status cr_selftest_p2p(int32_t world, int64_t N, int32_t nrb, const float *colpart, double *c) {
    if (world < 1 || world > kP2PTab || N < 1 || nrb < 1 || !colpart || !c) return CR_ERR_INVALID_ARG;
    const int64_t S = shard_rows(N, world, 1);
    if (S % 128) return CR_ERR_UNSUPPORTED;
    const int64_t ldT = (N + 3) / 4 * 4;
    float *dcp = nullptr;
    double *dc = nullptr;
    cudaStream_t st = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&dcp, sizeof(float) * (size_t)world * nrb * ldT);
    if (e == cudaSuccess) e = cudaMalloc(&dc, sizeof(double) * (size_t)N);
    // inputs staged on the test's own (non-blocking) stream, so they are ordered before the kernel
    if (e == cudaSuccess) e = cudaMemsetAsync(dcp, 0, sizeof(float) * (size_t)world * nrb * ldT, st);
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(dcp, ldT * sizeof(float), colpart, N * sizeof(float), N * sizeof(float),
                              (size_t)world * nrb, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = p2p_selftest(world, N, nrb, dcp, ldT, dc, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(c, dc, sizeof(double) * N, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (dcp) cudaFree(dcp);
    if (dc) cudaFree(dc);
    if (st) cudaStreamDestroy(st);
    return e == cudaSuccess ? CR_OK : CR_ERR_CUDA;
}

cr_status cr_selftest_p2p_allgather(int32_t world, int64_t N, const float *y, float *out) {
    if (world < 1 || world > kP2PTab || N < 1 || !y || !out) return CR_ERR_INVALID_ARG;
    float *dy = nullptr, *dout = nullptr;
    cudaStream_t st = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&dy, sizeof(float) * (size_t)N);
    if (e == cudaSuccess) e = cudaMalloc(&dout, sizeof(float) * (size_t)world * N);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dy, y, sizeof(float) * (size_t)N, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = p2p_selftest_y(world, N, dy, dout, st);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out, dout, sizeof(float) * (size_t)world * N, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (dy) cudaFree(dy);
    if (dout) cudaFree(dout);
    if (st) cudaStreamDestroy(st);
    return e == cudaSuccess ? CR_OK : CR_ERR_CUDA;
}

cr_status cr_set_gamma(cr_ctx *ctx, double gamma, double L) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (!(gamma > 0.0) || !std::isfinite(gamma) || L < 0.0 || !std::isfinite(L))
        return fail(ctx, CR_ERR_INVALID_ARG, "cr_set_gamma: gamma must be > 0, L >= 0");
    if (L == 0.0 && gamma > 1.0)
        return fail(ctx, CR_ERR_INVALID_ARG, "cr_set_gamma: sigma_max(C)^2/gamma bounds the gradient only for gamma <= 1");
    drop_graphs(ctx);                       // gamma and 1/L are baked into the captured launches
    ctx->gamma = gamma;
    ctx->L = L > 0.0 ? L : ctx->sigma2 / gamma;
    if (ctx->rule == CR_STEP_ADAPTIVE) {                        // s_0 = L_gamma, l = 0
        const double v[2] = {ctx->L, ctx->backtrack ? ctx->L : ctx->L * std::pow(ctx->ups, -1.0)};
        const double l0 = 0.0;
        DevScalars *ts = ctx->at<DevScalars>(ctx->lay.ts);
        CK(cudaMemcpyAsync(&ts->ad[AD_S], v, sizeof v, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(&ts->ad[AD_L], &l0, sizeof l0, cudaMemcpyHostToDevice, ctx->stream));
    }
    // restart Fig. 2 at the current iterate: theta~^1 = theta^0 := Theta^k, t_1 = 1;
    // (t_prev, t_cur) = (1, 1) makes beta_0 = 0, so Theta^{k-1}'s buffer is not read
    DevScalars h{};
    h.t_prev = 1.0;
    h.t_cur = 1.0;
    CK(cudaMemcpyAsync(ctx->ws + ctx->lay.ts, &h, 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CR_OK;
}

cr_status cr_continuation(cr_ctx *ctx, const cr_cont *p, cr_cont_report *out) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (!p || !(p->eps0 > 0.0) || !(p->beta > 1.0) || !(p->kappa_gamma > 0.0) || p->stages < 1 ||
        (!p->iters && p->iters_per_stage < 0) || (p->stop && p->stop->report_every < 1))
        return fail(ctx, CR_ERR_INVALID_ARG, "cr_continuation: bad parameters");
    for (int32_t t = 1; t <= p->stages; ++t) {
        const double g = p->kappa_gamma * p->eps0 / std::pow(p->beta, (double)t);
        if (!(g > 0.0) || g > 1.0) return fail(ctx, CR_ERR_INVALID_ARG, "cr_continuation: gamma_t must be in (0, 1]");
        if (p->iters && p->iters[t - 1] < 0) return fail(ctx, CR_ERR_INVALID_ARG, "cr_continuation: iters[t] < 0");
    }
    if (out) std::memset(out, 0, sizeof *out);
    for (int32_t t = 1; t <= p->stages; ++t) {
        // eps_t = eps0 / beta^t, gamma_t = kappa_gamma eps_t, L_t = sigma^2 / gamma_t
        const double g = p->kappa_gamma * p->eps0 / std::pow(p->beta, (double)t);
        if ((st = cr_set_gamma(ctx, g, 0.0)) != CR_OK) return st;
        cr_report rep{};
        if ((st = cr_solve(ctx, p->iters ? p->iters[t - 1] : p->iters_per_stage, p->stop, &rep)) != CR_OK) return st;
        if (out) {
            out->stages_run = t;
            out->iters_total += rep.iters;
            out->gamma_last = ctx->gamma;
            out->L_last = ctx->L;
        }
    }
    if (out) return eval_stats(ctx, &out->last);
    return CR_OK;
}

cr_status cr_predict(cr_ctx *ctx, const double *Z, int64_t M, double *out) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    if (M < 0 || (M > 0 && (!Z || !out))) return fail(ctx, CR_ERR_INVALID_ARG, "cr_predict: bad arguments");
    if (M == 0) return CR_OK;
    const Layout &Ly = ctx->lay;
    for (int64_t e = 0; e < M * Ly.n; ++e)
        if (!std::isfinite(Z[e])) return fail(ctx, CR_ERR_INVALID_ARG, "cr_predict: non-finite query");
    if ((st = compute_eta(ctx)) != CR_OK) return st;
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
    PredictParams p{};
    p.M = M;
    p.Ns = Ly.Ns;
    p.row0 = Ly.row0;
    p.n = Ly.n;
    p.splits = predict_splits(M, std::max<int64_t>(Ly.Ns, 1), nsm);
    p.y = ctx->at<double>(Ly.y64);
    p.a = ctx->at<double>(Ly.a64);
    p.Xi = ctx->at<double>(Ly.Xi64);
    double *dZ = nullptr, *dpart = nullptr, *dout = nullptr;
    const size_t zb = (size_t)M * Ly.n * 8, pb = (size_t)p.splits * M * 8, ob = (size_t)M * 8;
    // stream-ordered temporaries, released on every path
    struct Tmp {
        cudaStream_t s;
        double **ptrs[3];
        ~Tmp() {
            for (auto pp : ptrs)
                if (*pp) cudaFreeAsync(*pp, s);
        }
    } tmp{ctx->stream, {&dZ, &dpart, &dout}};
    CK(cudaMallocAsync(&dZ, zb, ctx->stream));
    CK(cudaMallocAsync(&dpart, pb, ctx->stream));
    CK(cudaMallocAsync(&dout, ob, ctx->stream));
    CK(cudaMemcpyAsync(dZ, Z, zb, cudaMemcpyHostToDevice, ctx->stream));
    p.Z = dZ;
    p.part = dpart;
    p.out = dout;
    if (Ly.Ns > 0) {
        CK(launch_predict(p, ctx->stream));
        ctx->launches += 2;
    } else {
        // no rows on this rank: -inf, the identity of the max all-reduce below (a NaN pattern
        // is not guaranteed to be ignored by ncclMax)
        std::vector<double> ninf((size_t)M, -std::numeric_limits<double>::infinity());
        CK(cudaMemcpyAsync(dout, ninf.data(), ob, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if (ctx->coll) CM(comm_allreduce_f64(ctx->comm, dout, (size_t)M, COLL_MAX, ctx->stream));
    CK(cudaMemcpyAsync(out, dout, ob, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return CR_OK;
}

double cr_lipschitz(const cr_ctx *ctx) { return ctx ? ctx->L : 0.0; }

int64_t cr_launch_count(const cr_ctx *ctx) { return ctx ? ctx->launches : 0; }

cr_kernel cr_active_kernel(const cr_ctx *ctx) { return ctx ? ctx->kernel : CR_KERNEL_AUTO; }

cr_status cr_set_pass_timing(cr_ctx *ctx, int32_t on) {
    if (!ctx) return CR_ERR_INVALID_ARG;
    ctx->timing = on != 0;
    ctx->ev_used = 0;
    ctx->ev_iters = 0;
    return CR_OK;
}

cr_status cr_pass_timing(cr_ctx *ctx, double *total_ms, int64_t *launches) {
    cr_status st = check_ctx(ctx);
    if (st != CR_OK) return st;
    CK(cudaStreamSynchronize(ctx->stream));
    double tot = 0.0;
    for (size_t i = 0; i + 1 < ctx->ev_used; i += 2) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]));
        tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = ctx->ev_iters;
    ctx->ev_used = 0;
    ctx->ev_iters = 0;
    ctx->bp_ms = 0.0;
    for (size_t i = 0; i + 1 < ctx->bp_ev_used; i += 2) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->bp_ev[i], ctx->bp_ev[i + 1]));
        ctx->bp_ms += ms;
    }
    ctx->bp_launches = (int64_t)(ctx->bp_ev_used / 2);
    ctx->bp_ev_used = 0;
    return CR_OK;
}

void cr_destroy(cr_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    // cr_solve is asynchronous: let queued work finish before the caller may reuse the workspace
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    drop_graphs(ctx);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->trace) cudaFree(ctx->trace);
    if (ctx->tc_check) cudaFree(ctx->tc_check);
    for (auto e : ctx->ev) cudaEventDestroy(e);
    for (auto e : ctx->bp_ev) cudaEventDestroy(e);
    if (ctx->comm.nccl) ncclCommDestroy(ctx->comm.nccl);
    for (void *ptr : ctx->p2p_opened) cudaIpcCloseMemHandle(ptr);
    if (ctx->p2p_buf) cudaFree(ctx->p2p_buf);
    if (ctx->p2p_tab) cudaFree(ctx->p2p_tab);
    delete ctx;
}

}  // extern "C"
