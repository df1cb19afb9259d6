// Fused pair pass on the 5th-gen tensor cores (tcgen05, kind::tf32, 3xTF32), sm_100a.
//
// Same mathematics as pass_simt.cu (Steps 2 and 4 of P-APG Fig. 2, plus the
// sums Step 1 of the next iteration needs), organised like a flash-attention forward:
//
//   GEMM1  S' = Xi'_I X_J^T        M=128 rows i, N=32 cols j, K=n  (A = Xi' in TMEM, B = X_J smem)
//   epilogue  Theta^k = (Theta^{k-1} + beta (Theta^{k-1} - Theta^{k-2}) + S' - y'_j - b'_i)_+
//   GEMM2  P_I += Theta^k_IJ X_J   M=128 rows i, N=n,  K=32 cols j  (A = Theta^k in TMEM, B = X_J^T smem)
//   row / column sums of Theta^k on CUDA cores (thread row sums, warp-butterfly column sums)
//
// Both GEMMs use 3xTF32 (hi*hi + hi*lo + lo*hi, hi = fp32 with the low 13 mantissa bits
// cleared, lo = remainder) so products carry ~fp32 accuracy.  Both B operands are K-major
// no-swizzle ("interleave") tiles prepared once at init: X_J as [j][k] and X_J^T as [d][j]
// core matrices (8 rows x 16 B), so each per-tile image is exactly 32 n fp32.  (MN-major
// tf32 operands would need the SW128_32B layout; two K-major images avoid it.)
// Theta is stored tile-major (each 128 x 32 tile 16 KB contiguous, already in the 128-B-swizzled
// smem image): Theta^{k-1}, Theta^{k-2} tiles arrive by one 1-D bulk copy each
// (cp.async.bulk), Theta^k leaves by a 1-D bulk store from the same smem slot.  The Theta X
// accumulator lives in TMEM and is flushed to fp64 (global, per CTA run slot) every `window` tiles.
// GEMM1 runs in kind::f16 (fp16 hi/lo with exact power-of-2 row scalings) for n > 56.
// Warp roles: 0 = bulk-copy producer, 1 = GEMM1 issuer (+ TMEM owner), 2 = bulk storer, 3 = GEMM2 issuer,
// 4..7 / 8..11 = two epilogue warpgroups that take alternate tiles (ping-pong).
// Persistent: CTA g owns tiles [g T / G, (g+1) T / G) of the row-major (row block, column
// tile) order, like the SIMT pass.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "../cr_internal.h"
#include "sm100.cuh"

namespace cr {
namespace {

using namespace sm100;

constexpr int TBM = kTcBM;      // 128 rows per tile (TMEM lanes)
constexpr int TBN = kTcBN;      // 32 columns per tile
constexpr int NTHR = 384;       // 12 warps
constexpr uint32_t TILE_BYTES = TBM * TBN * 4;     // 16 KB

struct __align__(8) TcBarriers {
    uint64_t full[kTcMaxStages], empty[kTcMaxStages];      // Theta ring (B1, B2 tiles, y'_J)
    uint64_t g1full[kTcMaxStages], g1empty[kTcMaxStages];  // X_J image ring (GEMM1 B operand)
    uint64_t g2full[kTcMaxStages], g2empty[kTcMaxStages];  // X_J^T image ring (GEMM2 B operand)
    // st_full is per stage (not per warpgroup): a stage is refilled only after the storer
    // released it, so no arrival can run two phases ahead of the storer's parity wait
    uint64_t st_full[kTcMaxStages];
    uint64_t d1_full[2], d1_empty[2], at_full[2], at_empty[2];
    uint64_t d2_full, d2_empty, xi_full;
    uint32_t tmem_base;
    uint32_t nzAT[2][4];         // per A-operand buffer, per epilogue warp: its 32 rows of Theta^k not all zero
    // CR_TC_CHECK tags: the tile index u (or run index) a slot / buffer holds, written by its
    // producer before the release (arrive) its consumer acquires (wait), checked after the wait
    int tagT[kTcMaxStages], tagX1[kTcMaxStages], tagX2[kTcMaxStages], tagAT[2], tagXi;
};

// ring-protocol violation codes (TcParams::check)
enum TcCheckCode { TCC_THETA_EPI = 1, TCC_THETA_G1 = 2, TCC_THETA_ST = 3, TCC_X1 = 4, TCC_X2 = 5, TCC_AT = 6,
                   TCC_XI = 7 };

// tf32 "hi" part of x: round to the nearest 10-bit-mantissa value (ties away), low 13 bits
// cleared, so the remainder x - hi (exact in fp32) is at most 2^-12 |x| and the product error
// of the 3xTF32 split is ~2^-23 relative.  The MMA reads hi exactly (its low bits are zero).
__device__ __forceinline__ float tf32_hi(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// butterfly step: lane keeps the half of v selected by its bit, adds the partner's other half
template <int H>
__device__ __forceinline__ void bfly(const float *v, float *o, int lane) {
    const bool up = (lane & H) != 0;
#pragma unroll
    for (int c = 0; c < H; ++c) {
        const float send = up ? v[c] : v[c + H];
        const float keep = up ? v[c + H] : v[c];
        o[c] = keep + __shfl_xor_sync(0xffffffffu, send, H);
    }
}

// 16 x 16 transpose inside each half-warp: lane l's v[c] <- lane (l & 16) + c's v[l & 15].  Four
// butterfly stages, stage H swapping bit H between the lane and the register index where they
// differ (the stages commute); register indices stay compile-time.
__device__ __forceinline__ void transpose16(uint32_t (&v)[16], int lane) {
#pragma unroll
    for (int H = 8; H >= 1; H >>= 1) {
        const bool up = (lane & H) != 0;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            if (c & H) continue;
            const uint32_t send = up ? v[c] : v[c + H];
            const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, H);
            if (up) v[c] = recv;
            else v[c + H] = recv;
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void tc_check_fail(const TcParams &p, int code, int u) {
    atomicCAS(p.check, 0ULL, ((unsigned long long)code << 56) | ((unsigned long long)blockIdx.x << 32) | (unsigned)u);
}
// ring-protocol checks exist only in the TC_CHECK instantiations (kernel template below): even
// guarded by a runtime flag they cost the C4 pass 3.5% and C5 6% (code size in the role loops)
#define tc_check(p, cond, code, u)                                                               \
    do {                                                                                         \
        if constexpr (CHECK) {                                                                   \
            if (!(cond)) tc_check_fail((p), (code), (u));                                        \
        }                                                                                        \
    } while (0)
#define tc_tag(p, stmt)                                                                          \
    do {                                                                                         \
        if constexpr (CHECK) { stmt; }                                                           \
    } while (0)

// kernel variants (template MODE): plain, ring-protocol checks (TcParams::check), or the P2P y'
// acquire fused into the producer with the own-columns-first rotation (TcParams::yflag)
enum TcMode { TC_PLAIN = 0, TC_CHECK = 1, TC_P2PY = 2, TC_ADAPT = 3 };

// Position of the u-th tile a CTA processes: segment k of its schedule (a row block rb and a
// column-tile range [cbb, cbe)), column tile cb, and the slot / phase parity of the Theta ring
// (s, ph), the X_J ring (x, xph) and the X_J^T ring (z, zph) (all incremental: no divisions).
struct Cursor {
    int u, k, rb, cb, cbb, cbe, s, ph, x, xph, z, zph;
};

// debug timeline (p.trace != nullptr): clock64 of role events for the first 256 tiles of CTA 0.
// Compiled in only with -DCR_TC_TRACE_BUILD (CR_NVCC_EXTRA): the per-tile checks of p.trace and
// the clock reads cost the production pass (ncu source view: their LDC / CS2R stalls).
#ifdef CR_TC_TRACE_BUILD
#define TC_TRACE(role, u, ev)                                                                   \
    do {                                                                                        \
        if (p.trace && blockIdx.x == 0 && (u) < 256)                                            \
            p.trace[((role) * 256 + (u)) * 8 + (ev)] = clock64();                               \
    } while (0)
#define TC_TRACE_ON 1
#else
#define TC_TRACE(role, u, ev) \
    do {                      \
    } while (0)
#define TC_TRACE_ON 0
#endif

// F16: GEMM1 in kind::f16 (TcParams::g1f16) -- a compile-time switch, so each instantiation keeps
// one GEMM1 / Xi'-load code path (the kernel is instruction-cache sensitive: a runtime switch with
// both paths unrolled cost the C4 pass 15%)
template <int NK, bool F16, int MODE>
__global__ void __launch_bounds__(NTHR, 1)
pass_tc_kernel(const TcParams p) {
    constexpr bool CHECK = MODE == TC_CHECK, P2PY = MODE == TC_P2PY;
    constexpr int NP2 = (NK + 15) / 16 * 16;           // GEMM2 N (multiple of 16 for M = 128)
    constexpr int NK16 = NP2;                          // GEMM1 K in kind::f16 (16 per instruction)
    extern __shared__ __align__(16) uint8_t smem_raw[];
    // 1024-byte alignment by offsetting the shared pointer itself (an integer round trip would
    // lose the shared address space and turn every access into a generic LD/ST)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    // Three rings, each with its own depth and release point:
    //   Theta ring, S slots  [B1 16K][B2 16K] (+ y'_J, 128 B, in a side array): HBM stream;
    //                        released by the storer once Theta^k has left the slot
    //   X_J ring,   S1 slots [X hi][X lo] (GEMM1 B operand): released when GEMM1 completes
    //   X_J^T ring, S2 slots [X^T hi][X^T lo] (GEMM2 B operand): released when GEMM2 completes
    // so the L2-resident operand images never wait on the epilogue of an older tile.
    const int S = p.stages, S1 = p.g1stages, S2 = p.g2stages;
    constexpr uint32_t stage_bytes = 2 * TILE_BYTES;
    // X slot images (hi, lo); the X_J slot holds X_hi only when GEMM1 runs 2 passes.  X_J image:
    // tf32 NK x 32 x 4 B, or fp16 NK16 x 32 x 2 B (kind::f16 GEMM1)
    constexpr bool f16 = F16;
    constexpr uint32_t g1_bytes = f16 ? (uint32_t)NK16 * 64 : (uint32_t)NK * 128;
    constexpr uint32_t g2_bytes = (uint32_t)NP2 * 128;
    const bool g1lo = p.g1passes >= 3;
    const uint32_t g1_slot = g1lo ? 2 * g1_bytes : g1_bytes;
    uint8_t *g1ring = smem + (size_t)S * stage_bytes;
    uint8_t *g2ring = g1ring + (size_t)S1 * g1_slot;
    uint8_t *yring = g2ring + (size_t)S2 * 2 * g2_bytes;
    TcBarriers *bar = reinterpret_cast<TcBarriers *>(yring + (size_t)kTcMaxStages * 128);
    float *colS = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(bar) + sizeof(TcBarriers) + 8);  // [2 wg][2][4][32]
    float *rowscale = colS + 2 * 2 * 4 * 32;          // [2 runs][128] f16 GEMM1: 2^-(e_i + xexp) per row

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) TC_TRACE(0, 0, 0);          // kernel entry
    if (TC_TRACE_ON && p.trace && threadIdx.x == 0 && blockIdx.x < 1024) p.trace[kTraceTile + 4 * blockIdx.x] = gtimer();
    const int t0 = (int)((int64_t)blockIdx.x * p.T / p.G), t1 = (int)((int64_t)(blockIdx.x + 1) * p.T / p.G);
    if (t0 >= t1) return;
    const int U = t1 - t0;
    const int nCB = p.nCB;
    constexpr int W = NP2 + 4;                         // rowpart row: Theta X | r (2 wg) | ||D||^2 (2 wg)
    const int wmask = p.window - 1;                    // flush window (power of two)
    constexpr uint32_t lbo2 = (uint32_t)NP2 * 16;      // X^T image: K-chunk (4 j) stride
    const int slot0 = p.cta_slot0[blockIdx.x];
    // Schedule.  The CTA owns the contiguous tiles [t0, t1) of the row-major (row block, column
    // tile) order: possibly a partial head row block, full row blocks, a partial tail row block.
    // It processes the FULL row blocks first (each swept from column tile 0), then the tail, then
    // the head: all CTAs then sweep the column tiles in near lockstep, so the per-column-tile X
    // operand images they stream are shared through L2 instead of being re-read from HBM.
    const int rbA = t0 / nCB, cbA = t0 - rbA * nCB;
    const int rbZ = (t1 - 1) / nCB, cbZ = (t1 - 1) - rbZ * nCB + 1;
    const bool single = rbA == rbZ;
    const bool hp = !single && cbA > 0, tp = !single && cbZ < nCB;
    const int full0 = hp ? rbA + 1 : rbA, nfull = single ? 0 : (tp ? rbZ - 1 : rbZ) - full0 + 1;
    const int nseg = single ? 1 : nfull + (tp ? 1 : 0) + (hp ? 1 : 0);
    auto seg = [&](Cursor &c) {             // load segment c.k into the cursor
        if (single) { c.rb = rbA; c.cbb = cbA; c.cbe = cbZ; }
        else if (c.k < nfull) { c.rb = full0 + c.k; c.cbb = 0; c.cbe = nCB; }
        else if (c.k == nfull && tp) { c.rb = rbZ; c.cbb = 0; c.cbe = cbZ; }
        else { c.rb = rbA; c.cbb = cbA; c.cbe = nCB; }
        c.cb = c.cbb;
    };

    auto stage_ptr = [&](int s) { return smem + (size_t)s * stage_bytes; };
    // actual column tile of virtual column tile cb (rotation by p.rot: own columns first, P2P)
    const int rot = P2PY ? p.rot : 0;
    auto acb = [&](int cb) {
        if constexpr (P2PY) {
            const int a = cb + rot;
            return a >= nCB ? a - nCB : a;
        } else {
            return cb;
        }
    };
    auto adv = [&](Cursor &c, int k) {
        for (int i = 0; i < k; ++i) {
            ++c.u;
            if (++c.cb == c.cbe && ++c.k < nseg) seg(c);
            if (++c.s == S) { c.s = 0; c.ph ^= 1; }
            if (++c.x == S1) { c.x = 0; c.xph ^= 1; }
            if (++c.z == S2) { c.z = 0; c.zph ^= 1; }
        }
    };
    auto start = [&]() {
        Cursor c{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        seg(c);
        return c;
    };
    auto run_start = [&](const Cursor &c) { return c.cb == c.cbb; };
    auto run_end = [&](const Cursor &c) { return c.cb + 1 == c.cbe; };
    auto flush_after = [&](const Cursor &c) { return run_end(c) || ((c.cb - c.cbb + 1) & wmask) == 0; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&bar->full[s], 1);
            mbar_init(&bar->empty[s], 1);           // storer: Theta^k left the slot
            mbar_init(&bar->st_full[s], 4);
        }
        for (int x = 0; x < S1; ++x) {
            mbar_init(&bar->g1full[x], 1);
            mbar_init(&bar->g1empty[x], 1);         // GEMM1 commit
        }
        for (int z = 0; z < S2; ++z) {
            mbar_init(&bar->g2full[z], 1);
            mbar_init(&bar->g2empty[z], 1);         // GEMM2 commit
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar->d1_full[b], 1); mbar_init(&bar->d1_empty[b], 4);
            mbar_init(&bar->at_full[b], 4); mbar_init(&bar->at_empty[b], 1);
        }
        mbar_init(&bar->d2_full, 1);
        mbar_init(&bar->d2_empty, 4);
        mbar_init(&bar->xi_full, 4);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&bar->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bar->tmem_base;
    // setup above (barriers, TMEM) overlaps the predecessor's tail under PDL; its outputs (y', b',
    // xi', Theta) are read only after this wait
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) TC_TRACE(0, 0, 4);          // predecessor complete
    if (TC_TRACE_ON && p.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
        p.trace[kTraceTile + 4 * blockIdx.x + 1] = gtimer();
        p.trace[kTraceTile + 4 * blockIdx.x + 3] = (unsigned long long)U;
    }
    // TMEM columns: D1[2] 0..63 | Theta^k A operand [2] x (hi 32, lo 32) 64..191 | D2 (NP2) | Xi' hi, lo
    // (tf32: NK columns each; fp16: NK16 / 2 columns each, two K elements per column)
    const uint32_t c_d1 = 0, c_at = 64, c_d2 = 192, c_xi = 192 + (uint32_t)NP2;
    constexpr uint32_t xi_lo_off = f16 ? (uint32_t)NK16 / 2 : (uint32_t)NK;

    if (warp == 0) {
        // ============================================================ TMA producer
        // One thread feeds the three rings, polling their free-slot barriers without blocking:
        // each ring's loads go out as soon as its next slot is released.
        if (lane == 0) {
            // Theta streams past L2 (evict-first) unless the whole state fits in it (p.theta_l2)
            const uint64_t pol_stream = (p.theta_l2 & 1) ? policy_evict_normal() : policy_evict_first();
            const uint64_t pol_keep = policy_evict_last();
            Cursor c = start(), c1 = start(), c2 = start();
            // P2P: peer y' acquired per source rank before its first column tile (see TcParams)
            uint32_t acquired = 0;
            const unsigned long long yep = P2PY ? *p.yepoch + 1 : 0;
            while (c.u < U || c1.u < U || c2.u < U) {
                bool issued = false;
                if (P2PY && c.u < U) {
                    const int q = (int)((int64_t)acb(c.cb) * TBN / p.S);
                    if (!((acquired >> q) & 1u)) {
                        const int64_t rows = max((int64_t)0, min(p.S, p.N - (int64_t)q * p.S));
                        const unsigned long long target = yep * (unsigned long long)rows;
                        unsigned long long v;
                        while (true) {
                            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p.yflag + q) : "memory");
                            if (v >= target) break;
                            __nanosleep(64);
                        }
                        asm volatile("fence.proxy.async.global;" ::: "memory");   // generic -> bulk-copy reads
                        acquired |= 1u << q;
                    }
                }
                if (c.u < U && mbar_test(&bar->empty[c.s], (uint32_t)(c.ph ^ 1))) {
                    issued = true;
                    TC_TRACE(0, c.u, 1);
                    uint8_t *st = stage_ptr(c.s);
                    uint64_t *fb = &bar->full[c.s];
                    tc_tag(p, bar->tagT[c.s] = c.u);
                    mbar_arrive_expect_tx(fb, 2 * TILE_BYTES + TBN * 4);
                    // tile-major Theta: each 128 x 32 tile is 16 KB contiguous, already in the
                    // 128-B-swizzled smem image (theta_off): one bulk copy per tile
                    const size_t toff = ((size_t)c.rb * nCB + acb(c.cb)) * (TILE_BYTES / 4);
                    bulk_load(st, p.B1 + toff, TILE_BYTES, fb, pol_stream);
                    bulk_load(st + TILE_BYTES, p.B2 + toff, TILE_BYTES, fb, pol_stream);
                    bulk_load(yring + c.s * 128, p.yv + acb(c.cb) * TBN, TBN * 4, fb, pol_keep);
                    adv(c, 1);
                }
                if (c1.u < U && mbar_test(&bar->g1empty[c1.x], (uint32_t)(c1.xph ^ 1))) {
                    issued = true;
                    TC_TRACE(0, c1.u, 2);
                    uint8_t *xs = g1ring + (size_t)c1.x * g1_slot;
                    uint64_t *fb = &bar->g1full[c1.x];
                    tc_tag(p, bar->tagX1[c1.x] = c1.u);
                    mbar_arrive_expect_tx(fb, g1_slot);
                    bulk_load(xs, p.g1_hi + (size_t)acb(c1.cb) * (g1_bytes / 4), g1_bytes, fb, pol_keep);
                    if (g1lo)
                        bulk_load(xs + g1_bytes, p.g1_lo + (size_t)acb(c1.cb) * (g1_bytes / 4), g1_bytes, fb, pol_keep);
                    adv(c1, 1);
                }
                if (c2.u < U && mbar_test(&bar->g2empty[c2.z], (uint32_t)(c2.zph ^ 1))) {
                    issued = true;
                    TC_TRACE(0, c2.u, 3);
                    uint8_t *xs = g2ring + (size_t)c2.z * 2 * g2_bytes;
                    uint64_t *fb = &bar->g2full[c2.z];
                    tc_tag(p, bar->tagX2[c2.z] = c2.u);
                    mbar_arrive_expect_tx(fb, 2 * g2_bytes);
                    bulk_load(xs, p.g2_hi + (size_t)acb(c2.cb) * NP2 * 32, g2_bytes, fb, pol_keep);
                    bulk_load(xs + g2_bytes, p.g2_lo + (size_t)acb(c2.cb) * NP2 * 32, g2_bytes, fb, pol_keep);
                    adv(c2, 1);
                }
                // nothing to issue: back off instead of spinning on the issue slots the
                // epilogue warps of this scheduler need
                if (!issued) __nanosleep(p.poll_ns);
            }
        }
    } else if (warp == 1 || warp == 3) {
        // ============================================================ MMA issuers (whole warp, convergent;
        // elect.sync inside the tcgen05 wrappers picks the issuing lane).  Warp 1 issues GEMM1
        // (S' into D1), warp 3 issues GEMM2 (Theta X into D2): the two accumulators are
        // independent, so the issue streams run in parallel.
        const uint32_t tmu = __shfl_sync(0xffffffffu, tmem, 0);   // warp-uniform copies
        const uint32_t g1base = __shfl_sync(0xffffffffu, smem_u32(g1ring), 0);
        const uint32_t g2base = __shfl_sync(0xffffffffu, smem_u32(g2ring), 0);
        if (warp == 1) {
            constexpr uint32_t id1 = f16 ? idesc_f16(TBM, TBN, 0, 0) : idesc_tf32(TBM, TBN, 0, 0);   // A, B K-major
            int run = 0;
            for (Cursor c = start(); c.u < U; adv(c, 1)) {
                const int b = c.u & 1;
                if (lane == 0) TC_TRACE(1, c.u, 0);
                if (run_start(c)) {                          // Xi' of this run loaded into TMEM
                    mbar_wait(&bar->xi_full, (uint32_t)(run & 1));
                    tc_check(p, bar->tagXi == run, TCC_XI, c.u);
                    ++run;
                }
                mbar_wait(&bar->g1full[c.x], (uint32_t)c.xph);
                tc_check(p, bar->tagX1[c.x] == c.u, TCC_X1, c.u);
                // GEMM1 needs only X_J and Xi'.  By default it also waits for the tile's Theta
                // (g1_runahead = 0); run-ahead lets S' of later tiles be computed while their Theta
                // is still in flight (ring invariants).
                if (!p.g1_runahead) {
                    mbar_wait(&bar->full[c.s], (uint32_t)c.ph);
                    tc_check(p, bar->tagT[c.s] == c.u, TCC_THETA_G1, c.u);
                }
                mbar_wait(&bar->d1_empty[b], (uint32_t)(((c.u >> 1) & 1) ^ 1));
                if (lane == 0) TC_TRACE(1, c.u, 1);
                tc_fence_after();
                const uint32_t xh = g1base + (uint32_t)c.x * g1_slot;
                const uint32_t d = tmu + c_d1 + (uint32_t)b * TBN;
                // K-major interleave: 4-k chunks LBO = 512 B apart, 8-row j groups SBO = 128 B;
                // K-step kk advances the start address by 1024 B (= 64 in the >>4 address field)
                const uint64_t bh = smem_desc_u32(xh, 512, 128, 0), bl = smem_desc_u32(xh + g1_bytes, 512, 128, 0);
#pragma unroll
                for (int pass = 0; pass < 3; ++pass) {
                    if (pass == 1 && !g1lo) continue;          // 2 passes: Xi_hi X_hi + Xi_lo X_hi
                    const uint64_t bd0 = pass == 1 ? bl : bh;
                    const uint32_t a0 = tmu + c_xi + (pass == 2 ? xi_lo_off : 0u);
                    if constexpr (f16) {
                        // K = 16 per instruction: 8 TMEM columns of A, two 8-element core matrices of B
#pragma unroll
                        for (int kk = 0; kk < NK16 / 16; ++kk)
                            mma_f16_ts_warp(d, a0 + (uint32_t)kk * 8, bd0 + (uint64_t)(kk * 64), id1, (pass | kk) != 0);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < NK / 8; ++kk)
                            mma_tf32_ts_warp(d, a0 + (uint32_t)kk * 8, bd0 + (uint64_t)(kk * 64), id1, (pass | kk) != 0);
                    }
                }
                mma_commit_warp(&bar->d1_full[b]);
                mma_commit_warp(&bar->g1empty[c.x]);
                if (lane == 0) TC_TRACE(1, c.u, 2);
            }
        } else {
            const uint32_t id2 = idesc_tf32(TBM, NP2, 0, 0);
            int flushes = 0;
            bool window_start = true;
            for (Cursor c = start(); c.u < U; adv(c, 1)) {
                const int a = c.u & 1;
                if (lane == 0) TC_TRACE(1, c.u, 3);
                mbar_wait(&bar->at_full[a], (uint32_t)((c.u >> 1) & 1));
                tc_check(p, bar->tagAT[a] == c.u, TCC_AT, c.u);
                mbar_wait(&bar->g2full[c.z], (uint32_t)c.zph);
                tc_check(p, bar->tagX2[c.z] == c.u, TCC_X2, c.u);
                if (window_start && flushes > 0) mbar_wait(&bar->d2_empty, (uint32_t)((flushes - 1) & 1));
                if (lane == 0) TC_TRACE(1, c.u, 4);
                tc_fence_after();
                const uint32_t xh = g2base + (uint32_t)c.z * 2 * g2_bytes;
                // X^T image, K-major interleave: 4-j chunks lbo2 apart, 8-row d groups 128 B;
                // K-step jj (8 j) advances the start address by 2 lbo2 bytes
                const uint64_t bh = smem_desc_u32(xh, lbo2, 128, 0), bl = smem_desc_u32(xh + g2_bytes, lbo2, 128, 0);
                const uint32_t ws = window_start ? 1u : 0u;
                // an all-zero Theta^k tile adds nothing to Theta X: its MMAs are skipped (exact), except
                // at a window start, whose MMAs reset the accumulator (accumulate = 0)
                const volatile uint32_t *nz = bar->nzAT[a];
                const bool issue = window_start || ((nz[0] | nz[1] | nz[2] | nz[3]) != 0u);
                if (issue) {
#pragma unroll
                    for (int pass = 0; pass < 3; ++pass) {
                        const uint64_t bd0 = pass == 1 ? bl : bh;
                        const uint32_t a0 = tmu + c_at + (uint32_t)a * 64 + (pass == 2 ? 32u : 0u);
#pragma unroll
                        for (int jj = 0; jj < TBN / 8; ++jj)
                            mma_tf32_ts_warp(tmu + c_d2, a0 + (uint32_t)jj * 8, bd0 + (uint64_t)(jj * 2 * lbo2 / 16), id2,
                                             (pass | jj) != 0 ? 1u : (ws ^ 1u));
                    }
                }
                mma_commit_warp(&bar->at_empty[a]);
                mma_commit_warp(&bar->g2empty[c.z]);
                if (lane == 0) TC_TRACE(1, c.u, 5);
                window_start = false;
                if (flush_after(c)) {
                    mma_commit_warp(&bar->d2_full);
                    ++flushes;
                    window_start = true;
                }
            }
        }
    } else if (warp == 2) {
        // ============================================================ TMA storer
        if (lane == 0) {
            const uint64_t pol_stream = (p.theta_l2 & 2) ? policy_evict_normal() : policy_evict_first();
            for (Cursor c = start(); c.u < U; adv(c, 1)) {
                TC_TRACE(2, c.u, 0);
                mbar_wait(&bar->st_full[c.s], (uint32_t)c.ph);
                tc_check(p, bar->tagT[c.s] == c.u, TCC_THETA_ST, c.u);
                TC_TRACE(2, c.u, 1);
                bulk_store(p.Bout + ((size_t)c.rb * nCB + acb(c.cb)) * (TILE_BYTES / 4), stage_ptr(c.s) + TILE_BYTES,
                           TILE_BYTES, pol_stream);
                bulk_commit();
                bulk_wait_read<0>();                      // slot read by the store engine
                TC_TRACE(2, c.u, 2);
                mbar_arrive(&bar->empty[c.s]);
            }
            bulk_wait<0>();
        }
    } else if (warp >= 4) {
        // ============================================================ epilogue: 2 warpgroups, ping-pong tiles
        const int wg = (warp - 4) >> 2;               // warpgroup: tiles u with u % 2 == wg
        const int q = warp & 3;                       // TMEM lane quarter
        const int r = q * 32 + lane;                  // row within the tile
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const float beta = (float)((p.ts[0] - 1.0) / p.ts[1]);   // beta_{k-1} = (t_{k-1}-1)/t_k
        int flushes = 0;
        int last_flush_slot = -1;
        double rrun = 0.0;                            // this warpgroup's row sum over the current run
        double drun = 0.0;                            // ... and sum of (Theta^k - theta~)^2 (adaptive step)
        // the adaptive-step sums are compiled out of the plain variant (a smaller epilogue loop;
        // adaptive runs use TC_ADAPT, the check / P2P variants keep the runtime switch)
        const bool adapt = MODE != TC_PLAIN && p.adapt != 0;
        float bi = 0.f;
        int cur_rb = -1;
        float *my_colS = colS + wg * 2 * 4 * 32;

        auto load_xi = [&](int rb, int run) {        // run: the segment index (GEMM1's run count)
            // Xi' row r of row block rb into TMEM (hi and lo columns)
            const float *src = p.XiR + ((int64_t)rb * TBM + r) * NK;
            if constexpr (f16) {
                // fp16 hi / lo of Xi' 2^e_r, e_r putting the row's largest |Xi'| just below 2^14
                // (compile-time trip count: the NK loads go out together, not one dependent
                // round trip per feature -- 12 us at n = 80 on the kernel's critical path)
                float mx = 0.f;
#pragma unroll
                for (int k = 0; k < NK; ++k) mx = fmaxf(mx, k < p.n ? fabsf(src[k]) : 0.f);
                // mx < 2^E, E = biased exponent - 126 (mx normal); e = 14 - E, clamped so 2^e is a float
                const int E = (int)((__float_as_uint(mx) >> 23) & 0xffu) - 126;
                const int e = mx > 0.f ? min(14 - E, 120) : 0;
                const float sc = __int_as_float((uint32_t)(127 + e) << 23);   // 2^e (exact scaling)
#pragma unroll 1
                for (int k0 = 0; k0 < NK16; k0 += 16) {
                    uint32_t hi[8], lo[8];
#pragma unroll
                    for (int e2 = 0; e2 < 8; ++e2) {
                        uint32_t hb[2], lb[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int k = k0 + 2 * e2 + h;
                            const float x = k < p.n ? src[k] * sc : 0.f;
                            const __half xh = __float2half_rn(x);
                            const __half xl = __float2half_rn(x - __half2float(xh));
                            hb[h] = __half_as_ushort(xh);
                            lb[h] = __half_as_ushort(xl);
                        }
                        hi[e2] = hb[0] | (hb[1] << 16);
                        lo[e2] = lb[0] | (lb[1] << 16);
                    }
                    tmem_st8(tmem + lane_off + c_xi + (uint32_t)(k0 / 2), hi);
                    tmem_st8(tmem + lane_off + c_xi + xi_lo_off + (uint32_t)(k0 / 2), lo);
                }
                rowscale[(run & 1) * TBM + r] = ldexpf(1.f, -(e + p.xexp));
            } else {
#pragma unroll
                for (int k0 = 0; k0 < NK; k0 += 8) {
                    uint32_t hi[8], lo[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float x = src[k0 + e];
                        const float h = tf32_hi(x);
                        hi[e] = __float_as_uint(h);
                        lo[e] = __float_as_uint(x - h);
                    }
                    tmem_st8(tmem + lane_off + c_xi + (uint32_t)k0, hi);
                    tmem_st8(tmem + lane_off + c_xi + (uint32_t)(NK + k0), lo);
                }
            }
            tmem_wait_st();
            tc_fence_before();
            // (the phase completes only with warp 0's arrive, which follows its tag store)
            tc_tag(p, if (q == 0 && lane == 0) bar->tagXi = run);
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->xi_full);
        };
        // Theta X flush after tile c (warpgroup 0 only, in tile order: each slot receives its
        // window partials from one thread in a fixed order -> deterministic)
        auto flush = [&](const Cursor &c) {
            mbar_wait(&bar->d2_full, (uint32_t)(flushes & 1));
            tc_fence_after();
            const int sl = slot0 + (c.rb - rbA);
            const bool first = sl != last_flush_slot;
            last_flush_slot = sl;
            // each thread holds its row's 16 columns d0..d0+15; transposed inside each half-warp,
            // one store instruction then writes 2 rows x 16 consecutive columns (whole 128-B lines,
            // not 32 rows' scattered words: the scattered form stalled the CTA ~5-8 us per flush)
            const int hl = lane & 15;
            double *dst = p.rowpart + ((int64_t)sl * TBM + q * 32 + (lane & 16)) * W + hl;
#pragma unroll 1
            for (int d0 = 0; d0 < NP2; d0 += 16) {
                uint32_t a[16];
                tmem_ld16(tmem + lane_off + c_d2 + (uint32_t)d0, a);
                tmem_wait_ld();
                transpose16(a, lane);                  // a[k] = (row q*32 + (lane & 16) + k, column d0 + hl)
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double v = (double)__uint_as_float(a[k]);
                    double *o = dst + (int64_t)k * W + d0;
                    // later windows: a fire-and-forget fp64 atomic add (RED) -- same single IEEE add per
                    // window in window order (one thread per element, same-address ordering), without
                    // the read-modify-write's load round trip (~8k cycles per flush at n = 80)
                    if (first) *o = v;
                    else atomicAdd(o, v);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->d2_empty);
            ++flushes;
        };

        Cursor c = start();
        if (wg == 1) adv(c, 1);
        if (wg == 0) load_xi(c.rb, 0);
        [[maybe_unused]] const bool tr = (q == 0 && lane == 0);
        for (; c.u < U; adv(c, 2)) {
            const int b = c.u & 1;
            const int rb = c.rb, cb = acb(c.cb);
            if (tr) TC_TRACE(3 + wg, c.u, 0);
            if (c.u > 0 && run_start(c)) {
                // new run: all GEMM1 of the previous run are complete once D1 of tile u-1 is
                mbar_wait(&bar->d1_full[b ^ 1], (uint32_t)(((c.u - 1) >> 1) & 1));
                load_xi(rb, c.k);
            }
            const int lr = rb * TBM + r;                  // local row (< 2^31: Rp * 128)
            if (rb != cur_rb) { bi = p.bv[lr]; cur_rb = rb; }
            // ---- Theta tiles landed? (B1, B2, y' of this tile); S' = Xi' X^T ready in TMEM?
            mbar_wait(&bar->full[c.s], (uint32_t)c.ph);
            tc_check(p, bar->tagT[c.s] == c.u, TCC_THETA_EPI, c.u);
            if (tr) TC_TRACE(3 + wg, c.u, 1);
            mbar_wait(&bar->d1_full[b], (uint32_t)((c.u >> 1) & 1));
            if (tr) TC_TRACE(3 + wg, c.u, 2);
            mbar_wait(&bar->at_empty[b], (uint32_t)(((c.u >> 1) & 1) ^ 1));   // GEMM2 of tile u-2 done
            if (tr) TC_TRACE(3 + wg, c.u, 3);
            tc_fence_after();
            uint8_t *st = stage_ptr(c.s);
            const float *yt = reinterpret_cast<const float *>(yring + c.s * 128);
            uint8_t *rowB1 = st + r * 128, *rowB2 = st + TILE_BYTES + r * 128;
            const int64_t j0 = (int64_t)cb * TBN;
            // masks in tile-local 32-bit terms: the diagonal column (if in this tile), the
            // number of real columns, and whether this row exists
            const int64_t dg = p.row0 + lr - j0;
            const int dcol = (dg >= 0 && dg < TBN) ? (int)dg : -1;
            const int nvalid = (int)min((int64_t)TBN, p.N - j0);
            const bool row_ok = lr < p.Ns;
            // valid-column bit mask of this thread's row; 'dirty' warps (diagonal / tails) take a
            // separate, warp-uniform masking branch
            uint32_t vmask = row_ok ? (nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u)) : 0u;
            if (p.nbar > 1) {
                // partition (Assumption 1): no dual variable on the intra-block pairs
                const int64_t bs = (p.row0 + lr) - (p.row0 + lr) % p.nbar - j0;
                const int lo = (int)max(bs, (int64_t)0), hi = (int)min(bs + p.nbar, (int64_t)TBN);
                if (lo < hi) vmask &= ~((hi - lo >= 32 ? 0xffffffffu : ((1u << (hi - lo)) - 1u)) << lo);
            } else if (dcol >= 0) {
                vmask &= ~(1u << dcol);
            }
            const bool dirty = __any_sync(0xffffffffu, vmask != 0xffffffffu);
            float rtile = 0.f, dtile = 0.f;
            float *colw = my_colS + ((((c.u >> 1) & 1) * 4) + q) * 32;
            // two 16-column halves, rolled (keeps the loop body small: instruction-cache resident)
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                uint32_t sv[16];
                tmem_ld16(tmem + lane_off + c_d1 + (uint32_t)b * TBN + 16 * half, sv);
                tmem_wait_ld();
                if constexpr (f16) {                       // undo the fp16 scalings (exact: powers of 2)
                    const float rs = rowscale[(c.k & 1) * TBM + r];
#pragma unroll
                    for (int e = 0; e < 16; ++e) sv[e] = __float_as_uint(__uint_as_float(sv[e]) * rs);
                }
                float th[16];
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                    const int k = 4 * half + k4;                       // 16-byte chunk in the 128-B row
                    const int off = ((k ^ (r & 7)) << 4);
                    const float4 v1 = *reinterpret_cast<const float4 *>(rowB1 + off);
                    const float4 v2 = *reinterpret_cast<const float4 *>(rowB2 + off);
                    const float4 yv4 = *reinterpret_cast<const float4 *>(yt + 4 * k);
                    const float b1[4] = {v1.x, v1.y, v1.z, v1.w}, b2[4] = {v2.x, v2.y, v2.z, v2.w};
                    const float yj[4] = {yv4.x, yv4.y, yv4.z, yv4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float acc = __uint_as_float(sv[4 * k4 + e]) - (yj[e] + bi);   // -(C eta)_ij / L
                        // theta~ - (C eta)/L = b1 + (beta (b1 - b2) + acc): the inner rounding is at
                        // the scale of the update, so the stored value carries ~one rounding of theta
                        const float v = b1[e] + fmaf(beta, b1[e] - b2[e], acc);
                        th[4 * k4 + e] = fmaxf(v, 0.f);                                     // ( . )_+
                    }
                    if (dirty) {                                                            // diag / tails
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (!((vmask >> (4 * k + e)) & 1u)) th[4 * k4 + e] = 0.f;
                    }
                    if (adapt) {           // D = Theta^k - theta~ = (Theta^k - b1) - beta (b1 - b2)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float d = (th[4 * k4 + e] - b1[e]) - beta * (b1[e] - b2[e]);
                            dtile = fmaf(d, d, dtile);
                        }
                    }
                    *reinterpret_cast<float4 *>(rowB2 + off) =                              // in place, for the store
                        make_float4(th[4 * k4], th[4 * k4 + 1], th[4 * k4 + 2], th[4 * k4 + 3]);
                }
                // Theta^k (hi = tf32 rounding, lo = remainder) into TMEM: GEMM2's A operand
                {
                    uint32_t h[16], l[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const float hx = tf32_hi(th[e]);
                        h[e] = __float_as_uint(hx);
                        l[e] = __float_as_uint(th[e] - hx);
                    }
                    tmem_st16(tmem + lane_off + c_at + (uint32_t)b * 64 + 16 * half, h);
                    tmem_st16(tmem + lane_off + c_at + (uint32_t)b * 64 + 32 + 16 * half, l);
                }
                // row sum of the half (pairwise)
                {
                    float s8[8];
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) s8[cc] = th[cc] + th[cc + 8];
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) s8[cc] += s8[cc + 4];
                    rtile += (s8[0] + s8[2]) + (s8[1] + s8[3]);
                }
            }
            // column sums over this warp's 32 rows from the staged Theta^k tile: lane = column,
            // rows in a fixed order (conflict-free: the 128-B swizzle spreads a row over all banks):
            // four independent chains over the 8-row groups (rows 8m + rr share the swizzle rr),
            // combined pairwise -- a 4x shorter dependent-add chain than one running sum
            __syncwarp();
            {
                const uint8_t *tile = st + TILE_BYTES + q * 32 * 128 + (lane & 3) * 4;
                float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
                for (int rr = 0; rr < 8; ++rr) {
                    const uint8_t *a = tile + rr * 128 + (((lane >> 2) ^ rr) << 4);
                    c0 += *reinterpret_cast<const float *>(a);
                    c1 += *reinterpret_cast<const float *>(a + 8 * 128);
                    c2 += *reinterpret_cast<const float *>(a + 16 * 128);
                    c3 += *reinterpret_cast<const float *>(a + 24 * 128);
                }
                colw[lane] = (c0 + c1) + (c2 + c3);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (tr) TC_TRACE(3 + wg, c.u, 4);
            tc_tag(p, if (q == 0 && lane == 0) bar->tagAT[b] = c.u);
            {
                // rows of Theta^k are >= 0, so a row is all zero iff its fp32 sum is 0
                const uint32_t wnz = __any_sync(0xffffffffu, rtile != 0.f) ? 1u : 0u;
                if (lane == 0) *reinterpret_cast<volatile uint32_t *>(&bar->nzAT[b][q]) = wnz;   // before the release below
            }
            if (lane == 0) {
                mbar_arrive(&bar->d1_empty[b]);
                mbar_arrive(&bar->at_full[b]);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->st_full[c.s]);
            rrun += (double)rtile;
            drun += (double)dtile;
            named_barrier(1 + wg, 128);
            if (tr) TC_TRACE(3 + wg, c.u, 5);
            if (q == 0) {
                const float *cs = my_colS + ((c.u >> 1) & 1) * 4 * 32;
                const float c4 = (cs[lane] + cs[32 + lane]) + (cs[64 + lane] + cs[96 + lane]);
                p.colpart[(int64_t)rb * p.ldT + j0 + lane] = c4;
            }
            // ---- this warpgroup's last tile of the run: its row-sum partial into the slot
            Cursor n2 = c;
            adv(n2, 2);
            if (n2.u >= U || n2.rb != rb) {
                double *rp = p.rowpart + ((int64_t)(slot0 + rb - rbA) * TBM + r) * W;
                rp[NP2 + wg] = rrun;
                if (adapt) rp[NP2 + 2 + wg] = drun;
                if (run_start(c) && run_end(c)) {   // 1-tile run: the other warpgroup has no tile in
                    rp[NP2 + 1 - wg] = 0.0;         // it, so its columns are written here (every
                    if (adapt) rp[NP2 + 3 - wg] = 0.0;   // slot column is rewritten by every pass)
                }
                rrun = 0.0;
                drun = 0.0;
            }
            // ---- Theta X flushes (warpgroup 0 handles those after tiles u and u+1)
            if (wg == 0) {
                if (flush_after(c)) flush(c);
                Cursor n1 = c;
                adv(n1, 1);
                if (n1.u < U && flush_after(n1)) flush(n1);
            }
            if (tr) TC_TRACE(3 + wg, c.u, 6);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TC_TRACE(0, 0, 5);          // all roles done
    if (TC_TRACE_ON && p.trace && threadIdx.x == 0 && blockIdx.x < 1024) p.trace[kTraceTile + 4 * blockIdx.x + 2] = gtimer();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// Per-32-column-tile B-operand images (K-major, no swizzle: 8-row x 16-B core matrices):
//   g1 = X_J   [j][k]: tf32: byte ((k/4) * 4 + j/8) * 128 + (j%8) * 16 + (k%4) * 4,   NK * 128 B / tile
//                      fp16: byte ((k/8) * 4 + j/8) * 128 + (j%8) * 16 + (k%8) * 2,   NK16 * 64 B / tile
//                      (values x 2^xexp, hi = fp16 rounding, lo = fp16 of the remainder)
//   g2 = X_J^T [d][j]: byte ((j/4) * NP2/8 + d/8) * 128 + (d%8) * 16 + (j%4) * 4, NP2 * 128 B / tile
// hi = tf32 truncation, lo = remainder; k >= n, d >= n and j >= N hold 0.
__global__ void tc_images_kernel(const double *X64, int64_t N, int n, int NK, int NP2, int nCB, float *g1h,
                                 float *g1l, float *g2h, float *g2l, int g1f16, int xexp) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)nCB * TBN * NP2;
    if (e >= total) return;
    const int d = (int)(e % NP2);
    const int64_t j = e / NP2;
    const int64_t cb = j / TBN;
    const int jj = (int)(j % TBN);
    const float x = (j < N && d < n) ? (float)X64[j * n + d] : 0.f;
    const float h = tf32_hi(x), l = x - h;
    if (g1f16) {
        // d < NP2 = NK16
        const float xs = ldexpf(x, xexp);
        const __half xh = __float2half_rn(xs);
        const __half xl = __float2half_rn(xs - __half2float(xh));
        const int64_t o = cb * (int64_t)NP2 * 32 + ((d / 8) * 4 + jj / 8) * 64 + (jj % 8) * 8 + (d % 8);
        reinterpret_cast<__half *>(g1h)[o] = xh;
        reinterpret_cast<__half *>(g1l)[o] = xl;
    } else if (d < NK) {
        const int64_t o = cb * (int64_t)NK * 32 + ((d / 4) * 4 + jj / 8) * 32 + (jj % 8) * 4 + (d % 4);
        g1h[o] = h;
        g1l[o] = l;
    }
    const int64_t o2 = cb * (int64_t)NP2 * 32 + ((jj / 4) * (NP2 / 8) + d / 8) * 32 + (d % 8) * 4 + (jj % 4);
    g2h[o2] = h;
    g2l[o2] = l;
}

}  // namespace

#define CR_TC_NK_LIST(X) X(8) X(16) X(24) X(32) X(40) X(48) X(56) X(64) X(72) X(80)

cudaError_t launch_pass_tc(const TcParams &p, cudaStream_t s) {
    switch (p.NK) {
#define CR_CASE(V)                                                                                           \
    case V: {                                                                                                \
        const dim3 g(p.G), b(NTHR);                                                                          \
        const size_t sm = (size_t)p.smem_bytes;                                                              \
        cudaError_t e = p.g1f16 ? (p.check   ? pdl_launch(pass_tc_kernel<V, true, TC_CHECK>, g, b, sm, s, p)  \
                                   : p.yflag ? pdl_launch(pass_tc_kernel<V, true, TC_P2PY>, g, b, sm, s, p)   \
                                   : p.adapt ? pdl_launch(pass_tc_kernel<V, true, TC_ADAPT>, g, b, sm, s, p)  \
                                             : pdl_launch(pass_tc_kernel<V, true, TC_PLAIN>, g, b, sm, s, p)) \
                                : (p.check   ? pdl_launch(pass_tc_kernel<V, false, TC_CHECK>, g, b, sm, s, p) \
                                   : p.yflag ? pdl_launch(pass_tc_kernel<V, false, TC_P2PY>, g, b, sm, s, p)  \
                                   : p.adapt ? pdl_launch(pass_tc_kernel<V, false, TC_ADAPT>, g, b, sm, s, p) \
                                             : pdl_launch(pass_tc_kernel<V, false, TC_PLAIN>, g, b, sm, s, p)); \
        if (e != cudaSuccess) return e;                                                                      \
    } break;
        CR_TC_NK_LIST(CR_CASE)
#undef CR_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t pass_tc_prepare(int NK, int smem_bytes) {
    switch (NK) {
#define CR_CASE(V)                                                                                           \
    case V: {                                                                                                \
        const auto A = cudaFuncAttributeMaxDynamicSharedMemorySize;                                          \
        cudaError_t e = cudaFuncSetAttribute(pass_tc_kernel<V, false, TC_PLAIN>, A, smem_bytes);            \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(pass_tc_kernel<V, true, TC_PLAIN>, A, smem_bytes);   \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(pass_tc_kernel<V, true, TC_CHECK>, A, smem_bytes);   \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(pass_tc_kernel<V, true, TC_P2PY>, A, smem_bytes);    \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(pass_tc_kernel<V, false, TC_CHECK>, A, smem_bytes);  \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(pass_tc_kernel<V, false, TC_P2PY>, A, smem_bytes);   \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(pass_tc_kernel<V, true, TC_ADAPT>, A, smem_bytes);   \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(pass_tc_kernel<V, false, TC_ADAPT>, A, smem_bytes);  \
        return e;                                                                                            \
    }
        CR_TC_NK_LIST(CR_CASE)
#undef CR_CASE
        default: return cudaErrorInvalidValue;
    }
}

size_t tc_barrier_bytes() {
    return (size_t)kTcMaxStages * 128 + sizeof(TcBarriers) + 8 + 2 * 2 * 4 * 32 * 4 + 2 * TBM * 4;
}

cudaError_t launch_tc_images(const double *X64, int64_t N, int n, int NK, int NP2, int nCB, float *g1h, float *g1l,
                             float *g2h, float *g2l, int g1f16, int xexp, cudaStream_t s) {
    const int64_t total = (int64_t)nCB * TBN * NP2;
    tc_images_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(X64, N, n, NK, NP2, nCB, g1h, g1l, g2h, g2l,
                                                                      g1f16, xexp);
    return cudaGetLastError();
}

}  // namespace cr
