// accumulate.cu — a6: per-tile accumulation of the closed-form optical depth
// (Eq.2-4) over the bucketed occluders of each 8x8 tile
// (P:L173), then T = exp(-tau) (Eq.4) into the atlas [L][K][H][W].
//
// Design (DESIGN.md §6 "a6"):
//  * one CTA = 64 threads = one 8x8 tile; thread <-> texel; each thread owns
//    one column acc[k][texel] of a K x 64 shared-memory table (conflict-free:
//    the bank is the texel index);
//  * the tile's depth-sorted Gaussian list is cut into chunks (work units);
//    a persistent grid pulls units from an atomic counter; multi-chunk tiles
//    combine their partial tau deterministically (chunk order) in the CTA that
//    finishes last;
//  * the 96-B footprint records of the listed Gaussians are gathered into
//    shared memory with TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx),
//    32 per stage; a transform pass rewrites each staged record once per work
//    unit into a compact fp32 form relative to the tile's reference direction
//    (f = fl32(d_i - d_c)), which frees the TMA buffer for the next stage while
//    the CTA computes on the compact copy;
//  * per (texel, Gaussian) pair the delta-formulation (R9): delta = e_t - f,
//    a = |g + W delta|^2, r = c - b^2/a = D^2 |g x W delta|^2 / a and s* - D =
//    -D (u . W delta)/a, all without cancellation in fp32;
//  * fp32 erf saturates to +-1 exactly for |x| >= 3.92, so a pair contributes
//    pref*(erf(x_k) - erf(x_0)) only on the few shells of its "window" and the
//    constant pref*(1 - erf(x_0)) beyond it: window shells and the step are
//    written as differences into acc and a prefix sum over k restores tau_k.
//    No tensor cores: this is not a dense contraction (FP32 FMA + MUFU bound).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
constexpr int kThreads = kTexels / kTileSplit;  // one warp = one half of an 8x8 tile
constexpr int kStage = 32;        // records per pipeline stage

// Staging of the records (template kTMA): TMA bulk copies into a raw shared
// buffer (kTMA), or 16-B loads into registers one stage ahead (no raw buffer).
// launch_accumulate takes TMA unless the raw buffer costs a CTA per SM.
constexpr size_t kRawBytesTMA = kStage * 96;
// Records per stage of the single-table kernel (K <= 64): 24 keep its shared memory
// (16 KB table + 1.9 KB compact copy) within 12 CTAs/SM, the register limit at 80
// registers, where 32 allowed 11: cfg2 a6 0.930 -> 0.917 ms, cfg3 6.31 -> 6.19 ms
// (16 records: 0.926 ms; 64: 0.953 ms at 10 CTAs/SM).  The band kernel keeps 32
// (its band filter compacts one warp's ballot).
constexpr int kStageA = 24;
constexpr size_t kRawBytesTMA_A = kStageA * 96;
// Shell bands: K <= kTableRows runs k_accumulate with a K-row table; larger K runs
// k_accumulate_band, one pass per band of kBandRows shells over the records meeting
// it (DESIGN.md §6 a6).  48 rows (3 bands at K = 128) leave 12 CTAs/SM (the register
// limit) where 64 rows (2 bands) leave 11: cfg5 a6 48.7 -> 45.7 ms (32 / 40 / 43 / 56
// rows: 52.2 / 51.5 / 50.8 / 47.7 ms).
constexpr int kTableRows = 64;
constexpr int kBandRows = 48;
constexpr int kMinBandRows = 32;  // DGSM_BAND_ROWS (A/B) is clamped to [32, 256]
constexpr int kMaxBands = DGSM_MAX_SHELLS / kMinBandRows;
constexpr int kAccMinBlocks = 11;  // band kernel: caps registers at 80 (ptxas otherwise takes 96-168)

// One-warp CTAs synchronise with __syncwarp (no CTA barrier between the halves
// of a tile: each half is an independent work unit).
__device__ __forceinline__ void cta_sync() {
    if (kThreads == 32) __syncwarp(); else __syncthreads();
}
constexpr float kXS = 3.92f;      // |x| >= kXS  ->  erf_fast(x) == +-1 exactly

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// T = exp(-tau) (Eq.4) as one MUFU ex2: relative error ~2^-22 (|dT| < 3e-7), exactly 1 at
// tau = 0 and 0 below 2^-126; the same function in every epilogue and in k_exp.
__device__ __forceinline__ float t_of_tau(float tau) { return ex2_approx(-1.4426950408889634f * tau); }
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Window bounds: ceil(kf) for kf in [0, K] as round-to-nearest(kf + 1/2) through
// the 1.5 * 2^23 magic constant (FADD instead of F2I/I2F on the XU pipe).  It is
// ceil(kf) + 1 when kf + 1/2 is a tie rounding up (kf an exact integer): the
// window then drops (klo) or adds (khi) one boundary shell with |x_k| = 3.92 up
// to rounding, whose erf is +-1 to 3e-8 either way.
constexpr float kMagic = 12582912.0f;
constexpr int kMagicBits = 0x4B400000;
__device__ __forceinline__ float win_round(float kfh, int K) {  // kfh = kf + 1/2
    return fminf(fmaxf(kfh, 0.0f), (float)K) + kMagic;
}
// band kernel: the window clamped to [wlo, whi] (the band's rows and its two dump
// rows), in the integer domain of the rounded value's bits: LO/HI = kMagicBits +
// wlo/whi are CTA-uniform integers (uniform registers).  Any kfh, even far out of
// the magic constant's range or NaN, lands in [wlo, whi].
__device__ __forceinline__ float win_round_b(float kfh, int LO, int HI) {
    return __int_as_float(min(max(__float_as_int(kfh + kMagic), LO), HI));
}
__device__ __forceinline__ f2_t win_round2_b(f2_t KFH, int LO, int HI) {
    const f2_t Y = f2add(KFH, f2bc(kMagic));
    return f2pack(__int_as_float(min(max(__float_as_int(f2lo(Y)), LO), HI)),
                  __int_as_float(min(max(__float_as_int(f2hi(Y)), LO), HI)));
}
__device__ __forceinline__ f2_t win_round2(f2_t KFH, int K) {
    const float fK = (float)K;
    return f2add(f2pack(fminf(fmaxf(f2lo(KFH), 0.0f), fK), fminf(fmaxf(f2hi(KFH), 0.0f), fK)), f2bc(kMagic));
}

// fp32 erf, branch-free: 1 - 2^Q(|x|) with Q of degree 7 on [0, 3.92]
// (max abs error 3.8e-7, tools/fit_erf.py 7), exactly +-1 for |x| >= 3.92.
// Error budget: |d tau| <= 2 * 3.8e-7 * sum(pref) -> < 1e-5 in T for tau <~ 10.
__device__ __forceinline__ float erf_fast(float x) {
    const float t = fminf(fabsf(x), kXS);
    float q = 6.113672134e-05f;
    q = fmaf(q, t, -2.010886819e-04f);
    q = fmaf(q, t, -2.966491506e-03f);
    q = fmaf(q, t, 3.027309850e-02f);
    q = fmaf(q, t, -1.494759023e-01f);
    q = fmaf(q, t, -9.181758761e-01f);
    q = fmaf(q, t, -1.627931952e+00f);
    q = fmaf(q, t, 5.166708092e-07f);
    // saturated: 2^-256 flushes to 0, so r == 1 exactly without a branch
    q = t >= kXS ? -256.0f : q;
    const float r = 1.0f - ex2_approx(q);
    return copysignf(r, x);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// TMA bulk copy global -> shared, completion counted on the mbarrier (bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// Texel-centre direction d(u_c, v_c) (R3), fp64.
__device__ __forceinline__ void texel_dir(int row, int col, int W, int H, double& d0, double& d1,
                                          double& d2) {
    const double uc = (col + 0.5) * 2.0 / W - 1.0;
    const double vc = (row + 0.5) * 2.0 / H - 1.0;
    double x = uc, y = vc;
    const double z = 1.0 - fabs(uc) - fabs(vc);
    if (z < 0.0) {
        x = (uc >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(vc));
        y = (vc >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(uc));
    }
    const double inv = 1.0 / sqrt(x * x + y * y + z * z);
    d0 = x * inv; d1 = y * inv; d2 = z * inv;
}

struct AccLights {
    float dt[DGSM_MAX_LIGHTS];     // t_max / K (fp32)
    float dtlo[DGSM_MAX_LIGHTS];   // t_max / K - dt (fp64 remainder)
    float idt[DGSM_MAX_LIGHTS];    // 1 / dt
};

// Compact per-(record, work unit) form: 20 fp32 fields (80 B) relative to the
// tile reference direction d_c, stored interleaved by record pairs (below).
constexpr int kCompact = 5;  // float4 per record

// s_acc read-modify-write through a 32-bit shared address (the generic pointer
// form had the shared window base recomputed on every use)
__device__ __forceinline__ void acc_add(uint32_t a, float v) {
    float x;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a) : "memory");
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x + v) : "memory");
}

// ---- per (texel, Gaussian) pair ---------------------------------------------
// delta-formulation (R9) of a (texel, record) pair up to the negligible-pair
// test (R8'): W delta, u = g + W delta, a = |u|^2, |g x W delta|^2 and u . W delta.

// ---- two records at once on the paired-FP32 pipe (sm_100 FFMA2/FADD2/FMUL2) --
// A packed value holds record A (even) in the low half and record B (odd) in
// the high half; one f32x2 instruction does both records' operation, halving
// the issue slots of the pair test (the kernel is issue/latency bound).
__device__ __forceinline__ void lds_f2x2(uint32_t a, f2_t& x, f2_t& y) {
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a) : "memory");
}

// Compact record pair: 20 packed fields (A, B), 160 B; field order
//  0-2 -W f (f = fl32(d_i - d_c)), 3 r_cut/D^2, 4-6 g = W d_i, 7 -D, 8-16 W (row-major),
//  17 e_D, 18 beta sqrt(pi/2), 19 k_D (int bits)
constexpr int kPairFields = 20;
constexpr int kPairBytes = kPairFields * 8;

struct PairTest2 {
    f2_t A, C2, DOT;      // a = |u|^2, |g x W delta|^2, u . W delta  (records A | B)
    f2_t ND, ED, BP;      // -D, e_D, beta sqrt(pi/2)
    f2_t KD;              // anchor shell k_D (as float)
    bool liveA, liveB;
};

__device__ __forceinline__ PairTest2 pair_test2(uint32_t addr, f2_t ETX, f2_t ETY, f2_t ETZ) {
    f2_t F[kPairFields];
#pragma unroll
    for (int j = 0; j < kPairFields / 2; ++j) lds_f2x2(addr + 16 * j, F[2 * j], F[2 * j + 1]);
    // W delta = W e_t - W f: one FMA chain from the record's -W f
    const f2_t WX = f2fma(F[8], ETX, f2fma(F[9], ETY, f2fma(F[10], ETZ, F[0])));
    const f2_t WY = f2fma(F[11], ETX, f2fma(F[12], ETY, f2fma(F[13], ETZ, F[1])));
    const f2_t WZ = f2fma(F[14], ETX, f2fma(F[15], ETY, f2fma(F[16], ETZ, F[2])));
    const f2_t UX = f2add(F[4], WX), UY = f2add(F[5], WY), UZ = f2add(F[6], WZ);
    const f2_t A = f2fma(UX, UX, f2fma(UY, UY, f2mul(UZ, UZ)));
    const f2_t Z = 0ull;
    const f2_t NGX = f2sub(Z, F[4]), NGY = f2sub(Z, F[5]), NGZ = f2sub(Z, F[6]);
    const f2_t CX = f2fma(F[5], WZ, f2mul(NGZ, WY));  // gy wz - gz wy
    const f2_t CY = f2fma(F[6], WX, f2mul(NGX, WZ));  // gz wx - gx wz
    const f2_t CZ = f2fma(F[4], WY, f2mul(NGY, WX));  // gx wy - gy wx
    const f2_t C2 = f2fma(CX, CX, f2fma(CY, CY, f2mul(CZ, CZ)));
    const f2_t T = f2mul(F[3], A);  // live  <=>  |g x W delta|^2 <= (r_cut/D^2) a
    PairTest2 R;
    R.A = A;
    R.C2 = C2;
    R.DOT = f2fma(UX, WX, f2fma(UY, WY, f2mul(UZ, WZ)));  // u . W delta (closest approach)
    R.ND = F[7]; R.ED = F[17]; R.BP = F[18];
    R.KD = F[19];
    R.liveA = f2lo(C2) <= f2lo(T);
    R.liveB = f2hi(C2) <= f2hi(T);
    return R;
}

// Shell bands (band kernel, K > band rows): the table holds the band's rows
// [kb0, kb0 + nrows) plus a dump row on each side, at kb0 - 1 (bands > 0) and
// kb0 + nrows; every window is clamped to [wlo, whi] = [max(kb0 - 1, 0), kb0 + nrows],
// so the first in-band difference is taken against the true value at kb0 - 1,
// shells beyond the band are never evaluated, and writes outside the band land in
// a dump row (acc_base points at row kb0 - 1 minus kb0 - 1 rows).
// Statistics count only in-band work (kStats).
template <bool kBand>
__device__ __forceinline__ uint32_t band_count(int klo, int khi, int kb0, int nrows) {
    if (!kBand) return (uint32_t)(khi - klo);
    const int a = max(klo, kb0), b = min(khi, kb0 + nrows);
    return b > a ? (uint32_t)(b - a) : 0u;
}
__device__ __forceinline__ bool band_live(int khi, int kb0, int nrows, int K) {  // count a live pair once
    return khi >= kb0 && (khi < kb0 + nrows || khi == K);
}

// The same live path executed by the whole warp when any lane is live
// (uniform branch, straight-line body): lanes that are not live compute and
// discard.  The first window shell is evaluated unconditionally, further
// shells in a rarely taken loop.
template <bool kStats, bool kBand>
__device__ __forceinline__ void pair_live_warp(float pa, float pc2, float pdot, bool live, float ND, float eD,
                                               float betap, float kD, uint32_t acc_base, int K, float dt, float dtlo, float idt,
                                               int kb0, int nrows, int wlo, int whi,
                                               uint32_t& st_live, uint32_t& st_win, uint32_t& st_step) {
    const float ia = rcp_approx(pa);
    const float r_over_D2 = pc2 * ia;
    const float qd = ND * ND * -0.72134752044448170f;  // -D^2 log2(e)/2, off the MUFU chain
    const float sD = ND * pdot * ia;  // s* - D (ND = -D)
    const float ra = rsqrt_approx(pa);
    const float h = 0.70710678118654752f * pa * ra;
    const float x0 = h * (ND - sD);  // -h (D + s* - D)
    float e0 = -1.0f;
    if (__any_sync(0xffffffffu, x0 > -kXS)) {  // a Gaussian near the light (rare): uniform branch
        const float t = erf_fast(x0);
        if (x0 > -kXS) e0 = t;
    }
    live = live && e0 < 1.0f;
    const float pref = betap * ra * ex2_approx(kBand ? -0.72134752044448170f * (r_over_D2 * ND * ND) : r_over_D2 * qd);
    const float e = eD - sD;
    const float xsh = (kXS * 1.41421356237309505f) * ra;
    // window [klo, khi): ceil of the clamped bounds by round-to-nearest of kf + 1/2 (win_round)
    const float kdh = kD + 0.5f;
    const float ylo = kBand ? win_round_b(fmaf(-xsh - e, idt, kdh), wlo, whi) : win_round(fmaf(-xsh - e, idt, kdh), K);
    const float yhi = kBand ? win_round_b(fmaf(xsh - e, idt, kdh), wlo, whi) : win_round(fmaf(xsh - e, idt, kdh), K);
    const int klo = __float_as_int(ylo) - kMagicBits;
    const int khi = max(__float_as_int(yhi) - kMagicBits, klo);
    const int n = live ? khi - klo : 0;
    const bool step = kBand ? live : (live && khi < K);
    if (kStats) {
        st_live += live && (!kBand || band_live(khi, kb0, nrows, K));
        st_win += band_count<kBand>(klo, klo + n, kb0, nrows);
        st_step += (step && khi < K && (!kBand || (khi >= kb0 && khi < kb0 + nrows))) ? 1u : 0u;
    }
    float fk = kBand ? (ylo - kMagic) - kD : ylo - (kD + kMagic);  // (the same: integers below 2^24)
    uint32_t ap = acc_base + (uint32_t)klo * (kThreads * 4);
    const float tk1 = fmaf(fk, dt, fmaf(fk, dtlo, e));
    const float w1 = pref * (erf_fast(h * tk1) - e0);
    float prev = 0.0f;
    if (n >= 1) { acc_add(ap, w1); prev = w1; }
    if (__any_sync(0xffffffffu, n > 1)) {
        fk += 1.0f;
        ap += kThreads * 4;
#pragma unroll 1
        for (int i = 1; i < n; ++i, fk += 1.0f, ap += kThreads * 4) {
            const float tk = fmaf(fk, dt, fmaf(fk, dtlo, e));
            const float w = pref * (erf_fast(h * tk) - e0);
            acc_add(ap, w - prev);
            prev = w;
        }
    }
    if (step) acc_add(acc_base + (uint32_t)khi * (kThreads * 4), fmaf(pref, 1.0f - e0, -prev));
}


// erf_fast of both halves: the polynomial on the paired pipe, clamp/select and
// the MUFU ex2 per half
__device__ __forceinline__ f2_t erf_fast2(f2_t X) {
    const float xa = f2lo(X), xb = f2hi(X);
    const float ta = fminf(fabsf(xa), kXS), tb = fminf(fabsf(xb), kXS);
    const f2_t Tt = f2pack(ta, tb);
    f2_t q = f2bc(6.113672134e-05f);
    q = f2fma(q, Tt, f2bc(-2.010886819e-04f));
    q = f2fma(q, Tt, f2bc(-2.966491506e-03f));
    q = f2fma(q, Tt, f2bc(3.027309850e-02f));
    q = f2fma(q, Tt, f2bc(-1.494759023e-01f));
    q = f2fma(q, Tt, f2bc(-9.181758761e-01f));
    q = f2fma(q, Tt, f2bc(-1.627931952e+00f));
    q = f2fma(q, Tt, f2bc(5.166708092e-07f));
    const float qa = ta >= kXS ? -256.0f : f2lo(q), qb = tb >= kXS ? -256.0f : f2hi(q);
    return f2pack(copysignf(1.0f - ex2_approx(qa), xa), copysignf(1.0f - ex2_approx(qb), xb));
}

// Window + step of one record after the shared setup (scalar: the rare longer
// windows and the ordered shared-memory updates).
template <bool kStats, bool kBand>
__device__ __forceinline__ void live_finish(bool live, int klo, int khi, float fk, float w1, float pref, float h,
                                            float e, float e0, uint32_t acc_base, int K, float dt, float dtlo,
                                            int kb0, int nrows,
                                            uint32_t& st_live, uint32_t& st_win, uint32_t& st_step) {
    const int n = live ? khi - klo : 0;
    const bool step = kBand ? live : (live && khi < K);
    if (kStats) {
        st_live += live && (!kBand || band_live(khi, kb0, nrows, K));
        st_win += band_count<kBand>(klo, klo + n, kb0, nrows);
        st_step += (step && khi < K && (!kBand || (khi >= kb0 && khi < kb0 + nrows))) ? 1u : 0u;
    }
    uint32_t ap = acc_base + (uint32_t)klo * (kThreads * 4);
    float prev = 0.0f;
    if (n >= 1) { acc_add(ap, w1); prev = w1; }
    if (__any_sync(0xffffffffu, n > 1)) {
        fk += 1.0f;
        ap += kThreads * 4;
#pragma unroll 1
        for (int i = 1; i < n; ++i, fk += 1.0f, ap += kThreads * 4) {
            const float tk = fmaf(fk, dt, fmaf(fk, dtlo, e));
            const float w = pref * (erf_fast(h * tk) - e0);
            acc_add(ap, w - prev);
            prev = w;
        }
    }
    if (step) acc_add(acc_base + (uint32_t)khi * (kThreads * 4), fmaf(pref, 1.0f - e0, -prev));
}

// Both records of the pair have a live lane in this warp: the setup and the
// first window shell of both on the paired-FP32 pipe, then the per-record
// updates in record order (A before B: the summation order of the scalar path).
// Two (texel, record) pairs at once on the paired FP32 pipe: two records at one
// texel (the two-warp kernel) or one record at two texels (the one-warp kernel).
// Setup and first window shell packed; the shared-memory updates per half, A
// before B (the summation order of the scalar path when both are one texel).
template <bool kStats, bool kBand>
__device__ __forceinline__ void live_packed(f2_t A2, f2_t C2, f2_t DOT, f2_t ND2, f2_t ED2, f2_t BP2, f2_t KD,
                                            bool liveA_in, bool liveB_in, uint32_t baseA, uint32_t baseB, int K,
                                            float dt, float dtlo, float idt, int kb0, int nrows, int wlo, int whi,
                                            uint32_t& st_live, uint32_t& st_win, uint32_t& st_step) {
    const float aA = f2lo(A2), aB = f2hi(A2);
    const f2_t IA = f2pack(rcp_approx(aA), rcp_approx(aB));
    const f2_t RA = f2pack(rsqrt_approx(aA), rsqrt_approx(aB));
    // single-table kernel: -r log2(e)/2 as (|g x W delta|^2 / a) (-D^2 log2(e)/2), the D
    // factor off the MUFU chain (cfg2 a6 -0.4 %; the band kernel measured +1 % with it)
    const f2_t QD = f2mul(f2mul(ND2, ND2), f2bc(-0.72134752044448170f));
    const f2_t SD = f2mul(f2mul(ND2, DOT), IA);  // s* - D = -D (u . W delta) / a
    const f2_t H = f2mul(f2mul(f2bc(0.70710678118654752f), A2), RA);
    const f2_t X0 = f2mul(H, f2sub(ND2, SD));  // -h (D + s* - D)
    float e0A = -1.0f, e0B = -1.0f;
    const float x0A = f2lo(X0), x0B = f2hi(X0);
    if (__any_sync(0xffffffffu, x0A > -kXS || x0B > -kXS)) {
        const float ta = erf_fast(x0A), tb = erf_fast(x0B);
        if (x0A > -kXS) e0A = ta;
        if (x0B > -kXS) e0B = tb;
    }
    const bool liveA = liveA_in && e0A < 1.0f, liveB = liveB_in && e0B < 1.0f;
    const f2_t E0 = f2pack(e0A, e0B);
    const f2_t M = kBand ? f2mul(f2bc(-0.72134752044448170f), f2mul(f2mul(f2mul(C2, IA), ND2), ND2))
                         : f2mul(f2mul(C2, IA), QD);
    const f2_t PREF = f2mul(f2mul(BP2, RA), f2pack(ex2_approx(f2lo(M)), ex2_approx(f2hi(M))));
    const f2_t E = f2sub(ED2, SD);
    const f2_t XSH = f2mul(f2bc(kXS * 1.41421356237309505f), RA);
    const f2_t KDH = f2add(KD, f2bc(0.5f));
    const f2_t KLO = f2fma(f2add(XSH, E), f2bc(-idt), KDH);
    const f2_t KHI = f2fma(f2sub(XSH, E), f2bc(idt), KDH);
    const f2_t YLO = kBand ? win_round2_b(KLO, wlo, whi) : win_round2(KLO, K);
    const f2_t YHI = kBand ? win_round2_b(KHI, wlo, whi) : win_round2(KHI, K);
    const int kloA = __float_as_int(f2lo(YLO)) - kMagicBits, kloB = __float_as_int(f2hi(YLO)) - kMagicBits;
    const int khiA = max(__float_as_int(f2lo(YHI)) - kMagicBits, kloA);
    const int khiB = max(__float_as_int(f2hi(YHI)) - kMagicBits, kloB);
    const f2_t FK = kBand ? f2sub(f2sub(YLO, f2bc(kMagic)), KD)
                          : f2sub(YLO, f2add(KD, f2bc(kMagic)));  // (the same: integers below 2^24)
    const f2_t TK1 = f2fma(FK, f2bc(dt), f2fma(FK, f2bc(dtlo), E));
    const f2_t W1 = f2mul(PREF, f2sub(erf_fast2(f2mul(H, TK1)), E0));
    live_finish<kStats, kBand>(liveA, kloA, khiA, f2lo(FK), f2lo(W1), f2lo(PREF), f2lo(H), f2lo(E), e0A, baseA, K,
                               dt, dtlo, kb0, nrows, st_live, st_win, st_step);
    live_finish<kStats, kBand>(liveB, kloB, khiB, f2hi(FK), f2hi(W1), f2hi(PREF), f2hi(H), f2hi(E), e0B, baseB, K,
                               dt, dtlo, kb0, nrows, st_live, st_win, st_step);
}

template <bool kStats, bool kBand>
__device__ __forceinline__ void pair_live_warp2(const PairTest2& T, uint32_t acc_base, int K, float dt, float dtlo,
                                                float idt, int kb0, int nrows, int wlo, int whi, uint32_t& st_live,
                                                uint32_t& st_win, uint32_t& st_step) {
    live_packed<kStats, kBand>(T.A, T.C2, T.DOT, T.ND, T.ED, T.BP, T.KD, T.liveA, T.liveB, acc_base, acc_base, K, dt,
                               dtlo, idt, kb0, nrows, wlo, whi, st_live, st_win, st_step);
}

template <bool kStats, bool kTMA>
// (no min-blocks bound: 72 registers; forcing 11 CTAs/SM capped it at 80 with
// extra instructions in the live path, and a wider combine batch raised it)
__global__ void __launch_bounds__(kThreads) k_accumulate(  // 11 CTAs/SM at K = 64 (80 registers)
    const WorkUnit* __restrict__ units, const uint32_t* __restrict__ n_units_dev,
    const uint32_t* __restrict__ vals, const PairRec* __restrict__ recs, int64_t n, AccLights al,
    int res, int K, uint32_t flags, float* __restrict__ scratch, uint32_t* tile_arrive,
    uint32_t* unit_counter, float* __restrict__ atlas, unsigned long long* __restrict__ stats,
    const uint64_t* __restrict__ slab_mask, const int2* __restrict__ slab_k) {
    pdl_begin();
    extern __shared__ __align__(128) unsigned char acc_smem[];
    constexpr size_t kRawBytes = kTMA ? kRawBytesTMA_A : 0;
    PairRec* s_raw = reinterpret_cast<PairRec*>(acc_smem);                                   // [kStageA] (TMA)
    float4* s_cr = reinterpret_cast<float4*>(acc_smem + kRawBytes);                          // [kStageA][5]
    float* s_acc = reinterpret_cast<float*>(acc_smem + kRawBytes + kStageA * kCompact * sizeof(float4));  // [K][64]
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_unit, s_last;

    const int tid = threadIdx.x;
    if (kTMA && tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t phase = 0u;
    cta_sync();
    const uint32_t n_units = *n_units_dev;
    const int TW = res / kTile;
    const int n_tiles = TW * TW;
    const int W = res, H = res;

    for (;;) {
        if (tid == 0) s_unit = atomicAdd(unit_counter, 1u);
        cta_sync();
        const uint32_t u = s_unit;
        if (u >= n_units) break;
        const WorkUnit wu = units[u];
        const int l = (int)(wu.tile / (uint32_t)n_tiles);
        const int tile = (int)(wu.tile - (uint32_t)l * n_tiles);
        const int row0 = (tile / TW) * kTile, col0 = (tile % TW) * kTile;
        const int tt = (int)wu.part * kThreads + tid;  // texel index within the tile
        const int row = row0 + (tt >> 3);
        const int col = col0 + (tt & 7);
        const uint32_t tslot = wu.tile * kTileSplit + wu.part;  // (tile, part) arrival counter

        // texel direction relative to the tile reference direction d_c (fp64 -> fp32)
        double c0, c1, c2, t0, t1, t2;
        texel_dir(row0 + 4, col0 + 4, W, H, c0, c1, c2);
        texel_dir(row, col, W, H, t0, t1, t2);
        const float etx = (float)(t0 - c0), ety = (float)(t1 - c1), etz = (float)(t2 - c2);
        const f2_t ETX = f2pack(etx, etx), ETY = f2pack(ety, ety), ETZ = f2pack(etz, etz);
        for (int k = 0; k < K; ++k) s_acc[k * kThreads + tid] = 0.0f;
        const uint32_t acc_base = smem_addr(s_acc) + 4u * (uint32_t)tid;  // &s_acc[0][tid]
        uint32_t st_live = 0, st_win = 0, st_step = 0, st_wany = 0, st_wmax = 0;

        const float dt = al.dt[l], dtlo = al.dtlo[l], idt = al.idt[l];
        const uint32_t n_rec = wu.jend - wu.jbeg;
        const uint32_t n_batches = (n_rec + kStageA - 1) / kStageA;
        const PairRec* lrecs = recs + (int64_t)l * n;

        auto issue = [&](uint32_t b) {  // TMA: bulk copies of the stage's records into s_raw
            const uint32_t j0 = wu.jbeg + b * kStageA;
            const uint32_t nb = min((uint32_t)kStageA, wu.jend - j0);
            if (tid == 0) mbar_arrive_expect_tx(&s_bar, nb * (uint32_t)sizeof(PairRec));
            if ((uint32_t)tid < nb) {
                const uint32_t gi = vals[j0 + tid];
                bulk_g2s(s_raw + tid, lrecs + gi, (uint32_t)sizeof(PairRec), &s_bar);
            }
        };
        // register staging: thread t < 32 holds record t of the next stage (6 x 16-B
        // loads issued before the current stage's compute)
        uint4 ru[6];  // PairRec as six 16-B words (no union: the loads land in place)
        auto fetch = [&](uint32_t b) {
            const uint32_t j0 = wu.jbeg + b * kStageA;
            if ((uint32_t)tid < min((uint32_t)kStageA, wu.jend - j0)) {
                const uint4* src = reinterpret_cast<const uint4*>(lrecs + vals[j0 + tid]);
#pragma unroll
                for (int k = 0; k < 6; ++k) ru[k] = __ldg(src + k);
            }
        };
        if (n_batches > 0) {
            if (kTMA) issue(0); else fetch(0);
        }

        for (uint32_t b = 0; b < n_batches; ++b) {
            if (kTMA) {
                mbar_wait(&s_bar, phase);
                phase ^= 1u;
            }
            const uint32_t nb = min((uint32_t)kStageA, n_rec - b * kStageA);
            if ((uint32_t)tid < nb) {  // transform: raw record -> compact, relative to d_c
                float* q = reinterpret_cast<float*>(s_cr) + (tid >> 1) * (2 * kPairFields) + (tid & 1);
                float v[kPairFields];
                if (kTMA) {
                    const PairRec& R = s_raw[tid];
                    const float vv[kPairFields] = {(float)(R.di[0] - c0), (float)(R.di[1] - c1), (float)(R.di[2] - c2),
                                                   R.rcut_D2, R.g[0], R.g[1], R.g[2], R.D,
                                                   R.W[0], R.W[1], R.W[2], R.W[3], R.W[4], R.W[5], R.W[6], R.W[7],
                                                   R.W[8], R.eD, R.betap, (float)R.kD};
#pragma unroll
                    for (int f = 0; f < kPairFields; ++f) v[f] = vv[f];
                } else {  // field offsets of PairRec (static_assert'ed 96 B layout)
                    const float vv[kPairFields] = {
                        (float)(__hiloint2double((int)ru[0].y, (int)ru[0].x) - c0),
                        (float)(__hiloint2double((int)ru[0].w, (int)ru[0].z) - c1),
                        (float)(__hiloint2double((int)ru[1].y, (int)ru[1].x) - c2),
                        __uint_as_float(ru[5].z),                                                   // rcut_D2
                        __uint_as_float(ru[1].z), __uint_as_float(ru[1].w), __uint_as_float(ru[2].x),  // g
                        __uint_as_float(ru[4].z),                                                   // D
                        __uint_as_float(ru[2].y), __uint_as_float(ru[2].z), __uint_as_float(ru[2].w),  // W
                        __uint_as_float(ru[3].x), __uint_as_float(ru[3].y), __uint_as_float(ru[3].z),
                        __uint_as_float(ru[3].w), __uint_as_float(ru[4].x), __uint_as_float(ru[4].y),
                        __uint_as_float(ru[4].w),                                                   // eD
                        __uint_as_float(ru[5].y),                                                   // betap
                        (float)(int)ru[5].x};                                                       // kD
#pragma unroll
                    for (int f = 0; f < kPairFields; ++f) v[f] = vv[f];
                }
                {  // fields 0-2: -W f, f = d_i - d_c (the pair test forms W delta = W e_t - W f); 7: -D
                    const float f0 = v[0], f1 = v[1], f2 = v[2];
                    v[0] = -fmaf(v[8], f0, fmaf(v[9], f1, v[10] * f2));
                    v[1] = -fmaf(v[11], f0, fmaf(v[12], f1, v[13] * f2));
                    v[2] = -fmaf(v[14], f0, fmaf(v[15], f1, v[16] * f2));
                    v[7] = -v[7];
                }
#pragma unroll
                for (int f = 0; f < kPairFields; ++f) q[2 * f] = v[f];
            }
            cta_sync();  // compact copy ready; raw buffer free
            if (b + 1 < n_batches) {
                if (kTMA) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(b + 1);
                } else {
                    fetch(b + 1);
                }
            }
            // two records per iteration: independent dependency chains for the pair test
            uint32_t my_live = 0;
            auto process = [&](PairTest2& T2) {
                if (kStats) {
                    const uint32_t ba = __ballot_sync(0xffffffffu, T2.liveA), bb = __ballot_sync(0xffffffffu, T2.liveB);
                    my_live += (uint32_t)T2.liveA + (uint32_t)T2.liveB;
                    st_wany += (ba != 0u) + (bb != 0u);
                }
                const bool anyA = __any_sync(0xffffffffu, T2.liveA), anyB = __any_sync(0xffffffffu, T2.liveB);
                if (anyA && anyB) {
                    pair_live_warp2<kStats, false>(T2, acc_base, K, dt, dtlo, idt, 0, K, 0, 0, st_live, st_win, st_step);
                    return;
                }
                if (anyA)
                    pair_live_warp<kStats, false>(f2lo(T2.A), f2lo(T2.C2), f2lo(T2.DOT), T2.liveA, f2lo(T2.ND),
                                                  f2lo(T2.ED), f2lo(T2.BP), f2lo(T2.KD), acc_base, K, dt, dtlo, idt, 0, K,
                                                  0, 0, st_live, st_win, st_step);
                if (anyB)
                    pair_live_warp<kStats, false>(f2hi(T2.A), f2hi(T2.C2), f2hi(T2.DOT), T2.liveB, f2hi(T2.ND),
                                                  f2hi(T2.ED), f2hi(T2.BP), f2hi(T2.KD), acc_base, K, dt, dtlo, idt, 0, K,
                                                  0, 0, st_live, st_win, st_step);
            };
            uint32_t pr_addr = smem_addr(s_cr);  // induction variable: record pair (r, r+1)
            uint32_t r = 0;
            // two record pairs' tests per iteration (twice the independent chains:
            // 0.95 -> 0.93 ms at 80 registers; four pairs need 128 and are slower)
            for (; r + 2 < nb; r += 4, pr_addr += 2 * kPairBytes) {
                PairTest2 Ta = pair_test2(pr_addr, ETX, ETY, ETZ);
                PairTest2 Tb = pair_test2(pr_addr + kPairBytes, ETX, ETY, ETZ);
                Tb.liveB = Tb.liveB && (r + 3 < nb);
                process(Ta);
                process(Tb);
            }
            for (; r < nb; r += 2, pr_addr += kPairBytes) {
                PairTest2 T2 = pair_test2(pr_addr, ETX, ETY, ETZ);
                T2.liveB = T2.liveB && (r + 1 < nb);
                process(T2);
            }
            if (kStats) st_wmax += __reduce_max_sync(0xffffffffu, my_live);
            cta_sync();  // compact copy consumed
        }

        if (kStats) {
            atomicAdd(&stats[1], (unsigned long long)st_live);
            atomicAdd(&stats[2], (unsigned long long)st_win);
            atomicAdd(&stats[3], (unsigned long long)st_step);
            if (tid == 0) {
                atomicAdd(&stats[0], (unsigned long long)n_rec * kThreads);
                atomicAdd(&stats[7], (unsigned long long)n_rec);  // records run through the pair tests
            }
            // warp-level: records entering the live path (any lane live) and the
            // per-stage max over lanes of live records (what a per-lane loop would cost)
            if ((tid & 31) == 0) {
                atomicAdd(&stats[4], (unsigned long long)n_rec);
                atomicAdd(&stats[5], (unsigned long long)st_wany);
                atomicAdd(&stats[6], (unsigned long long)st_wmax);
            }
        }
        // prefix sum over shells -> tau_k; epilogue T = exp(-tau) (Eq.4)
        const bool want_tau = (flags & DGSM_OUTPUT_TAU) != 0;
        const size_t plane = (size_t)H * W;
        float* out = atlas + ((size_t)l * K) * plane + (size_t)row * W + col;
        // NEXT-1 slab: outside P x [k_min, k_max] the table stays T = 1
        int klo = 0, khi = K - 1;
        if (slab_mask) {
            const int2 kr = slab_k[l];
            klo = kr.x;
            khi = ((slab_mask[wu.tile] >> tt) & 1ull) ? kr.y : -1;
        }
        const float one = want_tau ? 0.0f : 1.0f;
        if (wu.nchunks == 1) {
            float tau = 0.0f;
            // (one loop: a separate select-free path for the common case costs this
            // kernel 16 registers; the band kernel has one)
            for (int k = 0; k < K; ++k) {
                tau += s_acc[k * kThreads + tid];
                out[(size_t)k * plane] = (k < klo || k > khi) ? one : (want_tau ? tau : t_of_tau(tau));
            }
        } else {
            float* part = scratch + ((size_t)(wu.slot + wu.chunk) * K) * kThreads + tid;
            float tau = 0.0f;
            for (int k = 0; k < K; ++k) {
                tau += s_acc[k * kThreads + tid];
                part[(size_t)k * kThreads] = tau;
            }
            __threadfence();
            cta_sync();
            // (tiles of more than kInlineCombine chunks: k_combine_deferred sums them)
            if (tid == 0) s_last = wu.nchunks <= kInlineCombine &&
                                   atomicAdd(&tile_arrive[tslot], 1u) == wu.nchunks - 1 ? 1u : 0u;
            cta_sync();
            if (s_last) {
                __threadfence();
                const float* base = scratch + ((size_t)wu.slot * K) * kThreads + tid;
                // kCB shells at a time: kCB independent L2 loads per chunk in flight
                // (the summation order per shell stays chunk 0, 1, ...: deterministic)
                constexpr int kCB = 4;  // 2: slower; 6, 16: more registers for the whole kernel
                for (int k0 = 0; k0 < K; k0 += kCB) {
                    float t[kCB];
#pragma unroll
                    for (int u = 0; u < kCB; ++u) t[u] = 0.0f;
                    for (uint32_t c = 0; c < wu.nchunks; ++c) {
                        const float* pc = base + ((size_t)c * K + k0) * kThreads;
#pragma unroll
                        for (int u = 0; u < kCB; ++u)
                            if (k0 + u < K) t[u] += __ldcg(pc + (size_t)u * kThreads);
                    }
#pragma unroll
                    for (int u = 0; u < kCB; ++u) {
                        const int k = k0 + u;
                        if (k < K) out[(size_t)k * plane] = (k < klo || k > khi) ? one : (want_tau ? t[u] : t_of_tau(t[u]));
                    }
                }
                if (tid == 0) tile_arrive[tslot] = 0u;
            }
        }
        cta_sync();
    }
}

// Shell-band variant (K > kBandRows; DESIGN.md §6 a6): the table holds `rows` shells
// [kb0, kb0 + rows); each band is one pass over the unit's records that meet it.
// A pre-pass reads the records' shell bounds (PairRec::shells) and gives each band
// its index range [jb, je) of the depth-sorted list; within it the transform keeps
// (compacts) only the records whose bounds meet the band.  Same arithmetic per
// pair as k_accumulate; a write lands in the pass of the band holding its shell.
template <bool kStats, bool kTMA>
__global__ void __launch_bounds__(kThreads, kAccMinBlocks) k_accumulate_band(
    const WorkUnit* __restrict__ units, const uint32_t* __restrict__ n_units_dev,
    const uint32_t* __restrict__ vals, const PairRec* __restrict__ recs, int64_t n, AccLights al,
    int res, int K, int rows, uint32_t flags, float* __restrict__ scratch, uint32_t* tile_arrive,
    uint32_t* unit_counter, float* __restrict__ atlas, unsigned long long* __restrict__ stats,
    const uint64_t* __restrict__ slab_mask, const int2* __restrict__ slab_k) {
    pdl_begin();
    extern __shared__ __align__(128) unsigned char acc_smem[];
    constexpr size_t kRawBytes = kTMA ? kRawBytesTMA : 0;
    PairRec* s_raw = reinterpret_cast<PairRec*>(acc_smem);                                   // [kStage] (TMA)
    float4* s_cr = reinterpret_cast<float4*>(acc_smem + kRawBytes);                          // [kStage][5]
    float* s_acc = reinterpret_cast<float*>(acc_smem + kRawBytes + kStage * kCompact * sizeof(float4));  // [rows][64]
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_unit, s_last;
    __shared__ uint32_t s_nb;  // records kept by the band filter in the current stage
    __shared__ uint32_t s_jb[kMaxBands], s_je[kMaxBands];  // per band: records [jb, je) of the unit

    const int tid = threadIdx.x;
    if (kTMA && tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t phase = 0u;
    cta_sync();
    const uint32_t n_units = *n_units_dev;
    const int TW = res / kTile;
    const int n_tiles = TW * TW;
    const int W = res, H = res;
    const int n_bands = (K + rows - 1) / rows;
    for (int k = 0; k < rows + 2; ++k) s_acc[k * kThreads + tid] = 0.0f;  // (each epilogue re-zeroes what it reads)

    for (;;) {
        if (tid == 0) s_unit = atomicAdd(unit_counter, 1u);
        cta_sync();
        const uint32_t u = s_unit;
        if (u >= n_units) break;
        const WorkUnit wu = units[u];
        const int l = (int)(wu.tile / (uint32_t)n_tiles);
        const int tile = (int)(wu.tile - (uint32_t)l * n_tiles);
        const int row0 = (tile / TW) * kTile, col0 = (tile % TW) * kTile;
        const int tt = (int)wu.part * kThreads + tid;  // texel index within the tile
        const int row = row0 + (tt >> 3);
        const int col = col0 + (tt & 7);
        const uint32_t tslot = wu.tile * kTileSplit + wu.part;  // (tile, part) arrival counter

        // texel direction relative to the tile reference direction d_c (fp64 -> fp32)
        double c0, c1, c2, t0, t1, t2;
        texel_dir(row0 + 4, col0 + 4, W, H, c0, c1, c2);
        texel_dir(row, col, W, H, t0, t1, t2);
        const float etx = (float)(t0 - c0), ety = (float)(t1 - c1), etz = (float)(t2 - c2);
        const f2_t ETX = f2pack(etx, etx), ETY = f2pack(ety, ety), ETZ = f2pack(etz, etz);
        uint32_t st_live = 0, st_win = 0, st_step = 0, st_wany = 0, st_wmax = 0;

        const float dt = al.dt[l], dtlo = al.dtlo[l], idt = al.idt[l];
        const uint32_t n_rec = wu.jend - wu.jbeg;
        const PairRec* lrecs = recs + (int64_t)l * n;

        // band ranges: [s_jb[b], s_je[b]) = the records whose shell bounds meet band b
        if (tid < n_bands) { s_jb[tid] = 0xffffffffu; s_je[tid] = 0u; }
        cta_sync();
        {
            uint32_t fb[kMaxBands], eb[kMaxBands];
#pragma unroll
            for (int q = 0; q < kMaxBands; ++q) { fb[q] = 0xffffffffu; eb[q] = 0u; }
            constexpr int kPre = 8;  // loads in flight per thread
            for (uint32_t j0 = 0; j0 < n_rec; j0 += kPre * kThreads) {
                uint32_t gi[kPre], w[kPre];
#pragma unroll
                for (int u = 0; u < kPre; ++u) {
                    const uint32_t j = j0 + (uint32_t)(u * kThreads + tid);
                    gi[u] = j < n_rec ? __ldg(vals + wu.jbeg + j) : 0xffffffffu;
                }
#pragma unroll
                for (int u = 0; u < kPre; ++u)
                    w[u] = gi[u] != 0xffffffffu
                               ? __ldg(reinterpret_cast<const uint32_t*>(lrecs + gi[u]) + offsetof(PairRec, shells) / 4)
                               : 0xffffu;  // lo = 0xffff > any band: meets none
#pragma unroll
                for (int u = 0; u < kPre; ++u) {
                    const uint32_t j = j0 + (uint32_t)(u * kThreads + tid);
                    const int lo = (int)(w[u] & 0xffffu), hi = (int)(w[u] >> 16);
#pragma unroll
                    for (int q = 0; q < kMaxBands; ++q)
                        if (hi >= q * rows && lo < (q + 1) * rows) { fb[q] = min(fb[q], j); eb[q] = max(eb[q], j + 1u); }
                }
            }
#pragma unroll
            for (int q = 0; q < kMaxBands; ++q) {
                if (q >= n_bands) break;
                const uint32_t f = __reduce_min_sync(0xffffffffu, fb[q]), e = __reduce_max_sync(0xffffffffu, eb[q]);
                if ((tid & 31) == 0 && e != 0u) {
                    atomicMin(&s_jb[q], f);
                    atomicMax(&s_je[q], e);
                }
            }
        }
        cta_sync();
        // The table is all zero here (zeroed at kernel start, then by each band's
        // epilogue as it reads it); the epilogue of band b leaves the prefix tau
        // of its last shell in row 0 for band b + 1 (the carry).
        for (int band = 0; band < n_bands; ++band) {
            const int kb0 = band * rows;
            const int nrows = min(rows, K - kb0);
            const uint32_t jb = s_jb[band], nr = s_je[band] > jb ? s_je[band] - jb : 0u;
            // table row r = shell kb0 - 1 + r (r = 0 and nrows + 1: dump rows): shell k at acc_base + k * 256
            // (through an opaque move: ptxas otherwise rematerialises it from S2R TID in the pair loop)
            uint32_t acc_base;
            asm volatile("mov.b32 %0, %1;" : "=r"(acc_base)
                         : "r"(smem_addr(s_acc) + 4u * (uint32_t)tid - (uint32_t)(kb0 - 1) * (kThreads * 4)));
            const int wlo = kMagicBits + max(kb0 - 1, 0), whi = kMagicBits + kb0 + nrows;  // window clamp (bits)
            const uint32_t jbeg = wu.jbeg + jb, jend = jbeg + nr;
            const uint32_t n_batches = (nr + kStage - 1) / kStage;

            auto issue = [&](uint32_t b) {  // TMA: bulk copies of the stage's records into s_raw
                const uint32_t j0 = jbeg + b * kStage;
                const uint32_t nb = min((uint32_t)kStage, jend - j0);
                if (tid == 0) mbar_arrive_expect_tx(&s_bar, nb * (uint32_t)sizeof(PairRec));
                if ((uint32_t)tid < nb) {
                    const uint32_t gi = vals[j0 + tid];
                    bulk_g2s(s_raw + tid, lrecs + gi, (uint32_t)sizeof(PairRec), &s_bar);
                }
            };
            // register staging: thread t < 32 holds record t of the next stage (6 x 16-B
            // loads issued before the current stage's compute)
            uint4 ru[6];  // PairRec as six 16-B words (no union: the loads land in place)
            auto fetch = [&](uint32_t b) {
                const uint32_t j0 = jbeg + b * kStage;
                if ((uint32_t)tid < min((uint32_t)kStage, jend - j0)) {
                    const uint4* src = reinterpret_cast<const uint4*>(lrecs + vals[j0 + tid]);
#pragma unroll
                    for (int k = 0; k < 6; ++k) ru[k] = __ldg(src + k);
                }
            };
            if (n_batches > 0) {
                if (kTMA) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(0);
                } else {
                    fetch(0);
                }
            }

            for (uint32_t b = 0; b < n_batches; ++b) {
                if (kTMA) {
                    mbar_wait(&s_bar, phase);
                    phase ^= 1u;
                }
                uint32_t nb = min((uint32_t)kStage, nr - b * kStage);
                uint32_t slot = (uint32_t)tid;  // compact slot of this thread's record
                bool keep = (uint32_t)tid < nb;
                if (tid < 32) {  // band filter + compaction (the stage's records are in warp 0)
                    if (keep) {
                        const uint32_t w = kTMA ? s_raw[tid].shells : ru[5].w;
                        keep = (int)(w >> 16) >= kb0 && (int)(w & 0xffffu) < kb0 + nrows;
                    }
                    const uint32_t m = __ballot_sync(0xffffffffu, keep);
                    slot = __popc(m & ((1u << tid) - 1u));
                    if (tid == 0) s_nb = __popc(m);
                }
                if (keep) {  // transform: raw record -> compact, relative to d_c
                    float* q = reinterpret_cast<float*>(s_cr) + (slot >> 1) * (2 * kPairFields) + (slot & 1);
                    float v[kPairFields];
                    if (kTMA) {
                        const PairRec& R = s_raw[tid];
                        const float vv[kPairFields] = {(float)(R.di[0] - c0), (float)(R.di[1] - c1), (float)(R.di[2] - c2),
                                                       R.rcut_D2, R.g[0], R.g[1], R.g[2], R.D,
                                                       R.W[0], R.W[1], R.W[2], R.W[3], R.W[4], R.W[5], R.W[6], R.W[7],
                                                       R.W[8], R.eD, R.betap, (float)R.kD};
#pragma unroll
                        for (int f = 0; f < kPairFields; ++f) v[f] = vv[f];
                    } else {  // field offsets of PairRec (static_assert'ed 96 B layout)
                        const float vv[kPairFields] = {
                            (float)(__hiloint2double((int)ru[0].y, (int)ru[0].x) - c0),
                            (float)(__hiloint2double((int)ru[0].w, (int)ru[0].z) - c1),
                            (float)(__hiloint2double((int)ru[1].y, (int)ru[1].x) - c2),
                            __uint_as_float(ru[5].z),                                                   // rcut_D2
                            __uint_as_float(ru[1].z), __uint_as_float(ru[1].w), __uint_as_float(ru[2].x),  // g
                            __uint_as_float(ru[4].z),                                                   // D
                            __uint_as_float(ru[2].y), __uint_as_float(ru[2].z), __uint_as_float(ru[2].w),  // W
                            __uint_as_float(ru[3].x), __uint_as_float(ru[3].y), __uint_as_float(ru[3].z),
                            __uint_as_float(ru[3].w), __uint_as_float(ru[4].x), __uint_as_float(ru[4].y),
                            __uint_as_float(ru[4].w),                                                   // eD
                            __uint_as_float(ru[5].y),                                                   // betap
                            (float)(int)ru[5].x};                                                       // kD
#pragma unroll
                        for (int f = 0; f < kPairFields; ++f) v[f] = vv[f];
                    }
                    {  // fields 0-2: -W f, f = d_i - d_c (the pair test forms W delta = W e_t - W f); 7: -D
                        const float f0 = v[0], f1 = v[1], f2 = v[2];
                        v[0] = -fmaf(v[8], f0, fmaf(v[9], f1, v[10] * f2));
                        v[1] = -fmaf(v[11], f0, fmaf(v[12], f1, v[13] * f2));
                        v[2] = -fmaf(v[14], f0, fmaf(v[15], f1, v[16] * f2));
                        v[7] = -v[7];
                    }
#pragma unroll
                    for (int f = 0; f < kPairFields; ++f) q[2 * f] = v[f];
                }
                cta_sync();  // compact copy ready; raw buffer free
                nb = s_nb;
                if (kStats && tid == 0) atomicAdd(&stats[7], (unsigned long long)nb);
                if (b + 1 < n_batches) {
                    if (kTMA) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue(b + 1);
                    } else {
                        fetch(b + 1);
                    }
                }
                // two records per iteration: independent dependency chains for the pair test
                uint32_t my_live = 0;
                auto process = [&](PairTest2& T2) {
                    if (kStats) {
                        const uint32_t ba = __ballot_sync(0xffffffffu, T2.liveA), bb = __ballot_sync(0xffffffffu, T2.liveB);
                        my_live += (uint32_t)T2.liveA + (uint32_t)T2.liveB;
                        st_wany += (ba != 0u) + (bb != 0u);
                    }
                    const bool anyA = __any_sync(0xffffffffu, T2.liveA), anyB = __any_sync(0xffffffffu, T2.liveB);
                    if (anyA && anyB) {
                        pair_live_warp2<kStats, true>(T2, acc_base, K, dt, dtlo, idt, kb0, nrows, wlo, whi, st_live, st_win,
                                                       st_step);
                        return;
                    }
                    if (anyA)
                        pair_live_warp<kStats, true>(f2lo(T2.A), f2lo(T2.C2), f2lo(T2.DOT), T2.liveA, f2lo(T2.ND),
                                                      f2lo(T2.ED), f2lo(T2.BP), f2lo(T2.KD), acc_base, K, dt, dtlo, idt,
                                                      kb0, nrows, wlo, whi, st_live, st_win, st_step);
                    if (anyB)
                        pair_live_warp<kStats, true>(f2hi(T2.A), f2hi(T2.C2), f2hi(T2.DOT), T2.liveB, f2hi(T2.ND),
                                                      f2hi(T2.ED), f2hi(T2.BP), f2hi(T2.KD), acc_base, K, dt, dtlo, idt,
                                                      kb0, nrows, wlo, whi, st_live, st_win, st_step);
                };
                uint32_t pr_addr = smem_addr(s_cr);  // induction variable: record pair (r, r+1)
                uint32_t r = 0;
                // two record pairs' tests per iteration (twice the independent chains:
                // 0.95 -> 0.93 ms at 80 registers; four pairs need 128 and are slower)
                for (; r + 2 < nb; r += 4, pr_addr += 2 * kPairBytes) {
                    PairTest2 Ta = pair_test2(pr_addr, ETX, ETY, ETZ);
                    PairTest2 Tb = pair_test2(pr_addr + kPairBytes, ETX, ETY, ETZ);
                    Tb.liveB = Tb.liveB && (r + 3 < nb);
                    process(Ta);
                    process(Tb);
                }
                for (; r < nb; r += 2, pr_addr += kPairBytes) {
                    PairTest2 T2 = pair_test2(pr_addr, ETX, ETY, ETZ);
                    T2.liveB = T2.liveB && (r + 1 < nb);
                    process(T2);
                }
                if (kStats) st_wmax += __reduce_max_sync(0xffffffffu, my_live);
                cta_sync();  // compact copy consumed
            }

            // prefix sum over the band's shells -> tau_k; epilogue T = exp(-tau) (Eq.4)
            // (multi-chunk tiles: the partial tau_k to scratch, combined below);
            // each row is zeroed as it is read
            float tau = 0.0f;
            if (wu.nchunks == 1) {
                // NEXT-1 slab: outside P x [k_min, k_max] the table stays T = 1
                int sklo = 0, skhi = K - 1;
                if (slab_mask) {
                    const int2 kr = slab_k[l];
                    sklo = kr.x;
                    skhi = ((slab_mask[wu.tile] >> tt) & 1ull) ? kr.y : -1;
                }
                const bool want_tau = (flags & DGSM_OUTPUT_TAU) != 0;
                const float one = want_tau ? 0.0f : 1.0f;
                const size_t plane = (size_t)H * W;
                float* o = atlas + ((size_t)l * K + kb0) * plane + (size_t)row * W + col;
                if (!slab_mask && !want_tau) {  // the common case: no per-shell selects
#pragma unroll 4
                    for (int k = 0; k < nrows; ++k, o += plane) {
                        tau += s_acc[(k + 1) * kThreads + tid];
                        s_acc[(k + 1) * kThreads + tid] = 0.0f;
                        *o = t_of_tau(tau);
                    }
                } else {
                    for (int k = 0; k < nrows; ++k, o += plane) {
                        tau += s_acc[(k + 1) * kThreads + tid];
                        s_acc[(k + 1) * kThreads + tid] = 0.0f;
                        const int ks = kb0 + k;
                        *o = (ks < sklo || ks > skhi) ? one : (want_tau ? tau : t_of_tau(tau));
                    }
                }
            } else {
                float* part = scratch + ((size_t)(wu.slot + wu.chunk) * K + kb0) * kThreads + tid;
                for (int k = 0; k < nrows; ++k) {
                    tau += s_acc[(k + 1) * kThreads + tid];
                    s_acc[(k + 1) * kThreads + tid] = 0.0f;
                    part[(size_t)k * kThreads] = tau;
                }
            }
            s_acc[tid] = 0.0f;                              // the dump rows
            s_acc[(nrows + 1) * kThreads + tid] = 0.0f;
            if (band + 1 < n_bands) s_acc[kThreads + tid] = tau;  // carry into the next band's first row
        }

        if (kStats) {
            atomicAdd(&stats[1], (unsigned long long)st_live);
            atomicAdd(&stats[2], (unsigned long long)st_win);
            atomicAdd(&stats[3], (unsigned long long)st_step);
            if (tid == 0) atomicAdd(&stats[0], (unsigned long long)n_rec * kThreads);
            // warp-level: records entering the live path (any lane live) and the
            // per-stage max over lanes of live records (what a per-lane loop would cost)
            // (banded: a record met by two bands is counted in both)
            if ((tid & 31) == 0) {
                atomicAdd(&stats[4], (unsigned long long)n_rec);
                atomicAdd(&stats[5], (unsigned long long)st_wany);
                atomicAdd(&stats[6], (unsigned long long)st_wmax);
            }
        }
        if (wu.nchunks > 1) {
            __threadfence();
            cta_sync();
            // (tiles of more than kInlineCombine chunks: k_combine_deferred sums them)
            if (tid == 0) s_last = wu.nchunks <= kInlineCombine &&
                                   atomicAdd(&tile_arrive[tslot], 1u) == wu.nchunks - 1 ? 1u : 0u;
            cta_sync();
            if (s_last) {
                __threadfence();
                int sklo = 0, skhi = K - 1;
                if (slab_mask) {
                    const int2 kr = slab_k[l];
                    sklo = kr.x;
                    skhi = ((slab_mask[wu.tile] >> tt) & 1ull) ? kr.y : -1;
                }
                const bool want_tau = (flags & DGSM_OUTPUT_TAU) != 0;
                const float one = want_tau ? 0.0f : 1.0f;
                const size_t plane = (size_t)H * W;
                float* out = atlas + ((size_t)l * K) * plane + (size_t)row * W + col;
                const float* base = scratch + ((size_t)wu.slot * K) * kThreads + tid;
                // kCB shells at a time: kCB independent L2 loads per chunk in flight
                // (the summation order per shell stays chunk 0, 1, ...: deterministic)
                constexpr int kCB = 4;  // 2: slower; 6, 16: more registers for the whole kernel
                for (int k0 = 0; k0 < K; k0 += kCB) {
                    float t[kCB];
#pragma unroll
                    for (int u = 0; u < kCB; ++u) t[u] = 0.0f;
                    for (uint32_t c = 0; c < wu.nchunks; ++c) {
                        const float* pc = base + ((size_t)c * K + k0) * kThreads;
#pragma unroll
                        for (int u = 0; u < kCB; ++u)
                            if (k0 + u < K) t[u] += __ldcg(pc + (size_t)u * kThreads);
                    }
#pragma unroll
                    for (int u = 0; u < kCB; ++u) {
                        const int k = k0 + u;
                        if (k < K) out[(size_t)k * plane] = (k < sklo || k > skhi) ? one : (want_tau ? t[u] : t_of_tau(t[u]));
                    }
                }
                if (tid == 0) tile_arrive[tslot] = 0u;
            }
        }
        cta_sync();
    }
}

// Tiles with more than kInlineCombine chunks (a few dense tiles, e.g. an avatar
// close to the light): their partial tau are summed here, by (tile, 4 shells)
// items over the whole GPU instead of by the one CTA that finished last (which
// made that CTA the kernel's tail).  Thread = (shell, texel); chunk order kept.
__global__ void __launch_bounds__(256) k_combine_deferred(const WorkUnit* __restrict__ units,
                                                          const uint32_t* __restrict__ deferred,
                                                          const uint32_t* deferred_count, const float* __restrict__ scratch,
                                                          int res, int K, uint32_t flags, float* __restrict__ atlas,
                                                          const uint64_t* __restrict__ slab_mask,
                                                          const int2* __restrict__ slab_k) {
    pdl_begin();
    const uint32_t nd = *deferred_count;
    const int groups = (K + 3) / 4;
    const int TW = res / kTile, n_tiles = TW * TW;
    const size_t plane = (size_t)res * res;
    const bool want_tau = (flags & DGSM_OUTPUT_TAU) != 0;
    const float one = want_tau ? 0.0f : 1.0f;
    for (uint32_t item = blockIdx.x; item < nd * (uint32_t)groups; item += gridDim.x) {
        const WorkUnit wu = units[deferred[item / groups]];
        const int k = (int)(item % groups) * 4 + (int)(threadIdx.x >> 6), tt = (int)(threadIdx.x & 63);
        if (k >= K) continue;
        const int l = (int)(wu.tile / (uint32_t)n_tiles), tile = (int)(wu.tile - (uint32_t)l * n_tiles);
        const int row = (tile / TW) * kTile + (tt >> 3), col = (tile % TW) * kTile + (tt & 7);
        const float* p = scratch + ((size_t)wu.slot * K + k) * kThreads + tt;
        const size_t cs = (size_t)K * kThreads;  // one chunk's partials
        float t = 0.0f;
        uint32_t c = 0;
        for (; c + 8 <= wu.nchunks; c += 8) {  // 8 loads in flight, added in chunk order
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (size_t)(c + u) * cs);
#pragma unroll
            for (int u = 0; u < 8; ++u) t += v[u];
        }
        for (; c < wu.nchunks; ++c) t += __ldcg(p + (size_t)c * cs);
        int klo = 0, khi = K - 1;
        if (slab_mask) {
            const int2 kr = slab_k[l];
            klo = kr.x;
            khi = ((slab_mask[wu.tile] >> tt) & 1ull) ? kr.y : -1;
        }
        atlas[((size_t)l * K + k) * plane + (size_t)row * res + col] =
            (k < klo || k > khi) ? one : (want_tau ? t : t_of_tau(t));
    }
}

__global__ void k_exp(const float* tau, float* T, int64_t count) {
    pdl_begin();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        T[i] = t_of_tau(tau[i]);
}
}  // namespace

thread_local bool last_staging_tma = false;
bool accumulate_last_used_tma() { return last_staging_tma; }

// Table rows of the accumulation for K shells: K up to kTableRows, else kBandRows
// (bands); DGSM_BAND_ROWS overrides kBandRows (A/B), clamped to [32, 256].
int accumulate_rows(int K) {
    static const int band_rows = [] {
        int r = kBandRows;
        if (const char* e = getenv("DGSM_BAND_ROWS")) r = atoi(e);
        return std::min(std::max(r, kMinBandRows), DGSM_MAX_SHELLS);
    }();
    return K <= kTableRows ? K : std::min(K, band_rows);
}

size_t accumulate_smem_bytes(int K, bool tma) {
    const int rows = accumulate_rows(K);
    if (rows == K)  // single-table kernel
        return (tma ? kRawBytesTMA_A : 0) + kStageA * kCompact * sizeof(float4) + (size_t)K * kThreads * sizeof(float);
    return (tma ? kRawBytesTMA : 0) + kStage * kCompact * sizeof(float4) +
           (size_t)(rows < K ? rows + 2 : rows) * kThreads * sizeof(float);  // (+2 dump rows with bands)
}

void launch_accumulate(const WorkUnit* units, const uint32_t* n_units_dev, uint32_t max_units,
                       const uint32_t* vals, const PairRec* recs, int64_t n, const LightsParam& lp,
                       int n_lights, int res, int K, uint32_t flags, float* scratch,
                       uint32_t* tile_arrive, uint32_t* unit_counter, float* atlas,
                       unsigned long long* stats, const uint64_t* slab_mask, const int2* slab_k,
                       const uint32_t* deferred, const uint32_t* deferred_count, cudaEvent_t ev_before,
                       cudaEvent_t ev_after, cudaStream_t s) {
    AccLights al;
    for (int l = 0; l < DGSM_MAX_LIGHTS; ++l) {
        const double dt = l < n_lights ? (double)lp.l[l].w / K : 1.0;
        al.dt[l] = (float)dt;
        al.dtlo[l] = (float)(dt - (double)al.dt[l]);
        al.idt[l] = (float)(1.0 / dt);
    }
    const int rows = accumulate_rows(K);
    const bool band = rows < K;
    // The dynamic shared-memory limit is a process-wide attribute of the kernel
    // (per device): set it once to the largest size any K needs, so a launch on
    // one thread never runs under a smaller limit set by another; the occupancy
    // figures (which depend on K) are cached per thread.
    static std::atomic<uint64_t> attr_set_mask{0};  // bit = device ordinal
    thread_local int dev_cached = -1, n_sm = 0;
    thread_local int cached_K = -1, per_sm_tma = 0, per_sm_reg = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem_tma = accumulate_smem_bytes(K, true), smem_reg = accumulate_smem_bytes(K, false);
    if (dev < 64 && !(attr_set_mask.load() & (1ull << dev))) {
        // (the largest table of either kernel: DGSM_MAX_SHELLS rows + 2 dump rows)
        const int smax = (int)(kRawBytesTMA + kStage * kCompact * sizeof(float4) +
                               (size_t)(DGSM_MAX_SHELLS + 2) * kThreads * sizeof(float));
#define DGSM_ACC_ATTR(F) cudaFuncSetAttribute(F, cudaFuncAttributeMaxDynamicSharedMemorySize, smax)
        DGSM_ACC_ATTR((k_accumulate<false, true>)); DGSM_ACC_ATTR((k_accumulate<true, true>));
        DGSM_ACC_ATTR((k_accumulate<false, false>)); DGSM_ACC_ATTR((k_accumulate<true, false>));
        DGSM_ACC_ATTR((k_accumulate_band<false, true>)); DGSM_ACC_ATTR((k_accumulate_band<true, true>));
        DGSM_ACC_ATTR((k_accumulate_band<false, false>)); DGSM_ACC_ATTR((k_accumulate_band<true, false>));
#undef DGSM_ACC_ATTR
        attr_set_mask.fetch_or(1ull << dev);
    }
    if (dev != dev_cached || K != cached_K) {
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        if (band) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_tma, k_accumulate_band<false, true>, kThreads, smem_tma);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_reg, k_accumulate_band<false, false>, kThreads, smem_reg);
        } else {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_tma, k_accumulate<false, true>, kThreads, smem_tma);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_reg, k_accumulate<false, false>, kThreads, smem_reg);
        }
        dev_cached = dev;
        cached_K = K;
    }
    // TMA staging unless its raw buffer costs a CTA per SM (K = 64 on sm_100: 10 vs 12 CTAs;
    // register staging measured 0.917 vs 0.998 ms on cfg2; ncu: profiles/r02_k_accumulate_cfg2_tma.md)
    bool tma = per_sm_tma >= per_sm_reg;
    if (const char* f = getenv("DGSM_ACC_STAGING")) {  // tests: force "tma" or "reg"
        if (!strcmp(f, "tma")) tma = true;
        else if (!strcmp(f, "reg")) tma = false;
    }
    const int per_sm = std::max(1, tma ? per_sm_tma : per_sm_reg);
    const size_t smem = tma ? smem_tma : smem_reg;
    uint32_t grid = (uint32_t)per_sm * (uint32_t)n_sm;
    if (grid > max_units) grid = max_units;
    if (grid == 0) grid = 1;
    if (ev_before) cudaEventRecord(ev_before, s);
    const bool st = (flags & DGSM_COLLECT_STATS) != 0;
#define DGSM_ACC_ARGS units, n_units_dev, vals, recs, n, al, res, K, flags, scratch, tile_arrive, unit_counter, \
                      atlas, stats, slab_mask, slab_k
#define DGSM_ACC_BAND_ARGS units, n_units_dev, vals, recs, n, al, res, K, rows, flags, scratch, tile_arrive, \
                           unit_counter, atlas, stats, slab_mask, slab_k
    if (band) {
        if (st && tma) pdl_launch(k_accumulate_band<true, true>, grid, kThreads, smem, s, DGSM_ACC_BAND_ARGS);
        else if (st) pdl_launch(k_accumulate_band<true, false>, grid, kThreads, smem, s, DGSM_ACC_BAND_ARGS);
        else if (tma) pdl_launch(k_accumulate_band<false, true>, grid, kThreads, smem, s, DGSM_ACC_BAND_ARGS);
        else pdl_launch(k_accumulate_band<false, false>, grid, kThreads, smem, s, DGSM_ACC_BAND_ARGS);
    } else {
        if (st && tma) pdl_launch(k_accumulate<true, true>, grid, kThreads, smem, s, DGSM_ACC_ARGS);
        else if (st) pdl_launch(k_accumulate<true, false>, grid, kThreads, smem, s, DGSM_ACC_ARGS);
        else if (tma) pdl_launch(k_accumulate<false, true>, grid, kThreads, smem, s, DGSM_ACC_ARGS);
        else pdl_launch(k_accumulate<false, false>, grid, kThreads, smem, s, DGSM_ACC_ARGS);
    }
#undef DGSM_ACC_BAND_ARGS
#undef DGSM_ACC_ARGS
    pdl_launch(k_combine_deferred, (unsigned)n_sm * 8, 256, 0, s, units, deferred, deferred_count, scratch, res, K, flags, atlas,
                                                         slab_mask, slab_k);
    last_staging_tma = tma;
    if (ev_after) cudaEventRecord(ev_after, s);
}

void launch_exp(const float* tau, float* T, int64_t count, cudaStream_t s) {
    if (count <= 0) return;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    pdl_launch(k_exp, (unsigned)blocks, 256, 0, s, tau, T, count);
}

}  // namespace dgsm
