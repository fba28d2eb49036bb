// accumulate.cu — a6: per-tile accumulation of the closed-form optical depth
// (Eq.2-4) over the bucketed occluders of each 8x8 tile
// (P:L173), then T = exp(-tau) (Eq.4) into the atlas [L][K][H][W].
//
// Design (DESIGN.md §"a6"):
//  * one CTA = 64 threads = one 8x8 tile; thread <-> texel; each thread owns
//    one column acc[k][texel] of a K x 64 shared-memory table (conflict-free:
//    the bank is the texel index);
//  * the tile's depth-sorted Gaussian list is cut into chunks (work units);
//    a persistent grid pulls units from an atomic counter; multi-chunk tiles
//    combine their partial tau deterministically (chunk order) in the CTA that
//    finishes last;
//  * the 96-B footprint records of the listed Gaussians are gathered into
//    shared memory with TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx),
//    64 records per stage, double-buffered;
//  * per (texel, Gaussian) pair the delta-formulation (R9) gives a, r = c - b^2/a
//    and s* - D without cancellation; fp32 erf saturates to +-1 exactly for
//    |x| >= 3.92, so a pair contributes pref*(erf(x_k) - erf(x_0)) only on the
//    few shells of its "window" and the constant pref*(1 - erf(x_0)) beyond it:
//    the window shells and the step are written as differences into acc and a
//    prefix sum over k at the end restores tau_k.  No tensor cores: this is not
//    a dense contraction (FP32 FMA + MUFU bound).
#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
constexpr int kThreads = 64;      // one 8x8 tile
constexpr int kStage = 64;        // records per pipeline stage
constexpr float kXS = 3.92f;      // |x| >= kXS  ->  erf_fast(x) == +-1 exactly
constexpr float kRCut = 180.0f;   // r > kRCut -> ex2.approx.ftz(-r/(2 ln 2)) == 0 exactly

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// fp32 erf with max abs error ~1.3e-7 on [0, 3.92) and exactly +-1 beyond.
// |x| < 0.75: x * P(x^2); 0.75 <= |x| < 3.92: 1 - 2^Q(|x|).  Coefficients from
// tools/fit_erf.py (weighted least squares toward minimax, fp32 Horner).
__device__ __forceinline__ float erf_fast(float x) {
    const float t = fabsf(x);
    if (t >= kXS) return copysignf(1.0f, x);
    if (t < 0.75f) {
        const float z = x * x;
        float p = -6.768997409e-04f;
        p = fmaf(p, z, 5.116294138e-03f);
        p = fmaf(p, z, -2.683510073e-02f);
        p = fmaf(p, z, 1.128337309e-01f);
        p = fmaf(p, z, -3.761261702e-01f);
        p = fmaf(p, z, 1.128379107e+00f);
        return x * p;
    }
    float q = -2.865754504e-05f;
    q = fmaf(q, t, 6.052364479e-04f);
    q = fmaf(q, t, -5.908878520e-03f);
    q = fmaf(q, t, 3.594445437e-02f);
    q = fmaf(q, t, -1.557482034e-01f);
    q = fmaf(q, t, -9.141569138e-01f);
    q = fmaf(q, t, -1.629331112e+00f);
    q = fmaf(q, t, 2.074461663e-04f);
    return copysignf(1.0f - ex2_approx(q), x);
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

struct AccLights {
    float dt[DGSM_MAX_LIGHTS];     // t_max / K (fp32)
    float dtlo[DGSM_MAX_LIGHTS];   // t_max / K - dt (fp64 remainder)
    float idt[DGSM_MAX_LIGHTS];    // 1 / dt
};

// kStats: count the work (live pairs, window shells, steps) for the benchmark's
// roofline accounting; the timed path is <false>.
template <bool kStats>
__global__ void __launch_bounds__(kThreads) k_accumulate(
    const WorkUnit* __restrict__ units, const uint32_t* __restrict__ n_units_dev,
    const uint32_t* __restrict__ vals, const PairRec* __restrict__ recs, int64_t n, AccLights al,
    int res, int K, uint32_t flags, float* __restrict__ scratch, uint32_t* tile_arrive,
    uint32_t* unit_counter, float* __restrict__ atlas, unsigned long long* __restrict__ stats) {
    extern __shared__ __align__(128) unsigned char acc_smem[];
    PairRec* s_rec = reinterpret_cast<PairRec*>(acc_smem);                       // [2][kStage]
    float* s_acc = reinterpret_cast<float*>(acc_smem + 2 * kStage * sizeof(PairRec));  // [K][64]
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_unit, s_last;

    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase[2] = {0u, 0u};
    const uint32_t n_units = *n_units_dev;
    const int TW = res / kTile;
    const int n_tiles = TW * TW;
    const int W = res, H = res;

    for (;;) {
        if (tid == 0) s_unit = atomicAdd(unit_counter, 1u);
        __syncthreads();
        const uint32_t u = s_unit;
        if (u >= n_units) break;
        const WorkUnit wu = units[u];
        const int l = (int)(wu.tile / (uint32_t)n_tiles);
        const int tile = (int)(wu.tile - (uint32_t)l * n_tiles);
        const int row = (tile / TW) * kTile + (tid >> 3);
        const int col = (tile % TW) * kTile + (tid & 7);

        // texel-centre direction d(u_c, v_c) in fp64 (R3)
        double d0, d1, d2;
        {
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
        for (int k = 0; k < K; ++k) s_acc[k * kThreads + tid] = 0.0f;
        uint32_t st_live = 0, st_win = 0, st_step = 0;

        const float dt = al.dt[l], dtlo = al.dtlo[l], idt = al.idt[l];
        const uint32_t n_rec = wu.jend - wu.jbeg;
        const uint32_t n_batches = (n_rec + kStage - 1) / kStage;
        const PairRec* lrecs = recs + (int64_t)l * n;

        auto issue = [&](uint32_t b) {
            const uint32_t j0 = wu.jbeg + b * kStage;
            const uint32_t nb = min((uint32_t)kStage, wu.jend - j0);
            PairRec* dst = s_rec + (b & 1) * kStage;
            if (tid == 0) mbar_arrive_expect_tx(&s_bar[b & 1], nb * (uint32_t)sizeof(PairRec));
            if ((uint32_t)tid < nb) {
                const uint32_t gi = vals[j0 + tid];
                bulk_g2s(dst + tid, lrecs + gi, (uint32_t)sizeof(PairRec), &s_bar[b & 1]);
            }
        };
        if (n_batches > 0) issue(0);
        if (n_batches > 1) issue(1);

        for (uint32_t b = 0; b < n_batches; ++b) {
            const int buf = b & 1;
            mbar_wait(&s_bar[buf], phase[buf]);
            phase[buf] ^= 1u;
            const uint32_t nb = min((uint32_t)kStage, n_rec - b * kStage);
            const PairRec* sr = s_rec + buf * kStage;
            for (uint32_t r = 0; r < nb; ++r) {
                const PairRec& R = sr[r];
                // delta = d - d_i (fp64 difference, rounded to fp32)
                const float ex = (float)(d0 - R.di[0]);
                const float ey = (float)(d1 - R.di[1]);
                const float ez = (float)(d2 - R.di[2]);
                // W delta, u = W d = g + W delta, a = |u|^2 = d^T A d (Eq.2)
                const float wx = fmaf(R.W[0], ex, fmaf(R.W[1], ey, R.W[2] * ez));
                const float wy = fmaf(R.W[3], ex, fmaf(R.W[4], ey, R.W[5] * ez));
                const float wz = fmaf(R.W[6], ex, fmaf(R.W[7], ey, R.W[8] * ez));
                const float gx = R.g[0], gy = R.g[1], gz = R.g[2];
                const float ux = gx + wx, uy = gy + wy, uz = gz + wz;
                const float a = fmaf(ux, ux, fmaf(uy, uy, uz * uz));
                // r = c - b^2/a = D^2 |g x W delta|^2 / a  (Lagrange identity)
                const float cx = fmaf(gy, wz, -gz * wy);
                const float cy = fmaf(gz, wx, -gx * wz);
                const float cz = fmaf(gx, wy, -gy * wx);
                const float ia = __frcp_rn(a);
                const float D = R.D;
                const float rr = D * D * fmaf(cx, cx, fmaf(cy, cy, cz * cz)) * ia;
                if (!(rr <= kRCut)) continue;  // exp(-r/2) == 0 in fp32: no contribution
                // s* - D = -D (u . W delta)/a: closest approach relative to D
                const float sD = -D * fmaf(ux, wx, fmaf(uy, wy, uz * wz)) * ia;
                const float ra = rsqrtf(a);
                const float h = 0.70710678118654752f * a * ra;  // sqrt(a/2)
                const float x0 = -h * (D + sD);                    // sqrt(a/2) * (b/a) of Eq.3
                const float e0 = erf_fast(x0);
                if (e0 >= 1.0f) continue;  // whole Gaussian behind the light
                if (kStats) ++st_live;
                // Eq.3 prefactor beta sqrt(pi/(2a)) exp(-(c - b^2/a)/2)
                const float pref = R.betap * ra * ex2_approx(-0.72134752044448170f * rr);
                // t_k - s* = (k - kD) dt + e
                const float e = R.eD - sD;
                const float xsh = kXS / h;
                float flo = (-xsh - e) * idt, fhi = (xsh - e) * idt;
                flo = fminf(fmaxf(flo, -(float)(K + 2)), (float)(K + 2));
                fhi = fminf(fmaxf(fhi, -(float)(K + 2)), (float)(K + 2));
                int klo = R.kD + (int)floorf(flo) + 1;
                int khi = R.kD + (int)ceilf(fhi);
                klo = max(klo, 0);
                khi = min(max(khi, klo), K);
                if (kStats) { st_win += (uint32_t)(khi - klo); st_step += khi < K ? 1u : 0u; }
                float prev = 0.0f;
                for (int k = klo; k < khi; ++k) {
                    const float fk = (float)(k - R.kD);
                    const float tk = fmaf(fk, dt, fmaf(fk, dtlo, e));
                    const float w = pref * (erf_fast(h * tk) - e0);
                    s_acc[k * kThreads + tid] += w - prev;
                    prev = w;
                }
                if (khi < K) s_acc[khi * kThreads + tid] += fmaf(pref, 1.0f - e0, -prev);
            }
            __syncthreads();  // everyone is done with this buffer
            if (b + 2 < n_batches) issue(b + 2);
        }

        if (kStats) {
            atomicAdd(&stats[1], (unsigned long long)st_live);
            atomicAdd(&stats[2], (unsigned long long)st_win);
            atomicAdd(&stats[3], (unsigned long long)st_step);
            if (tid == 0) atomicAdd(&stats[0], (unsigned long long)n_rec * kThreads);
        }
        // prefix sum over shells -> tau_k; epilogue T = exp(-tau) (Eq.4)
        const bool want_tau = (flags & DGSM_OUTPUT_TAU) != 0;
        const size_t plane = (size_t)H * W;
        float* out = atlas + ((size_t)l * K) * plane + (size_t)row * W + col;
        if (wu.nchunks == 1) {
            float tau = 0.0f;
            for (int k = 0; k < K; ++k) {
                tau += s_acc[k * kThreads + tid];
                out[(size_t)k * plane] = want_tau ? tau : expf(-tau);
            }
        } else {
            float* part = scratch + ((size_t)(wu.slot + wu.chunk) * K) * kThreads + tid;
            float tau = 0.0f;
            for (int k = 0; k < K; ++k) {
                tau += s_acc[k * kThreads + tid];
                part[(size_t)k * kThreads] = tau;
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = (atomicAdd(&tile_arrive[wu.tile], 1u) == wu.nchunks - 1) ? 1u : 0u;
            __syncthreads();
            if (s_last) {
                __threadfence();
                const float* base = scratch + ((size_t)wu.slot * K) * kThreads + tid;
                for (int k = 0; k < K; ++k) {
                    float t = 0.0f;
                    for (uint32_t c = 0; c < wu.nchunks; ++c)
                        t += __ldcg(base + ((size_t)c * K + k) * kThreads);
                    out[(size_t)k * plane] = want_tau ? t : expf(-t);
                }
                if (tid == 0) tile_arrive[wu.tile] = 0u;
            }
        }
        __syncthreads();
    }
}

__global__ void k_exp(const float* tau, float* T, int64_t count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        T[i] = expf(-tau[i]);
}
}  // namespace

size_t accumulate_smem_bytes(int K) {
    return 2 * kStage * sizeof(PairRec) + (size_t)K * kThreads * sizeof(float);
}

void launch_accumulate(const WorkUnit* units, const uint32_t* n_units_dev, uint32_t max_units,
                       const uint32_t* vals, const PairRec* recs, int64_t n, const LightsParam& lp,
                       int n_lights, int res, int K, uint32_t flags, float* scratch,
                       uint32_t* tile_arrive, uint32_t* unit_counter, float* atlas,
                       unsigned long long* stats, cudaEvent_t ev_before, cudaEvent_t ev_after,
                       cudaStream_t s) {
    AccLights al;
    for (int l = 0; l < DGSM_MAX_LIGHTS; ++l) {
        const double dt = l < n_lights ? (double)lp.l[l].w / K : 1.0;
        al.dt[l] = (float)dt;
        al.dtlo[l] = (float)(dt - (double)al.dt[l]);
        al.idt[l] = (float)(1.0 / dt);
    }
    const size_t smem = accumulate_smem_bytes(K);
    static int dev_cached = -1, n_sm = 0;
    static size_t smem_set = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != dev_cached) {
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        dev_cached = dev;
        smem_set = 0;
    }
    if (smem > smem_set) {
        cudaFuncSetAttribute(k_accumulate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_accumulate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        smem_set = smem;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_accumulate<false>, kThreads, smem);
    if (per_sm < 1) per_sm = 1;
    uint32_t grid = (uint32_t)per_sm * (uint32_t)n_sm;
    if (grid > max_units) grid = max_units;
    if (grid == 0) grid = 1;
    if (ev_before) cudaEventRecord(ev_before, s);
    if (flags & DGSM_COLLECT_STATS)
        k_accumulate<true><<<grid, kThreads, smem, s>>>(units, n_units_dev, vals, recs, n, al, res, K, flags,
                                                        scratch, tile_arrive, unit_counter, atlas, stats);
    else
        k_accumulate<false><<<grid, kThreads, smem, s>>>(units, n_units_dev, vals, recs, n, al, res, K, flags,
                                                         scratch, tile_arrive, unit_counter, atlas, stats);
    if (ev_after) cudaEventRecord(ev_after, s);
}

void launch_exp(const float* tau, float* T, int64_t count, cudaStream_t s) {
    if (count <= 0) return;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_exp<<<(unsigned)blocks, 256, 0, s>>>(tau, T, count);
}

}  // namespace dgsm
