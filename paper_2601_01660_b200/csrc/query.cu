// query.cu — a8: DGSM sampling (§3.3).  Each receiver
// centre x fetches T[psi(d), t(x)] "via trilinear interpolation" per light:
// octahedral bilinear with mirror-wrapped taps across the atlas border (Q12) x
// radial linear with t clamped to [t_0, t_{K-1}]; T = 1 at the light (Q18);
// product over lights (Q13); optional colour *= T ("multiply the direct term").
// Index math in fp64 (at 2048^2 the fp32 texel coordinate has ulp 2.4e-4).
// HBM/L2 bound: 12 B position + 8 x 4 B taps per light + 4 B output per query.
#include <algorithm>
#include <cstring>

#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
__device__ __forceinline__ void wrap_tap(int& col, int& row, int W, int H) {
    if (col < 0) { col = -1 - col; row = H - 1 - row; }
    else if (col > W - 1) { col = 2 * W - 1 - col; row = H - 1 - row; }
    if (row < 0) { row = -1 - row; col = W - 1 - col; }
    else if (row > H - 1) { row = 2 * H - 1 - row; col = W - 1 - col; }
}

// Per-light constants of the sampler, fp64 (host-computed once per call).
struct QLight {
    double ox, oy, oz;  // o_L
    double kscale;      // K / t_max: fk = t K / t_max - 1/2
};
struct QueryLights {
    QLight l[DGSM_MAX_LIGHTS];
};

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

// Border taps (a footprint that crosses the atlas edge): each of the 8 taps
// mirror-wrapped on its own (Q12).  Rare: only receivers whose bilinear cell
// touches the border of the octahedral square.
__device__ __noinline__ float sample_border(const float* __restrict__ A, int W, int plane, int k0, int k1, int ix,
                                            int iy, float wx, float wy, float wk, int kb, int ke) {
    // shells outside [kb, ke) are not held (a multi-GPU shell chunk): their taps count 0
    const float w0 = (k0 >= kb && k0 < ke) ? 1.0f - wk : 0.0f, w1 = (k1 >= kb && k1 < ke) ? wk : 0.0f;
    k0 = w0 != 0.0f ? k0 - kb : 0;
    k1 = w1 != 0.0f ? k1 - kb : 0;
    float acc = 0.0f;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            int c = ix + dx, r = iy + dy;
            wrap_tap(c, r, W, W);
            const int o = r * W + c;
            const float wxy = (dx ? wx : 1.0f - wx) * (dy ? wy : 1.0f - wy);
            if (w0 != 0.0f) acc = fmaf(wxy * w0, __ldg(A + k0 * plane + o), acc);
            if (w1 != 0.0f) acc = fmaf(wxy * w1, __ldg(A + k1 * plane + o), acc);
        }
    return acc;
}

// Trilinear T_l at x (fp64 position): octahedral bilinear x radial linear
// (R10).  Index math in fp64 — at 2048^2 an fp32 texel
// coordinate has ulp 2.4e-4 — with the reciprocal and square root as an fp32
// MUFU seed plus one fp64 Newton step (relative error ~1e-14, not correctly
// rounded: no integer decision here needs bit-exactness, the trilinear
// result is continuous in them).  Taps in fp32.
// kRange: A holds only shells [kb, ke) of the light (a multi-GPU shell chunk,
// A = shell kb); taps on other shells count 0, so the sum over the chunks of
// all ranks is the full trilinear value (it is linear in the atlas).
template <bool kRange = false>
__device__ __forceinline__ float sample_light(const float* __restrict__ A, const QLight& L, int W, int K,
                                              double px, double py, double pz, int kb = 0, int ke = 0) {
    const double mx = px - L.ox, my = py - L.oy, mz = pz - L.oz;
    const double t2 = fma(mx, mx, fma(my, my, mz * mz));
    if (t2 == 0.0) return 1.0f;  // at the light (Q18)
    // psi(m): q = m / |m|_1, folded for q_z < 0, sgn(0) = +1 (Q4)
    const double n1 = (fabs(mx) + fabs(my)) + fabs(mz);
    double r = (double)rcp_approx((float)n1);
    r = fma(r, fma(-n1, r, 1.0), r);
    const double qx = mx * r, qy = my * r;
    double u = qx, v = qy;
    if (mz < 0.0) {
        u = (qx >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(qy));
        v = (qy >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(qx));
    }
    // texel-centre coordinates: fx = (u + 1) W/2 - 1/2
    const double hw = 0.5 * W;
    const double fx = fma(u, hw, hw - 0.5), fy = fma(v, hw, hw - 0.5);
    const double x0 = floor(fx), y0 = floor(fy);
    const float wx = (float)(fx - x0), wy = (float)(fy - y0);
    // shell coordinate fk = t K / t_max - 1/2, clamped to [0, K-1]
    double y = (double)rsqrt_approx((float)t2);
    y = y * fma(-0.5 * t2, y * y, 1.5);
    double fk = fma(t2 * y, L.kscale, -0.5);
    fk = fmin(fmax(fk, 0.0), (double)(K - 1));
    const double k0d = floor(fk);
    const float wk = (float)(fk - k0d);
    const int k0 = (int)k0d, k1 = k0 + 1 < K ? k0 + 1 : K - 1;
    const int ix = (int)x0, iy = (int)y0;
    const int plane = W * W;  // K * plane < 2^31 for K <= 256, W <= 2048
    if ((unsigned)ix >= (unsigned)(W - 1) || (unsigned)iy >= (unsigned)(W - 1))
        return sample_border(A, W, plane, k0, k1, ix, iy, wx, wy, wk, kRange ? kb : 0, kRange ? ke : K);
    // interior: each of the 4 tap rows (2 rows x 2 shells) is one aligned 16-B
    // load holding both column taps, plus a 4-B load when the pair straddles
    // the 16-B boundary; the column weights are placed at the taps' positions
    // in that 5-float window once per light, so the rows need no selects
    const int sub = ix & 3;
    const float cx0 = 1.0f - wx, cx1 = wx;
    const float c0 = sub == 0 ? cx0 : 0.0f;
    const float c1 = sub == 0 ? cx1 : (sub == 1 ? cx0 : 0.0f);
    const float c2 = sub == 1 ? cx1 : (sub == 2 ? cx0 : 0.0f);
    const float c3 = sub == 2 ? cx1 : (sub == 3 ? cx0 : 0.0f);
    const float c4 = sub == 3 ? cx1 : 0.0f;
    const int cofs = iy * W + (ix - sub);
    if (kRange) {
        const bool own0 = k0 >= kb && k0 < ke, own1 = k1 >= kb && k1 < ke;
        const float* p00 = A + ((own0 ? k0 - kb : 0) * plane + cofs);
        const float* p10 = A + ((own1 ? k1 - kb : 0) * plane + cofs);
        const float* rows[4] = {p00, p00 + W, p10, p10 + W};
        const bool own[4] = {own0, own0, own1, own1};
        float4 q[4];
        float e[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            q[j] = own[j] ? __ldg(reinterpret_cast<const float4*>(rows[j])) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int j = 0; j < 4; ++j) e[j] = (own[j] && sub == 3) ? __ldg(rows[j] + 4) : 0.0f;
        float s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) s[j] = fmaf(c4, e[j], fmaf(c3, q[j].w, fmaf(c2, q[j].z, fmaf(c1, q[j].y, c0 * q[j].x))));
        const float wy0 = 1.0f - wy, wk0 = 1.0f - wk;
        return fmaf(wy * wk, s[3], fmaf(wy0 * wk, s[2], fmaf(wy * wk0, s[1], wy0 * wk0 * s[0])));
    }
    const float* p00 = A + (k0 * plane + cofs);
    const float* p10 = A + (k1 * plane + cofs);
    const float* rows[4] = {p00, p00 + W, p10, p10 + W};
    float4 q[4];
    float e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = __ldg(reinterpret_cast<const float4*>(rows[j]));
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = sub == 3 ? __ldg(rows[j] + 4) : 0.0f;
    float s[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = fmaf(c4, e[j], fmaf(c3, q[j].w, fmaf(c2, q[j].z, fmaf(c1, q[j].y, c0 * q[j].x))));
    const float wy0 = 1.0f - wy, wk0 = 1.0f - wk;
    return fmaf(wy * wk, s[3], fmaf(wy0 * wk, s[2], fmaf(wy * wk0, s[1], wy0 * wk0 * s[0])));
}

__device__ __forceinline__ void apply_colors(float* colors, int64_t q, float T) {
    if (colors) {
        colors[3 * q] *= T;
        colors[3 * q + 1] *= T;
        colors[3 * q + 2] *= T;
    }
}

#ifndef DGSM_QPT
#define DGSM_QPT 1
#endif
// kQPT receivers per thread (strided by the block size: loads stay coalesced),
// their light loops interleaved: independent index chains and tap gathers in flight.
constexpr int kQPT = DGSM_QPT;
constexpr int kQThreads = 256;
// 8 CTAs of 256 per SM (32 registers, full occupancy): more gathers in flight.
// Measured (tools/query_bench2.py, L2 flushed, pre-permuted receivers): cfg2
// 20.5 -> 18.5 us, cfg5 397 -> 358 us against no bound (56 registers, 4 CTAs/SM);
// 5 and 6 CTAs/SM lie between.
#ifndef DGSM_QMINB
#define DGSM_QMINB 8
#endif
// k_query_chunks (the multi-GPU step's query, also at N = 1): 6 CTAs/SM (40 registers);
// cfg5 0.427 / 0.374 / 0.458 ms at no bound / 6 / 8 (8: 32 registers with spills)
#ifndef DGSM_QCMINB
#define DGSM_QCMINB 6
#endif

__global__ void __launch_bounds__(kQThreads, DGSM_QMINB) k_query(const float* __restrict__ atlas, QueryLights ql,
                                                     int n_lights, int res, int K,
                                                     const float* __restrict__ pos, int64_t m,
                                                     float* __restrict__ T_out, float* __restrict__ colors) {
    pdl_begin();
    const int64_t base = (int64_t)blockIdx.x * (kQThreads * kQPT) + threadIdx.x;
    const size_t per_light = (size_t)K * res * res;
    double px[kQPT], py[kQPT], pz[kQPT];
    float T[kQPT];
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
        const int64_t q = min(base + j * kQThreads, m - 1);
        px[j] = __ldg(pos + 3 * q); py[j] = __ldg(pos + 3 * q + 1); pz[j] = __ldg(pos + 3 * q + 2);
        T[j] = 1.0f;
    }
    for (int l = 0; l < n_lights; ++l) {
        const float* A = atlas + l * per_light;
#pragma unroll
        for (int j = 0; j < kQPT; ++j) T[j] *= sample_light(A, ql.l[l], res, K, px[j], py[j], pz[j]);
    }
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
        const int64_t q = base + j * kQThreads;
        if (q < m) {
            T_out[q] = T[j];
            apply_colors(colors, q, T[j]);
        }
    }
}

// Receivers in a spatially coherent order (dgsm_receiver_order): thread j
// serves receiver order[j] — its position gathered, its T scattered — so the
// 32 lanes of a warp sit next to each other in space and, for every light, hit
// neighbouring atlas texels and shells: shared 32-B sectors, open DRAM pages,
// few TLB entries, instead of one random gather per lane into a multi-GiB atlas.
__global__ void __launch_bounds__(kQThreads, DGSM_QMINB) k_query_ordered(const float* __restrict__ atlas, QueryLights ql,
                                                             int n_lights, int res, int K,
                                                             const float* __restrict__ pos,
                                                             const uint32_t* __restrict__ order, int64_t m,
                                                             float* __restrict__ T_out, float* __restrict__ colors) {
    pdl_begin();
    const int64_t base = (int64_t)blockIdx.x * (kQThreads * kQPT) + threadIdx.x;
    const size_t per_light = (size_t)K * res * res;
    double px[kQPT], py[kQPT], pz[kQPT];
    int64_t qi[kQPT];
    float T[kQPT];
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
        qi[j] = __ldg(order + min(base + j * kQThreads, m - 1));
        const int64_t q = qi[j];
        px[j] = __ldg(pos + 3 * q); py[j] = __ldg(pos + 3 * q + 1); pz[j] = __ldg(pos + 3 * q + 2);
        T[j] = 1.0f;
    }
    for (int l = 0; l < n_lights; ++l) {
        const float* A = atlas + l * per_light;
#pragma unroll
        for (int j = 0; j < kQPT; ++j) T[j] *= sample_light(A, ql.l[l], res, K, px[j], py[j], pz[j]);
    }
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
        if (base + j * kQThreads < m) {
            T_out[qi[j]] = T[j];
            apply_colors(colors, qi[j], T[j]);
        }
    }
}

// Order-preserving float <-> uint32 map (for atomicMin/Max on floats).
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Four receivers per thread as three aligned 16-B loads (12 floats = 4 x xyz);
// the m % 4 tail one point at a time.
__device__ __forceinline__ void load4(const float* __restrict__ pos, int64_t m, int64_t g, float x[4], float y[4],
                                      float z[4], int& cnt) {
    const int64_t i0 = 4 * g;
    cnt = (int)(m - i0 < 4 ? m - i0 : 4);
    if (cnt == 4) {
        const float4* p = reinterpret_cast<const float4*>(pos + 3 * i0);
        const float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
        x[0] = a.x; y[0] = a.y; z[0] = a.z; x[1] = a.w; y[1] = b.x; z[1] = b.y;
        x[2] = b.z; y[2] = b.w; z[2] = c.x; x[3] = c.y; y[3] = c.z; z[3] = c.w;
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + (u < cnt ? u : 0);
            x[u] = __ldg(pos + 3 * i); y[u] = __ldg(pos + 3 * i + 1); z[u] = __ldg(pos + 3 * i + 2);
        }
    }
}

// Bounding box of the receivers: box[0..2] = min, box[3..5] = max (ordered uints;
// the caller sets them to 0xffffffff / 0 first).  Non-finite coordinates are
// skipped.  Warp shuffles, then one shared-memory merge per CTA, then one
// atomic per CTA and axis.
__global__ void __launch_bounds__(256) k_aabb(const float* __restrict__ pos, int64_t m, uint32_t* box) {
    pdl_begin();
    __shared__ uint32_t s_box[6];
    if (threadIdx.x < 6) s_box[threadIdx.x] = threadIdx.x < 3 ? 0xffffffffu : 0u;
    __syncthreads();
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    const int64_t groups = (m + 3) / 4;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        float x[4], y[4], z[4];
        int cnt;
        load4(pos, m, g, x, y, z, cnt);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float v[3] = {x[u], y[u], z[u]};
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (isfinite(v[a])) { lo[a] = fminf(lo[a], v[a]); hi[a] = fmaxf(hi[a], v[a]); }
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a)
            if (lo[a] <= hi[a]) {
                atomicMin(&s_box[a], f2ord(lo[a]));
                atomicMax(&s_box[3 + a], f2ord(hi[a]));
            }
    __syncthreads();
    if (threadIdx.x < 3) {
        if (s_box[threadIdx.x] != 0xffffffffu) atomicMin(box + threadIdx.x, s_box[threadIdx.x]);
    } else if (threadIdx.x < 6) {
        if (s_box[threadIdx.x] != 0u) atomicMax(box + threadIdx.x, s_box[threadIdx.x]);
    }
}

#ifndef DGSM_ORDER_BITS
#define DGSM_ORDER_BITS 30
#endif
// Sharded atlases (multi-GPU): per light, the chunk of shells
// [kb, ke) this rank holds.  Complete lights (every shell held) multiply into
// T_out; split lights write the partial trilinear sum of their held taps into
// partial_out[j][q] (j = running index of the split lights), to be summed over
// the ranks sharing the light (all-reduce SUM) and multiplied in by
// k_query_combine.
struct ChunkParam {
    const float* data[DGSM_MAX_LIGHTS];
    int kb[DGSM_MAX_LIGHTS], ke[DGSM_MAX_LIGHTS];
    int split[DGSM_MAX_LIGHTS];
};

__global__ void __launch_bounds__(kQThreads, DGSM_QCMINB) k_query_chunks(ChunkParam cp, QueryLights ql, int n_lights, int res,
                                                            int K, const float* __restrict__ pos, int64_t m,
                                                            float* __restrict__ T_out,
                                                            float* __restrict__ partial_out) {
    pdl_begin();
    const int64_t q = (int64_t)blockIdx.x * kQThreads + threadIdx.x;
    if (q >= m) return;
    const double px = __ldg(pos + 3 * q), py = __ldg(pos + 3 * q + 1), pz = __ldg(pos + 3 * q + 2);
    float T = 1.0f;
    int j = 0;
    for (int l = 0; l < n_lights; ++l) {
        if (cp.kb[l] >= cp.ke[l] && !cp.split[l]) continue;  // (an empty complete chunk cannot occur)
        const float v = sample_light<true>(cp.data[l], ql.l[l], res, K, px, py, pz, cp.kb[l], cp.ke[l]);
        if (cp.split[l]) partial_out[(size_t)(j++) * m + q] = v;
        else T *= v;
    }
    if (T_out) T_out[q] = T;
}

// T *= prod_j partial[j] (the product over lights, Q13, of the summed shell chunks)
__global__ void __launch_bounds__(256) k_query_combine(const float* __restrict__ partial, int n, int64_t m,
                                                       float* __restrict__ T) {
    pdl_begin();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    float t = T[q];
    for (int j = 0; j < n; ++j) t *= __ldg(partial + (size_t)j * m + q);
    T[q] = t;
}

// 30-bit Morton code (10 bits per axis) of each receiver in its bounding box
// (positions outside are clamped: they only sort less tightly), value = index;
// the onesweep digit histograms of the keys are counted here (no k_hist pass).
__device__ __forceinline__ uint32_t spread10(uint32_t x) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__global__ void __launch_bounds__(256) k_morton(const float* __restrict__ pos, int64_t m,
                                                const uint32_t* __restrict__ box,
                                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                PassDigits pd, uint32_t* __restrict__ hist) {
    pdl_begin();
    __shared__ uint32_t sh[kSortMaxPasses][kSortRadix];
    for (int t = threadIdx.x; t < pd.passes * kSortRadix; t += blockDim.x) (&sh[0][0])[t] = 0u;
    float lo[3], ie[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = ord2f(box[a]);
        const float ext = ord2f(box[3 + a]) - lo[a];
        ie[a] = ext > 0.0f ? 1024.0f / ext : 0.0f;
    }
    __syncthreads();
    auto cell = [](float v, float l, float ie) {
        const float c = (v - l) * ie;  // in [0, 1024]; NaN -> 0
        return (uint32_t)fminf(fmaxf(c, 0.0f), 1023.0f);
    };
    const int64_t groups = (m + 3) / 4;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        float x[4], y[4], z[4];
        int cnt;
        load4(pos, m, g, x, y, z, cnt);
        uint32_t k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            k[u] = (spread10(cell(x[u], lo[0], ie[0])) | (spread10(cell(y[u], lo[1], ie[1])) << 1) |
                    (spread10(cell(z[u], lo[2], ie[2])) << 2)) >> (30 - DGSM_ORDER_BITS);
            if (u < cnt)
                for (int p = 0; p < pd.passes; ++p) atomicAdd(&sh[p][(k[u] >> pd.shift[p]) & ((1u << pd.bits[p]) - 1u)], 1u);
        }
        if (cnt == 4) {
            const uint32_t i0 = (uint32_t)(4 * g);
            reinterpret_cast<uint4*>(keys)[g] = make_uint4(k[0], k[1], k[2], k[3]);
            reinterpret_cast<uint4*>(vals)[g] = make_uint4(i0, i0 + 1, i0 + 2, i0 + 3);
        } else {
            for (int u = 0; u < cnt; ++u) {
                keys[4 * g + u] = k[u];
                vals[4 * g + u] = (uint32_t)(4 * g + u);
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < pd.passes * kSortRadix; t += blockDim.x) {
        const uint32_t c = (&sh[0][0])[t];
        if (c) atomicAdd(&hist[t], c);
    }
}

// NEXT-2 ("sampling only at Gaussian centers ... rather than integrating
// over each receiver's footprint"; "sampling only the Gaussian center
// ... tends to underestimate soft shadowing"): the receiver's transmittance is
// the footprint average  T_g = prod_l sum_i w_i T_l(mu_g + R_g (s_g . z_i))
// over caller-given standard-normal offsets z_i (a quadrature stencil or Monte
// Carlo draws).  R_g and the sample points in fp64, like the oracle; the
// offsets live in the kernel parameters (<= 64 samples).
__global__ void __launch_bounds__(128) k_query_footprint(const float* __restrict__ atlas, QueryLights ql,
                                                         FootprintParam fp, int n_lights, int res, int K,
                                                         const float* __restrict__ means,
                                                         const float* __restrict__ scales,
                                                         const float* __restrict__ rots, int64_t m,
                                                         float* __restrict__ T_out, float* __restrict__ colors) {
    pdl_begin();
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= m) return;
    const double mx = __ldg(means + 3 * g), my = __ldg(means + 3 * g + 1), mz = __ldg(means + 3 * g + 2);
    const double sx = __ldg(scales + 3 * g), sy = __ldg(scales + 3 * g + 1), sz = __ldg(scales + 3 * g + 2);
    double qw = __ldg(rots + 4 * g), qx = __ldg(rots + 4 * g + 1), qy = __ldg(rots + 4 * g + 2),
           qz = __ldg(rots + 4 * g + 3);
    const double qn = sqrt(((qw * qw + qx * qx) + qy * qy) + qz * qz);
    qw /= qn; qx /= qn; qy /= qn; qz /= qn;
    // columns of R scaled by s: M = R diag(s)
    const double m00 = (1.0 - 2.0 * (qy * qy + qz * qz)) * sx, m01 = 2.0 * (qx * qy - qw * qz) * sy,
                 m02 = 2.0 * (qx * qz + qw * qy) * sz;
    const double m10 = 2.0 * (qx * qy + qw * qz) * sx, m11 = (1.0 - 2.0 * (qx * qx + qz * qz)) * sy,
                 m12 = 2.0 * (qy * qz - qw * qx) * sz;
    const double m20 = 2.0 * (qx * qz - qw * qy) * sx, m21 = 2.0 * (qy * qz + qw * qx) * sy,
                 m22 = (1.0 - 2.0 * (qx * qx + qy * qy)) * sz;
    const size_t per_light = (size_t)K * res * res;
    float T = 1.0f;
    for (int l = 0; l < n_lights; ++l) {
        const float* A = atlas + l * per_light;
        const QLight& L = ql.l[l];
        float acc = 0.0f;
        for (int i = 0; i < fp.n; ++i) {
            const float4 z = fp.zw[i];
            const double zx = z.x, zy = z.y, zz = z.z;
            const double x = mx + ((m00 * zx + m01 * zy) + m02 * zz);
            const double y = my + ((m10 * zx + m11 * zy) + m12 * zz);
            const double w = mz + ((m20 * zx + m21 * zy) + m22 * zz);
            acc = fmaf(z.w, sample_light(A, L, res, K, x, y, w), acc);
        }
        T *= acc;
    }
    T_out[g] = T;
    apply_colors(colors, g, T);
}

QueryLights query_lights(const LightsParam& lp, int n_lights, int K) {
    QueryLights ql;
    for (int l = 0; l < DGSM_MAX_LIGHTS; ++l) {
        const bool on = l < n_lights;
        ql.l[l].ox = on ? (double)lp.l[l].x : 0.0;
        ql.l[l].oy = on ? (double)lp.l[l].y : 0.0;
        ql.l[l].oz = on ? (double)lp.l[l].z : 0.0;
        ql.l[l].kscale = on ? (double)K / (double)lp.l[l].w : 0.0;
    }
    return ql;
}

unsigned query_blocks(int64_t m) { return (unsigned)((m + kQThreads * kQPT - 1) / (kQThreads * kQPT)); }
}  // namespace

void launch_query(const float* atlas, const LightsParam& lp, int n_lights, int res, int K,
                  const float* positions, int64_t m, float* T_out, float* colors, cudaStream_t s) {
    if (m <= 0) return;
    pdl_launch(k_query, query_blocks(m), kQThreads, 0, s, atlas, query_lights(lp, n_lights, K), n_lights, res, K, positions,
                                                  m, T_out, colors);
}

void launch_query_ordered(const float* atlas, const LightsParam& lp, int n_lights, int res, int K,
                          const float* positions, const uint32_t* order, int64_t m, float* T_out, float* colors,
                          cudaStream_t s) {
    if (m <= 0) return;
    pdl_launch(k_query_ordered, query_blocks(m), kQThreads, 0, s, atlas, query_lights(lp, n_lights, K), n_lights, res, K,
                                                          positions, order, m, T_out, colors);
}

void launch_query_chunks(const float* const* chunks, const int* kb, const int* ke, const int* split,
                         const LightsParam& lp, int n_lights, int res, int K, const float* positions, int64_t m,
                         float* T_out, float* partial_out, cudaStream_t s) {
    if (m <= 0) return;
    ChunkParam cp;
    memset(&cp, 0, sizeof(cp));
    for (int l = 0; l < n_lights; ++l) {
        cp.data[l] = chunks[l];
        cp.kb[l] = kb[l];
        cp.ke[l] = ke[l];
        cp.split[l] = split[l];
    }
    pdl_launch(k_query_chunks, (unsigned)((m + kQThreads - 1) / kQThreads), kQThreads, 0, s, 
        cp, query_lights(lp, n_lights, K), n_lights, res, K, positions, m, T_out, partial_out);
}

void launch_query_combine(const float* partial, int n, int64_t m, float* T, cudaStream_t s) {
    if (m <= 0) return;
    pdl_launch(k_query_combine, (unsigned)((m + 255) / 256), 256, 0, s, partial, n, m, T);
}

void launch_morton(const float* positions, int64_t m, uint32_t* box, uint32_t* keys, uint32_t* vals,
                   const PassDigits& pd, uint32_t* hist, cudaStream_t s) {
    if (m <= 0) return;
    cudaMemsetAsync(box, 0xff, 3 * sizeof(uint32_t), s);
    cudaMemsetAsync(box + 3, 0, 3 * sizeof(uint32_t), s);
    const int64_t groups = (m + 3) / 4;
    const unsigned blocks = (unsigned)std::min<int64_t>((groups + 255) / 256, 148 * 4);
    pdl_launch(k_aabb, blocks, 256, 0, s, positions, m, box);
    pdl_launch(k_morton, blocks, 256, 0, s, positions, m, box, keys, vals, pd, hist);
}

void launch_query_footprint(const float* atlas, const LightsParam& lp, const FootprintParam& fp, int n_lights,
                            int res, int K, const float* means, const float* scales, const float* rotations,
                            int64_t m, float* T_out, float* colors, cudaStream_t s) {
    if (m <= 0) return;
    pdl_launch(k_query_footprint, (unsigned)((m + 127) / 128), 128, 0, s, atlas, query_lights(lp, n_lights, K), fp, n_lights, res, K, means, scales,
                                                                  rotations, m, T_out, colors);
}

}  // namespace dgsm
