// query.cu — a8: DGSM sampling (§3.3).  Each receiver
// centre x fetches T[psi(d), t(x)] "via trilinear interpolation" per light:
// octahedral bilinear with mirror-wrapped taps across the atlas border (Q12) x
// radial linear with t clamped to [t_0, t_{K-1}]; T = 1 at the light (Q18);
// product over lights (Q13); optional colour *= T ("multiply the direct term").
// Index math in fp64 (at 2048^2 the fp32 texel coordinate has ulp 2.4e-4).
// HBM/L2 bound: 12 B position + 8 x 4 B taps per light + 4 B output per query.
#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
__device__ __forceinline__ void wrap_tap(int& col, int& row, int W, int H) {
    if (col < 0) { col = -1 - col; row = H - 1 - row; }
    else if (col > W - 1) { col = 2 * W - 1 - col; row = H - 1 - row; }
    if (row < 0) { row = -1 - row; col = W - 1 - col; }
    else if (row > H - 1) { row = 2 * H - 1 - row; col = W - 1 - col; }
}

// Trilinear T_l at x (fp64 position): octahedral bilinear x radial linear.
__device__ __forceinline__ float sample_light(const float* __restrict__ A, const float4 L, int res, int K,
                                              double px, double py, double pz) {
    const int W = res, H = res;
    const size_t plane = (size_t)H * W;
    const double mx = px - (double)L.x;
    const double my = py - (double)L.y;
    const double mz = pz - (double)L.z;
    const double t = sqrt((mx * mx + my * my) + mz * mz);
    if (t == 0.0) return 1.0f;
    const double inv1 = 1.0 / ((fabs(mx) + fabs(my)) + fabs(mz));
    const double qx = mx * inv1, qy = my * inv1, qz = mz * inv1;
    double u, v;
    if (qz >= 0.0) { u = qx; v = qy; }
    else {
        u = (qx >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(qy));
        v = (qy >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(qx));
    }
    const double fx = (u + 1.0) * (0.5 * W) - 0.5;
    const double fy = (v + 1.0) * (0.5 * H) - 0.5;
    const double x0 = floor(fx), y0 = floor(fy);
    const float wx = (float)(fx - x0), wy = (float)(fy - y0);
    double fk = (t * K) / (double)L.w - 0.5;
    fk = fk < 0.0 ? 0.0 : (fk > K - 1 ? (double)(K - 1) : fk);
    const double k0d = floor(fk);
    const float wk = (float)(fk - k0d);
    const int k0 = (int)k0d, k1 = k0 + 1 < K ? k0 + 1 : K - 1;
    const float* A0 = A + (size_t)k0 * plane;
    const float* A1 = A + (size_t)k1 * plane;
    float acc = 0.0f;
    const int ix = (int)x0, iy = (int)y0;
    if (ix >= 0 && ix + 1 <= W - 1 && iy >= 0 && iy + 1 <= H - 1) {
        // interior: both column taps of a row from one aligned 16-B load (one L1
        // wavefront per row instead of two; the gather is L1-wavefront bound),
        // a second load only when the pair straddles the 16-B boundary
        const int c4 = ix & ~3, sub = ix & 3;
        float v[2][2][2];  // [shell][row][col]
#pragma unroll
        for (int dk = 0; dk < 2; ++dk)
#pragma unroll
            for (int dy = 0; dy < 2; ++dy) {
                const float* rp = (dk ? A1 : A0) + (size_t)(iy + dy) * W;
                const float4 q = __ldg(reinterpret_cast<const float4*>(rp + c4));
                v[dk][dy][0] = sub == 0 ? q.x : sub == 1 ? q.y : sub == 2 ? q.z : q.w;
                v[dk][dy][1] = sub == 0 ? q.y : sub == 1 ? q.z : sub == 2 ? q.w : __ldg(rp + ix + 1);
            }
#pragma unroll
        for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                const float wxy = (dx ? wx : 1.0f - wx) * (dy ? wy : 1.0f - wy);
                acc = fmaf(wxy * (1.0f - wk), v[0][dy][dx], acc);
                acc = fmaf(wxy * wk, v[1][dy][dx], acc);
            }
        return acc;
    }
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            int c = (int)x0 + dx, r = (int)y0 + dy;
            wrap_tap(c, r, W, H);
            const size_t o = (size_t)r * W + c;
            const float wxy = (dx ? wx : 1.0f - wx) * (dy ? wy : 1.0f - wy);
            acc = fmaf(wxy * (1.0f - wk), __ldg(A0 + o), acc);
            acc = fmaf(wxy * wk, __ldg(A1 + o), acc);
        }
    return acc;
}

__device__ __forceinline__ void apply_colors(float* colors, int64_t q, float T) {
    if (colors) {
        colors[3 * q] *= T;
        colors[3 * q + 1] *= T;
        colors[3 * q + 2] *= T;
    }
}

// kQPT receivers per thread: independent fp64 index chains and tap gathers in
// flight together (the kernel is latency bound, not bandwidth bound).
constexpr int kQPT = 1;

__global__ void __launch_bounds__(256, 6) k_query(const float* __restrict__ atlas, LightsParam lp,
                                               int n_lights, int res, int K,
                                               const float* __restrict__ pos, int64_t m,
                                               float* __restrict__ T_out, float* __restrict__ colors) {
    const int64_t q0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kQPT;
    if (q0 >= m) return;
    const size_t per_light = (size_t)K * res * res;
    double px[kQPT], py[kQPT], pz[kQPT];
    float T[kQPT];
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
        const int64_t q = q0 + j < m ? q0 + j : m - 1;
        px[j] = __ldg(pos + 3 * q); py[j] = __ldg(pos + 3 * q + 1); pz[j] = __ldg(pos + 3 * q + 2);
        T[j] = 1.0f;
    }
    for (int l = 0; l < n_lights; ++l) {
#pragma unroll
        for (int j = 0; j < kQPT; ++j)
            T[j] *= sample_light(atlas + l * per_light, lp.l[l], res, K, px[j], py[j], pz[j]);
    }
#pragma unroll
    for (int j = 0; j < kQPT; ++j) {
        if (q0 + j < m) {
            T_out[q0 + j] = T[j];
            apply_colors(colors, q0 + j, T[j]);
        }
    }
}

// NEXT-2 ("sampling only at Gaussian centers ... rather than integrating
// over each receiver's footprint"; "sampling only the Gaussian center
// ... tends to underestimate soft shadowing"): the receiver's transmittance is
// the footprint average  T_g = prod_l sum_i w_i T_l(mu_g + R_g (s_g . z_i))
// over caller-given standard-normal offsets z_i (a quadrature stencil or Monte
// Carlo draws).  R_g and the sample points in fp64, like the oracle; the
// offsets live in the kernel parameters (<= 64 samples).
__global__ void __launch_bounds__(128) k_query_footprint(const float* __restrict__ atlas, LightsParam lp,
                                                         FootprintParam fp, int n_lights, int res, int K,
                                                         const float* __restrict__ means,
                                                         const float* __restrict__ scales,
                                                         const float* __restrict__ rots, int64_t m,
                                                         float* __restrict__ T_out, float* __restrict__ colors) {
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
        const float4 L = lp.l[l];
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
}  // namespace

void launch_query(const float* atlas, const LightsParam& lp, int n_lights, int res, int K,
                  const float* positions, int64_t m, float* T_out, float* colors, cudaStream_t s) {
    if (m <= 0) return;
    const int64_t threads = (m + kQPT - 1) / kQPT;
    k_query<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(atlas, lp, n_lights, res, K, positions, m, T_out,
                                                              colors);
}

void launch_query_footprint(const float* atlas, const LightsParam& lp, const FootprintParam& fp, int n_lights,
                            int res, int K, const float* means, const float* scales, const float* rotations,
                            int64_t m, float* T_out, float* colors, cudaStream_t s) {
    if (m <= 0) return;
    k_query_footprint<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(atlas, lp, fp, n_lights, res, K, means, scales,
                                                                  rotations, m, T_out, colors);
}

}  // namespace dgsm
