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

__global__ void __launch_bounds__(256) k_query(const float* __restrict__ atlas, LightsParam lp,
                                               int n_lights, int res, int K,
                                               const float* __restrict__ pos, int64_t m,
                                               float* __restrict__ T_out, float* __restrict__ colors) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    const float px = __ldg(pos + 3 * q), py = __ldg(pos + 3 * q + 1), pz = __ldg(pos + 3 * q + 2);
    const int W = res, H = res;
    const size_t plane = (size_t)H * W;
    float T = 1.0f;
    for (int l = 0; l < n_lights; ++l) {
        const float4 L = lp.l[l];
        const double mx = (double)px - (double)L.x;
        const double my = (double)py - (double)L.y;
        const double mz = (double)pz - (double)L.z;
        const double t = sqrt((mx * mx + my * my) + mz * mz);
        if (t == 0.0) continue;
        const double n1 = (fabs(mx) + fabs(my)) + fabs(mz);
        const double qx = mx / n1, qy = my / n1, qz = mz / n1;
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
        const float* A0 = atlas + ((size_t)l * K + k0) * plane;
        const float* A1 = atlas + ((size_t)l * K + k1) * plane;
        float acc = 0.0f;
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
        T *= acc;
    }
    T_out[q] = T;
    if (colors) {
        colors[3 * q] *= T;
        colors[3 * q + 1] *= T;
        colors[3 * q + 2] *= T;
    }
}
}  // namespace

void launch_query(const float* atlas, const LightsParam& lp, int n_lights, int res, int K,
                  const float* positions, int64_t m, float* T_out, float* colors, cudaStream_t s) {
    if (m <= 0) return;
    k_query<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(atlas, lp, n_lights, res, K, positions, m, T_out,
                                                        colors);
}

}  // namespace dgsm
