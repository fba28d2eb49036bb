// slab.cu — NEXT-1: receiver-driven ROI and active voxel slab (§3.2,
// P:L155-160).  "For scene Gaussians whose centers lie in B, we project their
// light rays into atlas pixels, collect the unique set P, and infer a tight
// radial range k in [k_min, k_max] from their light-space distances."
//
// One thread per receiver; the pixel set is a bit per texel grouped by 8x8
// tile (one u64 word per tile: the accumulation CTA of a tile reads its word
// once), written with atomicOr after a plain read (most receivers land on
// pixels another receiver already marked).  The k range is min/max reduced
// per warp, then one atomic per warp and light.  Compiled with -fmad=false:
// the pixel and bin decisions are fp64 in the oracle's operation order
// (bit-exact, reading R-ROI).
#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
__device__ __forceinline__ void wrap_px(long long& col, long long& row, int W, int H) {
    if (col < 0) { col = -1 - col; row = H - 1 - row; }
    else if (col > W - 1) { col = 2LL * W - 1 - col; row = H - 1 - row; }
    if (row < 0) { row = -1 - row; col = W - 1 - col; }
    else if (row > H - 1) { row = 2LL * H - 1 - row; col = W - 1 - col; }
}

__global__ void k_slab_init(uint64_t* __restrict__ mask, int64_t words, int2* __restrict__ kr, int n_lights,
                            int K) {
    pdl_begin();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < words) mask[i] = 0ull;
    if (i < n_lights) kr[i] = make_int2(K, -1);
}

__global__ void __launch_bounds__(256) k_active_slab(const float* __restrict__ x, int64_t m, float cx, float cy,
                                                     float R, float zmin, float zmax, LightsParam lp,
                                                     int n_lights, int res, int K,
                                                     unsigned long long* __restrict__ mask,
                                                     int2* __restrict__ kr) {
    pdl_begin();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool in = false;
    double px = 0.0, py = 0.0, pz = 0.0;
    if (q < m) {
        px = __ldg(x + 3 * q); py = __ldg(x + 3 * q + 1); pz = __ldg(x + 3 * q + 2);
        const double ex = fabs(px - (double)cx), ey = fabs(py - (double)cy);
        const double inf = ex > ey ? ex : ey;
        in = inf <= (double)R && pz >= (double)zmin && pz <= (double)zmax;
    }
    if (!__any_sync(0xffffffffu, in)) return;  // whole warp outside B (uniform exit)
    const int W = res, H = res, TW = res / kTile;
    const int64_t nt = (int64_t)TW * TW;
    for (int l = 0; l < n_lights; ++l) {
        const float4 L = lp.l[l];
        int lo = K, hi = -1;
        if (in) {
            const double mx = px - (double)L.x, my = py - (double)L.y, mz = pz - (double)L.z;
            const double t = sqrt((mx * mx + my * my) + mz * mz);
            if (t != 0.0) {
                // psi, the oracle's or_oct_encode operation order
                const double n1 = (fabs(mx) + fabs(my)) + fabs(mz);
                const double qx = mx / n1, qy = my / n1, qz = mz / n1;
                double u, v;
                if (qz >= 0.0) { u = qx; v = qy; }
                else {
                    u = (qx >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(qy));
                    v = (qy >= 0.0 ? 1.0 : -1.0) * (1.0 - fabs(qx));
                }
                long long col = (long long)floor((u + 1.0) * (0.5 * W));
                long long row = (long long)floor((v + 1.0) * (0.5 * H));
                if (col > W - 1) col = W - 1;
                if (row > H - 1) row = H - 1;
                unsigned long long* ml = mask + (int64_t)l * nt;
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx) {
                        long long c = col + dx, r = row + dy;
                        wrap_px(c, r, W, H);
                        const int64_t w = (r >> 3) * TW + (c >> 3);
                        const unsigned long long bit = 1ull << (((int)r & 7) * 8 + ((int)c & 7));
                        if (!(ml[w] & bit)) atomicOr(ml + w, bit);
                    }
                const double fb = floor((t * K) / (double)L.w);
                const int b = fb > K - 1 ? K - 1 : (int)fb;
                lo = b - 1 < 0 ? 0 : b - 1;
                hi = b + 1 > K - 1 ? K - 1 : b + 1;
            }
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if ((threadIdx.x & 31) == 0 && hi >= 0) {
            atomicMin(&kr[l].x, lo);
            atomicMax(&kr[l].y, hi);
        }
    }
}
}  // namespace

void launch_active_slab(const float* x, int64_t m, const dgsm_roi_t& roi, const LightsParam& lp, int n_lights,
                        int res, int K, uint64_t* mask, int2* kr, cudaStream_t s, int* launches) {
    const int64_t words = (int64_t)n_lights * (res / kTile) * (res / kTile);
    const int64_t init = words > n_lights ? words : n_lights;
    pdl_launch(k_slab_init, (unsigned)((init + 255) / 256), 256, 0, s, mask, words, kr, n_lights, K);
    *launches += 1;
    if (m <= 0) return;
    pdl_launch(k_active_slab, (unsigned)((m + 255) / 256), 256, 0, s, x, m, roi.center[0], roi.center[1], roi.radius,
                                                              roi.z_min, roi.z_max, lp, n_lights, res, K,
                                                              (unsigned long long*)mask, kr);
    *launches += 1;
}

}  // namespace dgsm
