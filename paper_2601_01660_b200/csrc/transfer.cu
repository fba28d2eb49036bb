// transfer.cu — NEXT-4: SH lighting transfer (§3.5).
//
//   L_c(w_j) = max(0, B(w_j) A_c)                      radiance of the fitted SH probe
//   S(w, n)  = max(0, <w, n>)^q                        cosine lobe (Lambertian q = 1)
//   s_c(n)   = clip_[0, s_max]( sum_j w_j L_c S / (sum_j w_j S + eps) )
//   c'       = max(0, gamma c (.) s(n))
//
// over a lat-long grid w_j with w_j ~ sin(theta_j) (reading R-SH).
// A dense per-Gaussian contraction over M directions, but with a max(0,.)^q
// nonlinearity between its two factors, so it is not a GEMM: FP32 FMA work
// (8 ops per (Gaussian, direction) at q = 1), ALU-bound.
//
//  k_transfer_grid: one thread per direction: w_j, and w_j L_c(w_j) from the
//                   real SH basis (Cartesian polynomials, degree <= 3).
//  k_transfer_part: kG Gaussians per thread, directions staged through shared
//                   memory (broadcast reads), a chunk of the grid per blockIdx.y;
//                   partial sums [chunk][n][4] (fixed layout: deterministic).
//  k_transfer_fin:  sums the chunks in order, ratio, clip, relit colour.
#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
constexpr int kG = 4;            // Gaussians per thread
constexpr int kThreadsT = 128;
constexpr int kTileDirs = 512;   // directions per shared-memory tile (16 KB)

// Real SH basis, orthonormal, Condon-Shortley phase, index l^2 + l + m, written
// out as Cartesian polynomials of the unit direction (degree <= 3).
__device__ __forceinline__ void sh_basis3(float x, float y, float z, int d, float* B) {
    B[0] = 0.28209479177387814f;
    if (d < 1) return;
    B[1] = -0.4886025119029199f * y;
    B[2] = 0.4886025119029199f * z;
    B[3] = -0.4886025119029199f * x;
    if (d < 2) return;
    const float xx = x * x, yy = y * y, zz = z * z;
    B[4] = 1.0925484305920792f * x * y;
    B[5] = -1.0925484305920792f * y * z;
    B[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
    B[7] = -1.0925484305920792f * x * z;
    B[8] = 0.5462742152960396f * (xx - yy);
    if (d < 3) return;
    B[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
    B[10] = 2.890611442640554f * x * y * z;
    B[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
    B[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    B[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
    B[14] = 1.445305721320277f * z * (xx - yy);
    B[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

__global__ void k_transfer_grid(ShParam sp, int n_theta, int n_phi, float4* __restrict__ dirs,
                                float4* __restrict__ wl) {
    pdl_begin();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_theta * n_phi) return;
    const int i = j / n_phi, k = j - i * n_phi;
    const double th = ((double)i + 0.5) * 3.141592653589793 / n_theta;
    const double ph = ((double)k + 0.5) * 2.0 * 3.141592653589793 / n_phi;
    double st, ct, sp_, cp;
    sincos(th, &st, &ct);
    sincos(ph, &sp_, &cp);
    const float x = (float)(st * cp), y = (float)(st * sp_), z = (float)ct;
    const float w = (float)(st * (3.141592653589793 / n_theta) * (2.0 * 3.141592653589793 / n_phi));
    float B[16];
    sh_basis3(x, y, z, sp.d, B);
    const int K = (sp.d + 1) * (sp.d + 1);
    float L[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float v = 0.0f;
        for (int q = 0; q < K; ++q) v = fmaf(B[q], sp.a[c][q], v);
        L[c] = fmaxf(v, 0.0f);  // negative SH ringing clamped (R-SH)
    }
    dirs[j] = make_float4(x, y, z, 0.0f);
    wl[j] = make_float4(w * L[0], w * L[1], w * L[2], w);
}

// S = max(0, x)^q: q = 1 and q = 2 exactly, other q by exp2(q log2 x)
template <int kQ>
__device__ __forceinline__ float lobe(float x, float q) {
    if (kQ == 1) return fmaxf(x, 0.0f);
    if (kQ == 2) { const float t = fmaxf(x, 0.0f); return t * t; }
    return x > 0.0f ? exp2f(q * __log2f(x)) : 0.0f;
}

template <int kQ>
__global__ void __launch_bounds__(kThreadsT) k_transfer_part(const float4* __restrict__ dirs,
                                                             const float4* __restrict__ wl, int M, int chunk,
                                                             const float* __restrict__ normals, int64_t n,
                                                             float q, float4* __restrict__ part) {
    pdl_begin();
    __shared__ float4 s_dir[kTileDirs], s_wl[kTileDirs];
    const int64_t g0 = ((int64_t)blockIdx.x * kThreadsT + threadIdx.x) * kG;
    float nx[kG], ny[kG], nz[kG];
    float4 acc[kG];
#pragma unroll
    for (int u = 0; u < kG; ++u) {
        const int64_t g = g0 + u < n ? g0 + u : n - 1;
        nx[u] = __ldg(normals + 3 * g); ny[u] = __ldg(normals + 3 * g + 1); nz[u] = __ldg(normals + 3 * g + 2);
        acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int j_begin = blockIdx.y * chunk, j_end = min(M, j_begin + chunk);
    for (int t0 = j_begin; t0 < j_end; t0 += kTileDirs) {
        const int nt = min(kTileDirs, j_end - t0);
        __syncthreads();
        for (int t = threadIdx.x; t < nt; t += kThreadsT) {
            s_dir[t] = dirs[t0 + t];
            s_wl[t] = wl[t0 + t];
        }
        __syncthreads();
        // per tile in fp32, tile sums added once (short fp32 sums)
        if constexpr (kQ == 1 || kQ == 2) {
            // Gaussian pairs on the paired FP32 pipe: (u, u+1) in one f32x2 register,
            // the direction's values broadcast
            f2_t TX[kG / 2], TY[kG / 2], TZ[kG / 2], TW[kG / 2], NX[kG / 2], NY[kG / 2], NZ[kG / 2];
#pragma unroll
            for (int p = 0; p < kG / 2; ++p) {
                TX[p] = TY[p] = TZ[p] = TW[p] = 0ull;
                NX[p] = f2pack(nx[2 * p], nx[2 * p + 1]);
                NY[p] = f2pack(ny[2 * p], ny[2 * p + 1]);
                NZ[p] = f2pack(nz[2 * p], nz[2 * p + 1]);
            }
#pragma unroll 4
            for (int t = 0; t < nt; ++t) {
                const float4 dv = s_dir[t], wv = s_wl[t];
                const f2_t DX = f2bc(dv.x), DY = f2bc(dv.y), DZ = f2bc(dv.z);
                const f2_t WX = f2bc(wv.x), WY = f2bc(wv.y), WZ = f2bc(wv.z), WW = f2bc(wv.w);
#pragma unroll
                for (int p = 0; p < kG / 2; ++p) {
                    const f2_t X = f2fma(NX[p], DX, f2fma(NY[p], DY, f2mul(NZ[p], DZ)));
                    f2_t S = f2pack(fmaxf(f2lo(X), 0.0f), fmaxf(f2hi(X), 0.0f));
                    if (kQ == 2) S = f2mul(S, S);
                    TX[p] = f2fma(S, WX, TX[p]);
                    TY[p] = f2fma(S, WY, TY[p]);
                    TZ[p] = f2fma(S, WZ, TZ[p]);
                    TW[p] = f2fma(S, WW, TW[p]);
                }
            }
#pragma unroll
            for (int p = 0; p < kG / 2; ++p) {
                acc[2 * p].x += f2lo(TX[p]); acc[2 * p + 1].x += f2hi(TX[p]);
                acc[2 * p].y += f2lo(TY[p]); acc[2 * p + 1].y += f2hi(TY[p]);
                acc[2 * p].z += f2lo(TZ[p]); acc[2 * p + 1].z += f2hi(TZ[p]);
                acc[2 * p].w += f2lo(TW[p]); acc[2 * p + 1].w += f2hi(TW[p]);
            }
        } else {
            float4 tacc[kG];
#pragma unroll
            for (int u = 0; u < kG; ++u) tacc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
            for (int t = 0; t < nt; ++t) {
                const float4 dv = s_dir[t], wv = s_wl[t];
#pragma unroll
                for (int u = 0; u < kG; ++u) {
                    const float S = lobe<kQ>(fmaf(nx[u], dv.x, fmaf(ny[u], dv.y, nz[u] * dv.z)), q);
                    tacc[u].x = fmaf(S, wv.x, tacc[u].x);
                    tacc[u].y = fmaf(S, wv.y, tacc[u].y);
                    tacc[u].z = fmaf(S, wv.z, tacc[u].z);
                    tacc[u].w = fmaf(S, wv.w, tacc[u].w);
                }
            }
#pragma unroll
            for (int u = 0; u < kG; ++u) {
                acc[u].x += tacc[u].x; acc[u].y += tacc[u].y; acc[u].z += tacc[u].z; acc[u].w += tacc[u].w;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < kG; ++u)
        if (g0 + u < n) part[(int64_t)blockIdx.y * n + g0 + u] = acc[u];
}

__global__ void k_transfer_fin(const float4* __restrict__ part, int n_chunks, int64_t n,
                               const float* __restrict__ colors, float eps, float s_max, float gamma,
                               float* __restrict__ scales_out, float* __restrict__ colors_out) {
    pdl_begin();
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    double num[3] = {0.0, 0.0, 0.0}, den = 0.0;
    for (int c = 0; c < n_chunks; ++c) {  // chunk order: deterministic
        const float4 p = part[(int64_t)c * n + g];
        num[0] += p.x; num[1] += p.y; num[2] += p.z; den += p.w;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float s = (float)(num[c] / (den + (double)eps));
        s = fminf(fmaxf(s, 0.0f), s_max);
        if (scales_out) scales_out[3 * g + c] = s;
        if (colors_out && colors) colors_out[3 * g + c] = fmaxf(gamma * colors[3 * g + c] * s, 0.0f);
    }
}
}  // namespace

size_t transfer_workspace_bytes(int n_theta, int n_phi, int64_t n) {
    const int64_t M = (int64_t)n_theta * n_phi;
    const int chunks = transfer_chunks(n, M);
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    return al(sizeof(float4) * M) * 2 + al(sizeof(float4) * (size_t)chunks * (size_t)(n > 0 ? n : 1));
}

int transfer_chunks(int64_t n, int64_t M) {
    // enough CTAs to fill the GPU: ~4 waves of 148 x 8 CTAs, chunks >= one tile
    const int64_t blocks_x = (n + (int64_t)kThreadsT * kG - 1) / ((int64_t)kThreadsT * kG);
    int64_t c = (148 * 8 * 2 + blocks_x - 1) / (blocks_x > 0 ? blocks_x : 1);
    const int64_t cmax = (M + kTileDirs - 1) / kTileDirs;
    if (c > cmax) c = cmax;
    if (c < 1) c = 1;
    return (int)c;
}

void launch_transfer(const ShParam& sp, int n_theta, int n_phi, float q, float eps, float s_max, float gamma,
                     const float* normals, const float* colors, int64_t n, float* scales_out, float* colors_out,
                     void* ws, cudaStream_t s, int* launches) {
    const int M = n_theta * n_phi;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    float4* dirs = (float4*)ws;
    float4* wl = (float4*)((char*)ws + al(sizeof(float4) * M));
    float4* part = (float4*)((char*)ws + 2 * al(sizeof(float4) * M));
    pdl_launch(k_transfer_grid, (M + 255) / 256, 256, 0, s, sp, n_theta, n_phi, dirs, wl);
    *launches += 1;
    if (n <= 0) return;
    const int chunks = transfer_chunks(n, M);
    const int chunk = ((M + chunks - 1) / chunks + kTileDirs - 1) / kTileDirs * kTileDirs;
    const int n_chunks = (M + chunk - 1) / chunk;
    dim3 grid((unsigned)((n + (int64_t)kThreadsT * kG - 1) / ((int64_t)kThreadsT * kG)), (unsigned)n_chunks);
    if (q == 1.0f)
        pdl_launch(k_transfer_part<1>, grid, kThreadsT, 0, s, dirs, wl, M, chunk, normals, n, q, part);
    else if (q == 2.0f)
        pdl_launch(k_transfer_part<2>, grid, kThreadsT, 0, s, dirs, wl, M, chunk, normals, n, q, part);
    else
        pdl_launch(k_transfer_part<0>, grid, kThreadsT, 0, s, dirs, wl, M, chunk, normals, n, q, part);
    pdl_launch(k_transfer_fin, (unsigned)((n + 255) / 256), 256, 0, s, part, n_chunks, n, colors, eps, s_max, gamma,
                                                              scales_out, colors_out);
    *launches += 2;
}

}  // namespace dgsm
