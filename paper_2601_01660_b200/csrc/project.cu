// project.cu — N1: per (light, Gaussian) calibration + light-space footprint +
// 8x8 tile count (§3.2, Eq.5 and P:L162-173).
//
// Compiled with -fmad=false: the binning decisions (tile rectangle, tile count,
// depth key) are made in IEEE fp64 with the exact operation order of DESIGN.md's
// "binning arithmetic contract" (R4-R6) so that they are bit-identical to any
// implementation performing the same IEEE operations (the oracle is one).
#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
constexpr double kPi = 3.141592653589793;

__device__ __forceinline__ double sgn_pos(double x) { return x >= 0.0 ? 1.0 : -1.0; }  // sgn(0)=+1 (Q4)

__global__ void __launch_bounds__(256, 4) k_project(  // (256, 3) and (256, 2) measured slower
    const float* __restrict__ means, const float* __restrict__ scales,
    const float* __restrict__ rotations, const float* __restrict__ opacities, int64_t n, int64_t i0, int64_t cnt,
    LightsParam lp, int n_lights, int res, int K, double kappa, double k_sigma, double rho,
    int bin_mode, int absorption, bool no_cull, bool validate, const uint64_t* __restrict__ slab_mask,
    PairRec* __restrict__ recs, uint32_t* __restrict__ counts,
    uint4* __restrict__ dup,
    PlanStats* stats) {
    pdl_begin();
    // Gaussians [i0, i0 + cnt) of every light (a chunk of an upload pipeline, or all)
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = idx < (int64_t)n_lights * cnt;
    if (!active) idx = (int64_t)n_lights * cnt - 1;  // recompute the last element; results not stored twice
    const int l = (int)(idx / cnt);
    const int64_t i = i0 + (idx - (int64_t)l * cnt);
    const int64_t oi = (int64_t)l * n + i;  // output slot [l][i]
    uint32_t dbits = 0u;
    const float4 L = lp.l[l];
    const int W = res, H = res;

    // all inputs of the Gaussian loaded up front (one memory latency, not four)
    const float m0 = means[3 * i], m1 = means[3 * i + 1], m2 = means[3 * i + 2];
    const float q0 = rotations[4 * i], q1 = rotations[4 * i + 1], q2 = rotations[4 * i + 2], q3 = rotations[4 * i + 3];
    const float sc0 = scales[3 * i], sc1 = scales[3 * i + 1], sc2 = scales[3 * i + 2];
    const float alpha_in = opacities[i];
    const float kappa_f = (float)kappa;
    if (validate && active && l == 0) {  // DGSM_VALIDATE: once per Gaussian (light 0's thread)
        const bool ok = isfinite(m0) && isfinite(m1) && isfinite(m2) && isfinite(sc0) && isfinite(sc1) &&
                        isfinite(sc2) && sc0 > 0.0f && sc1 > 0.0f && sc2 > 0.0f && isfinite(q0) && isfinite(q1) &&
                        isfinite(q2) && isfinite(q3) && (q0 != 0.0f || q1 != 0.0f || q2 != 0.0f || q3 != 0.0f) &&
                        isfinite(alpha_in);
        if (!ok) {
            atomicAdd(&stats->n_invalid, 1u);
            atomicMin(&stats->first_invalid, (uint32_t)i);
        }
    }
    // R4: m = mu - o, D = |m|; excluded when D <= 1e-6 (Q17)
    const double mx = (double)m0 - (double)L.x;
    const double my = (double)m1 - (double)L.y;
    const double mz = (double)m2 - (double)L.z;
    const double D = sqrt((mx * mx + my * my) + mz * mz);
    uint32_t tcnt = 0;
    PairRec rec;
    int16_t rc0 = 1, rc1 = 0, rr0 = 1, rr1 = 0;  // packed footprint rect of the dup record
    if (D > 1e-6) {
        // footprint centre: octahedral encode psi(m) -> texel coords (pixel centres, Q3)
        const double inv1 = 1.0 / ((fabs(mx) + fabs(my)) + fabs(mz));  // contract v2: one division
        const double qx = mx * inv1, qy = my * inv1, qz = mz * inv1;
        double u, v;
        if (qz >= 0.0) { u = qx; v = qy; }
        else { u = sgn_pos(qx) * (1.0 - fabs(qy)); v = sgn_pos(qy) * (1.0 - fabs(qx)); }
        const double px = (u + 1.0) * (0.5 * W) - 0.5;
        const double py = (v + 1.0) * (0.5 * H) - 0.5;

        // rotation from the quaternion (w,x,y,z), normalised in fp64
        double qw = q0, qxr = q1, qyr = q2, qzr = q3;
        const double iqn = 1.0 / sqrt(((qw * qw + qxr * qxr) + qyr * qyr) + qzr * qzr);
        qw = qw * iqn; qxr = qxr * iqn; qyr = qyr * iqn; qzr = qzr * iqn;
        double R[3][3];
        R[0][0] = 1.0 - 2.0 * (qyr * qyr + qzr * qzr);
        R[0][1] = 2.0 * (qxr * qyr - qw * qzr);
        R[0][2] = 2.0 * (qxr * qzr + qw * qyr);
        R[1][0] = 2.0 * (qxr * qyr + qw * qzr);
        R[1][1] = 1.0 - 2.0 * (qxr * qxr + qzr * qzr);
        R[1][2] = 2.0 * (qyr * qzr - qw * qxr);
        R[2][0] = 2.0 * (qxr * qzr - qw * qyr);
        R[2][1] = 2.0 * (qyr * qzr + qw * qxr);
        R[2][2] = 1.0 - 2.0 * (qxr * qxr + qyr * qyr);

        // R5: lambda1 of Sigma_perp = [u v]^T Sigma [u v], basis-free form
        const double invD = 1.0 / D;
        const double dx = mx * invD, dy = my * invD, dz = mz * invD;
        double w[3], s2[3];
        const double s[3] = {(double)sc0, (double)sc1, (double)sc2};
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            w[j] = (R[0][j] * dx + R[1][j] * dy) + R[2][j] * dz;
            s2[j] = s[j] * s[j];
        }
        const double tr = (s2[0] * (1.0 - w[0] * w[0]) + s2[1] * (1.0 - w[1] * w[1])) +
                          s2[2] * (1.0 - w[2] * w[2]);
        const double det = ((s2[1] * s2[2]) * (w[0] * w[0]) + (s2[0] * s2[2]) * (w[1] * w[1])) +
                           (s2[0] * s2[1]) * (w[2] * w[2]);
        double disc = (tr * tr) * 0.25 - det;
        if (disc < 0.0) disc = 0.0;
        const double lam1 = tr * 0.5 + sqrt(disc);
        // rho = (rho_scale * (H + W)) / (2 pi) (Q5), the same IEEE double computed on the host
        const double p1 = ((k_sigma * sqrt(lam1)) * invD) * rho;

        // R6: integer texel range of the closed square, clamped to [-W, 2W-1]
        double c0 = ceil(px - p1), c1 = floor(px + p1), r0 = ceil(py - p1), r1 = floor(py + p1);
        if (c0 < -(double)W) c0 = -(double)W;
        if (c1 > 2.0 * W - 1.0) c1 = 2.0 * W - 1.0;
        if (r0 < -(double)H) r0 = -(double)H;
        if (r1 > 2.0 * H - 1.0) r1 = 2.0 * H - 1.0;
        if (no_cull) {  // ablation D: every tile of the atlas
            c0 = 0.0; c1 = W - 1.0; r0 = 0.0; r1 = H - 1.0;
        }
        const int ic0 = (int)c0, ic1 = (int)c1, ir0 = (int)r0, ir1 = (int)r1;
        if (ic0 > ic1 || ir0 > ir1) {
            tcnt = 0;
        } else if (slab_mask) {  // NEXT-1: only the tiles holding a texel of the ROI pixel set
            tcnt = count_active_tiles(ic0, ic1, ir0, ir1, res, bin_mode,
                                     slab_mask + (int64_t)l * (res / kTile) * (res / kTile));
        } else if (ic0 >= 0 && ic1 <= W - 1 && ir0 >= 0 && ir1 <= H - 1) {  // common case: inside the grid
            tcnt = (uint32_t)((ic1 >> 3) - (ic0 >> 3) + 1) * (uint32_t)((ir1 >> 3) - (ir0 >> 3) + 1);
        } else if (ic0 <= 0 && ic1 >= W - 1 && ir0 <= 0 && ir1 >= H - 1) {  // covers the grid: every tile once
            tcnt = (uint32_t)(W / kTile) * (uint32_t)(H / kTile);
        } else {
            TileRects TR;
            make_tile_rects(ic0, ic1, ir0, ir1, res, bin_mode, TR);
            tcnt = count_tiles(TR);
        }

        if (tcnt > 0) {
            rc0 = (int16_t)c0; rc1 = (int16_t)c1; rr0 = (int16_t)r0; rr1 = (int16_t)r1;
            rec.di[0] = dx; rec.di[1] = dy; rec.di[2] = dz;
            // record fields (not part of the binning contract; stored in fp32): fp32 math
            const float is[3] = {1.0f / sc0, 1.0f / sc1, 1.0f / sc2};  // 1/s_j
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                rec.g[j] = (float)w[j] * is[j];  // g = W d_i = diag(1/s) R^T d_i
#pragma unroll
                for (int c = 0; c < 3; ++c) rec.W[3 * j + c] = (float)R[c][j] * is[j];
            }
            const float Df = (float)D;
            rec.D = Df;
            const double dt = (double)L.w / K;
            int kD = (int)(D * ((double)K / (double)L.w));
            kD = kD < 0 ? 0 : (kD > K - 1 ? K - 1 : kD);
            rec.kD = kD;
            rec.eD = (float)((kD + 0.5) * dt - D);
            // Eq.5 with the clamp of Q16; times sqrt(pi/2) from Eq.3's prefactor
            // tau* in fp32 (log1pf: no fp64 table lookups; betap is stored in fp32)
            float alpha = alpha_in;
            alpha = alpha < 1e-4f ? 1e-4f : (alpha > 1.0f - 1e-4f ? 1.0f - 1e-4f : alpha);
            const float tau_star = -log1pf(-alpha);
            const float trA = is[0] * is[0] + is[1] * is[1] + is[2] * is[2];
            // beta * sqrt(pi/2) for the chosen alpha -> beta mapping (ablation B)
            float betap;
            if (absorption == DGSM_ABS_SIMPLE) betap = kappa_f * tau_star * 1.2533141373155003f;  // sqrt(pi/2)
            else if (absorption == DGSM_ABS_TRACEAVG) betap = kappa_f * tau_star * sqrtf(trA / 3.0f) * 0.5f;
            else betap = kappa_f * tau_star * (is[0] * is[1] * is[2]) * (float)(1.0 / (4.0 * kPi));  // MASS, DIAG
            rec.betap = betap;
            // negligible-pair cut (R8'): a pair contributes at most 2 pref <=
            // 2 betap s_max exp(-r/2) to any tau_k (1/sqrt(a) <= s_max); it is skipped
            // when that bound is < 2^-32, i.e. r > r_cut, never above 180 (beyond which
            // exp(-r/2) is exactly 0 in fp32).  fp32.
            {
                const float smax = fmaxf(sc0, fmaxf(sc1, sc2));
                const float rcut = fminf(2.0f * logf(2.0f * rec.betap * smax) + 44.3614195558365f, 180.0f);
                rec.rcut_D2 = rcut / (Df * Df);
                // Shell bounds of the writes of any live pair (r <= r_cut): its window
                // shells and step row lie where the ray is within Mahalanobis radius
                // rho = sqrt(r + 2 * 3.92^2) of mu (|x_k| < 3.92 in the window; +1 for the
                // rounding of the fp32 live test), i.e. at points mu + y with y^T A y <= rho^2.
                // Their distance t = |mu + y| from the light satisfies
                //   t >= D + y.d >= D - rho s_d,   s_d^2 = d^T Sigma d = sum_j s_j^2 w_j^2,
                //   t <= D + rho s_d + (rho s_max)^2 / (2 (D - rho s_d))   (|y_perp| <= rho s_max)
                // (t <= D + rho s_max when D <= rho s_d).  Shell k is at t_k = (k + 1/2) dt;
                // the kernel's window bounds are ceil((s* -+ xsh)/dt - 1/2) (+1 on a rounding
                // tie): 0.01 shell of slack for its fp32 arithmetic, one more row above.
                // Computed in fp32 (a conservative bound, not part of the binning
                // contract): 0.02 shell of slack more for its own rounding (~1e-4 shell).
                const float rho = sqrtf(fmaxf(rcut, 0.0f) + 31.7312f);
                const float wf0 = (float)w[0], wf1 = (float)w[1], wf2 = (float)w[2];
                const float s_d = sqrtf((sc0 * sc0) * (wf0 * wf0) + (sc1 * sc1) * (wf1 * wf1) + (sc2 * sc2) * (wf2 * wf2));
                const float rs = rho * smax, near = Df - rho * s_d;
                const float t_hi = near > 0.25f * Df ? Df + rho * s_d + rs * rs / (2.0f * near) : Df + rs;
                const float idt = (float)K / L.w;
                float klo = floorf(near * idt - 0.53f), khi = ceilf(t_hi * idt - 0.47f) + 1.0f;
                klo = klo < 0.0f ? 0.0f : (klo > K - 1.0f ? K - 1.0f : klo);
                khi = khi < klo ? klo : (khi > (float)K ? (float)K : khi);
                rec.shells = (uint32_t)klo | ((uint32_t)khi << 16);
            }
            dbits = __float_as_uint(Df);
        }
    }
    if (active) {
        counts[oi] = tcnt;
        recs[oi] = rec;
        dup[oi] = make_uint4(dbits, (uint32_t)(uint16_t)rc0 | ((uint32_t)(uint16_t)rc1 << 16),
                              (uint32_t)(uint16_t)rr0 | ((uint32_t)(uint16_t)rr1 << 16), tcnt);
    }
    // per-light min/max of the depth key over binned Gaussians: warp reductions
    // (no CTA barrier), a global atomic only when it would change the value
    // (the running extremes settle after a few warps)
    const uint32_t peers = __match_any_sync(0xffffffffu, l);  // lanes of the same light
    const uint32_t dmin = __reduce_min_sync(peers, tcnt > 0 ? dbits : 0xffffffffu);
    const uint32_t dmax = __reduce_max_sync(peers, tcnt > 0 ? dbits : 0u);
    if ((threadIdx.x & 31) == __ffs(peers) - 1 && dmax != 0u) {
        volatile uint32_t* vmin = &stats->depth_min[l];
        volatile uint32_t* vmax = &stats->depth_max[l];
        if (dmin < *vmin) atomicMin(&stats->depth_min[l], dmin);
        if (dmax > *vmax) atomicMax(&stats->depth_max[l], dmax);
    }
}

__global__ void k_init_stats(PlanStats* stats) {
    pdl_begin();
    int t = threadIdx.x;
    if (t < DGSM_MAX_LIGHTS) { stats->depth_min[t] = 0xffffffffu; stats->depth_max[t] = 0u; }
    if (t <= DGSM_MAX_LIGHTS) stats->light_key_begin[t] = 0ull;  // k_light_begin adds the totals
    if (t == 0) { stats->n_invalid = 0u; stats->first_invalid = 0xffffffffu; }
}
}  // namespace

void launch_project_init(PlanStats* stats, cudaStream_t s) {
    pdl_launch(k_init_stats, 1, DGSM_MAX_LIGHTS + 1, 0, s, stats);
}

void launch_project(const dgsm_gaussians_t& g, const LightsParam& lp, int n_lights, int res, int K,
                    const dgsm_build_opts_t& o, int64_t i0, int64_t cnt, PairRec* recs, uint32_t* counts,
                    uint4* dup, PlanStats* stats, cudaStream_t s) {
    const int64_t total = (int64_t)n_lights * cnt;
    if (total == 0) return;
    const int bs = 256;
    const int64_t grid = (total + bs - 1) / bs;
    pdl_launch(k_project, (unsigned)grid, bs, 0, s, g.means, g.scales, g.rotations, g.opacities, g.n, i0, cnt, lp,
                                            n_lights, res, K, (double)o.kappa, (double)o.k_sigma,
                                            (double)o.rho_scale * (double)(2 * res) / (2.0 * kPi), o.bin_mode,
                                            o.absorption, (o.flags & DGSM_NO_TILE_CULL) != 0,
                                            (o.flags & DGSM_VALIDATE) != 0,
                                            slab_mask_ptr(o.slab), recs, counts, dup,
                                            stats);
}

}  // namespace dgsm
