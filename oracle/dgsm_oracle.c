/*
 * dgsm_oracle.c — plain, slow, double-precision CPU oracle for the DGSM build
 * and query of arXiv 2601.01660 ("Deep Gaussian Shadow Maps").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header or constant table with the CUDA path under
 * paper_2601_01660_b200/csrc/ and must never be called by the product path.
 *
 * Every function cites the PAPER.md passage ("P:L<line>", section/equation)
 * it follows; where the paper is silent the DESIGN.md reading ("Q<n>") is
 * named.  Built with  gcc -O2 -ffp-contract=off  (no FMA contraction, strict
 * IEEE double) so that the integer binning decisions (R4-R7) are reproducible
 * bit for bit by any implementation that performs the same IEEE operations in
 * the same order.
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (SPEC/paper values, closed forms, quadrature, brute force); the culled-vs-
 * unculled gap is pinned only against our own unculled mode ("parity
 * unpinned against the paper": the paper prints no atlas values).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_PI 3.141592653589793

/* ------------------------------------------------------------------ */
/* R2  rotation and precision matrix ("precision A_i = Sigma_i^-1";   */
/*     Sigma = R diag(s^2) R^T, 3DGS quaternion convention w,x,y,z)          */
/* ------------------------------------------------------------------ */
static void or_rotation(const float q4[4], double R[3][3])
{
    double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    double inv = 1.0 / sqrt(((w * w + x * x) + y * y) + z * z);  /* binning contract v2: one division */
    w = w * inv; x = x * inv; y = y * inv; z = z * inv;
    R[0][0] = 1.0 - 2.0 * (y * y + z * z);
    R[0][1] = 2.0 * (x * y - w * z);
    R[0][2] = 2.0 * (x * z + w * y);
    R[1][0] = 2.0 * (x * y + w * z);
    R[1][1] = 1.0 - 2.0 * (x * x + z * z);
    R[1][2] = 2.0 * (y * z - w * x);
    R[2][0] = 2.0 * (x * z - w * y);
    R[2][1] = 2.0 * (y * z + w * x);
    R[2][2] = 1.0 - 2.0 * (x * x + y * y);
}

/* A = R diag(s^-2) R^T */
static void or_precision(const float s3[3], const float q4[4], double A[3][3])
{
    double R[3][3];
    or_rotation(q4, R);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j)
                acc += R[r][j] * (1.0 / ((double)s3[j] * (double)s3[j])) * R[c][j];
            A[r][c] = acc;
        }
}

/* Opacity clamp (Q16): alpha' = min(max(alpha,1e-4),1-1e-4). */
static double or_alpha_clamped(float alpha)
{
    double a = alpha;
    if (a < 1e-4) a = 1e-4;
    if (a > 1.0 - 1e-4) a = 1.0 - 1e-4;
    return a;
}

/* Eq.5 (TraceAvg): beta = kappa * tau* * sqrt(tr(A)/3)/sqrt(2 pi),
 * tau* = -ln(1 - alpha). */
double or_beta(const float s3[3], const float q4[4], float alpha, double kappa)
{
    double A[3][3];
    or_precision(s3, q4, A);
    double trA = A[0][0] + A[1][1] + A[2][2];
    double tau_star = -log1p(-or_alpha_clamped(alpha));
    return kappa * tau_star * sqrt(trA / 3.0) / sqrt(2.0 * OR_PI);
}

/* Ablation B alpha -> beta mappings, tau* = -ln(1 - alpha):
 *   0 TraceAvg  beta = kappa tau* sqrt(tr(A)/3) / sqrt(2 pi)       (Eq.5, the default)
 *   1 Simple    beta = kappa tau*                                   (mapping 1)
 *   2 Mass      beta = kappa tau* / ((2 pi)^{3/2} sqrt(det Sigma))  (mapping 3, unit-mass
 *               reading of the garbled "A is the covariance", Q14)
 *   3 Diag      beta = kappa tau* / ((2 pi)^{3/2} s_x s_y s_z)      (mapping 4)
 * Mass and Diag coincide for Sigma = R diag(s^2) R^T; both are kept because
 * the paper lists both. */
double or_beta_mode(const float s3[3], const float q4[4], float alpha, double kappa, int mode)
{
    double tau_star = -log1p(-or_alpha_clamped(alpha));
    if (mode == 0) return or_beta(s3, q4, alpha, kappa);
    if (mode == 1) return kappa * tau_star;
    double two_pi_32 = pow(2.0 * OR_PI, 1.5);
    if (mode == 2) {
        /* det Sigma from the explicit covariance R diag(s^2) R^T */
        double R[3][3], S[3][3];
        or_rotation(q4, R);
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j)
                    acc += R[r][j] * ((double)s3[j] * (double)s3[j]) * R[c][j];
                S[r][c] = acc;
            }
        double det = S[0][0] * (S[1][1] * S[2][2] - S[1][2] * S[2][1]) -
                     S[0][1] * (S[1][0] * S[2][2] - S[1][2] * S[2][0]) +
                     S[0][2] * (S[1][0] * S[2][1] - S[1][1] * S[2][0]);
        return kappa * tau_star / (two_pi_32 * sqrt(det));
    }
    return kappa * tau_star / (two_pi_32 * ((double)s3[0] * (double)s3[1] * (double)s3[2]));
}

/* ------------------------------------------------------------------ */
/* Octahedral map psi                                      */
/* ------------------------------------------------------------------ */
static double or_sgn(double x) { return x >= 0.0 ? 1.0 : -1.0; } /* sgn(0)=+1 (Q4) */

/* encode: q = d/(|x|+|y|+|z|); fold for q_z < 0.  Accepts any
 * non-zero vector (the normalisation by the 1-norm makes |d| irrelevant). */
void or_oct_encode(const double d[3], double uv[2])
{
    double n1 = (fabs(d[0]) + fabs(d[1])) + fabs(d[2]);
    double qx = d[0] / n1, qy = d[1] / n1, qz = d[2] / n1;
    if (qz >= 0.0) {
        uv[0] = qx;
        uv[1] = qy;
    } else {
        uv[0] = or_sgn(qx) * (1.0 - fabs(qy));
        uv[1] = or_sgn(qy) * (1.0 - fabs(qx));
    }
}

/* decode: z = 1-|u|-|v|; undo the fold; normalise. */
void or_oct_decode(double u, double v, double d[3])
{
    double x = u, y = v, z = 1.0 - fabs(u) - fabs(v);
    if (z < 0.0) {
        x = or_sgn(u) * (1.0 - fabs(v));
        y = or_sgn(v) * (1.0 - fabs(u));
    }
    double nrm = sqrt(x * x + y * y + z * z);
    d[0] = x / nrm; d[1] = y / nrm; d[2] = z / nrm;
}

/* Texel centre direction ("pixel centers"; Q3: u<->col, v<->row,
 * u_c = (col+0.5)*2/W - 1). */
void or_texel_dir(int row, int col, int H, int W, double d[3])
{
    double u = (col + 0.5) * 2.0 / W - 1.0;
    double v = (row + 0.5) * 2.0 / H - 1.0;
    or_oct_decode(u, v, d);
}

/* Radial bin centre t_k = (k + 1/2) t_max / K. */
double or_bin_center(int k, int K, double t_max) { return (k + 0.5) * t_max / K; }

/* ------------------------------------------------------------------ */
/* R4-R5  light-space footprint                            */
/* Output: fp[0]=D, fp[1]=px, fp[2]=py, fp[3]=p1, fp[4]=lambda1;         */
/*         rect[0..3] = c0,c1,r0,r1 (unclamped integer texel range).     */
/* Returns 0 when the Gaussian is excluded (D <= 1e-6, Q17), else 1.      */
/* The eigenvalue uses the basis-free form of Sigma_perp (Q7/R5):         */
/*   tr_perp = sum s_j^2 (1 - w_j^2),  det_perp = sum_j w_j^2 prod_{i!=j} s_i^2, */
/*   w = R^T (m/D); lambda1 = tr/2 + sqrt(max(tr^2/4 - det, 0)).          */
/* ------------------------------------------------------------------ */
int or_footprint(const float mu[3], const float s3[3], const float q4[4],
                 const float o[3], int res, double k_sigma, double rho_scale,
                 double fp[5], int64_t rect[4])
{
    int H = res, W = res;
    double mx = (double)mu[0] - (double)o[0];
    double my = (double)mu[1] - (double)o[1];
    double mz = (double)mu[2] - (double)o[2];
    double D = sqrt((mx * mx + my * my) + mz * mz);
    if (!(D > 1e-6)) return 0;

    /* psi(m) with one division: q = m * (1/|m|_1) (contract v2) */
    double inv1 = 1.0 / ((fabs(mx) + fabs(my)) + fabs(mz));
    double qx = mx * inv1, qy = my * inv1, qz = mz * inv1, u, v;
    if (qz >= 0.0) { u = qx; v = qy; }
    else { u = or_sgn(qx) * (1.0 - fabs(qy)); v = or_sgn(qy) * (1.0 - fabs(qx)); }
    double px = (u + 1.0) * (0.5 * W) - 0.5;
    double py = (v + 1.0) * (0.5 * H) - 0.5;

    double R[3][3];
    or_rotation(q4, R);
    double invD = 1.0 / D;
    double dx = mx * invD, dy = my * invD, dz = mz * invD;
    double w[3], s2[3];
    for (int j = 0; j < 3; ++j) {
        w[j] = (R[0][j] * dx + R[1][j] * dy) + R[2][j] * dz;
        s2[j] = (double)s3[j] * (double)s3[j];
    }
    double tr = (s2[0] * (1.0 - w[0] * w[0]) + s2[1] * (1.0 - w[1] * w[1])) +
                s2[2] * (1.0 - w[2] * w[2]);
    /* det_perp = prod s^2 * sum w_j^2/s_j^2, written without divisions */
    double det = ((s2[1] * s2[2]) * (w[0] * w[0]) + (s2[0] * s2[2]) * (w[1] * w[1])) +
                 (s2[0] * s2[1]) * (w[2] * w[2]);
    double disc = (tr * tr) * 0.25 - det;
    if (disc < 0.0) disc = 0.0;
    double lam1 = tr * 0.5 + sqrt(disc);
    double rho = (rho_scale * (double)(H + W)) / (2.0 * OR_PI); /* P:L172, Q5 */
    double p1 = ((k_sigma * sqrt(lam1)) * invD) * rho;

    fp[0] = D; fp[1] = px; fp[2] = py; fp[3] = p1; fp[4] = lam1;
    double c0 = ceil(px - p1), c1 = floor(px + p1);
    double r0 = ceil(py - p1), r1 = floor(py + p1);
    /* clamp to the extended lattice [-W, 2W-1] in double before the cast (R6);
     * px, py lie in [-0.5, W-0.5] so only these two sides can overflow. */
    if (c0 < -(double)W) c0 = -(double)W;
    if (c1 > 2.0 * W - 1.0) c1 = 2.0 * W - 1.0;
    if (r0 < -(double)H) r0 = -(double)H;
    if (r1 > 2.0 * H - 1.0) r1 = 2.0 * H - 1.0;
    rect[0] = (int64_t)c0; rect[1] = (int64_t)c1;
    rect[2] = (int64_t)r0; rect[3] = (int64_t)r1;
    return 1;
}

/* Mirror-wrap of an extended-lattice texel centre onto the atlas (R10/Q8,
 * SPEC S:L286): a column outside [0,W-1] reflects and flips the row; then a
 * row outside [0,H-1] reflects and flips the column. */
void or_mirror_wrap(int64_t col, int64_t row, int H, int W, int64_t out[2])
{
    if (col < 0) { col = -1 - col; row = H - 1 - row; }
    else if (col > W - 1) { col = 2 * (int64_t)W - 1 - col; row = H - 1 - row; }
    if (row < 0) { row = -1 - row; col = W - 1 - col; }
    else if (row > H - 1) { row = 2 * (int64_t)H - 1 - row; col = W - 1 - col; }
    out[0] = col; out[1] = row;
}

/* ------------------------------------------------------------------ */
/* R6-R7  binning into 8x8 tiles and the (light, tile, depth)   */
/* key order (Q10).                                                       */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t light, tile, depth_bits, index;
} or_entry;

static int or_entry_cmp(const void* pa, const void* pb)
{
    const or_entry* a = (const or_entry*)pa;
    const or_entry* b = (const or_entry*)pb;
    if (a->light != b->light) return a->light < b->light ? -1 : 1;
    if (a->tile != b->tile) return a->tile < b->tile ? -1 : 1;
    if (a->depth_bits != b->depth_bits) return a->depth_bits < b->depth_bits ? -1 : 1;
    if (a->index != b->index) return a->index < b->index ? -1 : 1;
    return 0;
}

static uint32_t or_float_bits(double D)
{
    float f = (float)D;
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

/* Tile set of one (light, Gaussian): every integer texel centre inside the
 * closed square [px-p1,px+p1]x[py-p1,py+p1] (clamped to the extended lattice)
 * is mapped (wrap: mirror-wrap; clamp: dropped if outside) and every tile
 * containing a mapped centre is listed once in `list` (the first time it is
 * seen; `mark` is the per-tile "already listed" flag, n_tiles bytes, all 0 on
 * entry and on return).  Returns the number of distinct tiles. */
static int64_t or_tile_set(const int64_t rect[4], int res, int bin_mode, unsigned char* mark,
                           int64_t* list)
{
    int H = res, W = res, TW = res / 8;
    int64_t n = 0;
    for (int64_t row = rect[2]; row <= rect[3]; ++row)
        for (int64_t col = rect[0]; col <= rect[1]; ++col) {
            int64_t cr[2];
            if (bin_mode == 1) { /* clamp (3DGS getRect) */
                if (col < 0 || col > W - 1 || row < 0 || row > H - 1) continue;
                cr[0] = col; cr[1] = row;
            } else {
                or_mirror_wrap(col, row, H, W, cr);
            }
            int64_t t = (cr[1] >> 3) * TW + (cr[0] >> 3);
            if (!mark[t]) { mark[t] = 1; list[n++] = t; }
        }
    for (int64_t j = 0; j < n; ++j) mark[list[j]] = 0;
    return n;
}

/* Bin every (light, Gaussian) and sort the entries by (light, tile, depth
 * bits, index) (R7); returns the malloc'd entries, *P_out = their number.
 * bin_mode: 0 = wrap (default), 1 = clamp. */
static or_entry* or_bin_sorted(const float* means, const float* scales, const float* rotations, int64_t n,
                               const float* light_pos /*[L][3]*/, int L, int res, double k_sigma,
                               double rho_scale, int bin_mode, int64_t* P_out)
{
    int64_t n_tiles = (int64_t)(res / 8) * (res / 8);
    unsigned char* mark = (unsigned char*)calloc((size_t)n_tiles, 1);
    int64_t* list = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_tiles);
    int64_t P = 0, cap = 1024;
    or_entry* e = (or_entry*)malloc(sizeof(or_entry) * cap);
    for (int l = 0; l < L; ++l)
        for (int64_t i = 0; i < n; ++i) {
            double fp[5];
            int64_t rect[4];
            if (!or_footprint(means + 3 * i, scales + 3 * i, rotations + 4 * i, light_pos + 3 * l,
                              res, k_sigma, rho_scale, fp, rect))
                continue;
            if (rect[0] > rect[1] || rect[2] > rect[3]) continue;
            int64_t cnt = or_tile_set(rect, res, bin_mode, mark, list);
            uint32_t db = or_float_bits(fp[0]);
            for (int64_t j = 0; j < cnt; ++j) {
                if (P == cap) {
                    cap *= 2;
                    e = (or_entry*)realloc(e, sizeof(or_entry) * cap);
                }
                e[P].light = (uint32_t)l;
                e[P].tile = (uint32_t)list[j];
                e[P].depth_bits = db;
                e[P].index = (uint32_t)i;
                ++P;
            }
        }
    qsort(e, (size_t)P, sizeof(or_entry), or_entry_cmp);
    free(list);
    free(mark);
    *P_out = P;
    return e;
}

/* Bin every (light, Gaussian); returns P (number of entries).  When
 * `capacity` >= P the sorted entries are written to the four output arrays. */
int64_t or_bin(const float* means, const float* scales, const float* rotations, int64_t n,
               const float* light_pos /*[L][3]*/, int L, int res, double k_sigma,
               double rho_scale, int bin_mode, uint32_t* out_light, uint32_t* out_tile,
               uint32_t* out_depth, uint32_t* out_index, int64_t capacity)
{
    int64_t P = 0;
    or_entry* e = or_bin_sorted(means, scales, rotations, n, light_pos, L, res, k_sigma, rho_scale,
                                bin_mode, &P);
    if (capacity >= P && out_light) {
        for (int64_t j = 0; j < P; ++j) {
            out_light[j] = e[j].light;
            out_tile[j] = e[j].tile;
            out_depth[j] = e[j].depth_bits;
            out_index[j] = e[j].index;
        }
    }
    free(e);
    return P;
}

/* or_bin in two calls without binning twice: or_bin_start bins and sorts and
 * returns the entries (opaque) and P; or_bin_take copies them into the four
 * arrays (NULL arrays: discard) and frees them. */
void* or_bin_start(const float* means, const float* scales, const float* rotations, int64_t n,
                   const float* light_pos, int L, int res, double k_sigma, double rho_scale, int bin_mode,
                   int64_t* P_out)
{
    return or_bin_sorted(means, scales, rotations, n, light_pos, L, res, k_sigma, rho_scale, bin_mode, P_out);
}

void or_bin_take(void* h, int64_t P, uint32_t* out_light, uint32_t* out_tile, uint32_t* out_depth,
                 uint32_t* out_index)
{
    or_entry* e = (or_entry*)h;
    if (out_light)
        for (int64_t j = 0; j < P; ++j) {
            out_light[j] = e[j].light;
            out_tile[j] = e[j].tile;
            out_depth[j] = e[j].depth_bits;
            out_index[j] = e[j].index;
        }
    free(e);
}

/* ------------------------------------------------------------------ */
/* Eq.2-3: optical depth of one Gaussian along o + s d, s in [0,t] */
/* ------------------------------------------------------------------ */
void or_ray_quadratic(const double A[3][3], const double mu[3], const double o[3],
                      const double d[3], double abc[3])
{
    double om[3] = {o[0] - mu[0], o[1] - mu[1], o[2] - mu[2]}; /* o_L - mu_i */
    double Ad[3], Aom[3];
    for (int r = 0; r < 3; ++r) {
        Ad[r] = A[r][0] * d[0] + A[r][1] * d[1] + A[r][2] * d[2];
        Aom[r] = A[r][0] * om[0] + A[r][1] * om[1] + A[r][2] * om[2];
    }
    abc[0] = d[0] * Ad[0] + d[1] * Ad[1] + d[2] * Ad[2];        /* a = d^T A d */
    abc[1] = d[0] * Aom[0] + d[1] * Aom[1] + d[2] * Aom[2];     /* b = d^T A (o-mu) */
    abc[2] = om[0] * Aom[0] + om[1] * Aom[1] + om[2] * Aom[2];  /* c */
}

/* Eq.3: int_0^t exp(-1/2 (a s^2 + 2 b s + c)) ds, times beta. */
double or_segment_depth(double a, double b, double c, double beta, double t)
{
    double pref = sqrt(OR_PI / (2.0 * a)) * exp(-0.5 * (c - b * b / a));
    double h = sqrt(a / 2.0);
    return beta * pref * (erf(h * (t + b / a)) - erf(h * (b / a)));
}

/* ------------------------------------------------------------------ */
/* R8  the atlas  T[l][k][row][col] = exp(-tau(d(row,col), t_k))  (Eq.4) */
/* ------------------------------------------------------------------ */
typedef struct {
    const float *means, *scales, *rotations, *opacities;
    int64_t n;
    const float* light_pos; /* [L][3] */
    const float* t_max;     /* [L]    */
    int L, res, K;
    double kappa, k_sigma, rho_scale;
    int bin_mode, culled;
    int64_t tile_stride; /* compute only work items with (l*n_tiles+tile) % stride == 0 */
    /* derived */
    double* A;    /* [n][9] */
    double* beta; /* [n] */
    int64_t n_tiles;
    /* culled lists */
    const uint32_t* e_index;
    const int64_t* range; /* [L*n_tiles+1] start offsets into the sorted entries */
    unsigned char* excluded; /* [L][n] */
    double* T;               /* [L][K][res][res] */
    const unsigned char* slab_mask; /* [L][res][res] or NULL: the ROI pixel set P */
    const int32_t* slab_krange;     /* [L][2] k_min, k_max (k_min > k_max: empty) */
    const int64_t* items;    /* or_build_tiles: the (light, tile) items to compute, or NULL (all) */
    int64_t n_items_list;
    double* T_items;         /* or_build_tiles output [n_items_list][K][8][8] */
    int64_t next;            /* work counter */
    int64_t evals;           /* (texel, Gaussian) evaluations performed */
    pthread_mutex_t lock;
} or_build_ctx;

/* T value of texel (row, col), shell k of work item `item` (list position q):
 * the atlas [L][K][H][W], or the compact [q][K][8][8] of or_build_tiles. */
static double* or_T_at(or_build_ctx* c, int64_t q, int l, int k, int row, int col)
{
    if (c->T_items) return c->T_items + ((q * c->K + k) * 8 + (row & 7)) * 8 + (col & 7);
    return c->T + (((int64_t)l * c->K + k) * c->res + row) * c->res + col;
}

static void or_build_item(or_build_ctx* c, int64_t item, int64_t q)
{
    int l = (int)(item / c->n_tiles);
    int64_t tile = item % c->n_tiles;
    int TW = c->res / 8, H = c->res, W = c->res, K = c->K;
    int ty = (int)(tile / TW), tx = (int)(tile % TW);
    double o[3] = {c->light_pos[3 * l], c->light_pos[3 * l + 1], c->light_pos[3 * l + 2]};
    double tmax = c->t_max[l];
    double* tau = (double*)malloc(sizeof(double) * K);
    for (int r = 0; r < 8; ++r)
        for (int cc = 0; cc < 8; ++cc) {
            int row = ty * 8 + r, col = tx * 8 + cc;
            int klo = 0, khi = K - 1;
            if (c->slab_mask) {
                /* "initialize T = 1 and only accumulate optical depth on the voxel
                 * slab R = P x {k_min..k_max}" */
                klo = c->slab_krange[2 * l];
                khi = c->slab_krange[2 * l + 1];
                if (!c->slab_mask[((int64_t)l * H + row) * W + col]) khi = -1;
                for (int k = 0; k < K; ++k)
                    if (k < klo || k > khi) *or_T_at(c, q, l, k, row, col) = 1.0;
                if (klo > khi) continue;
            }
            double d[3];
            or_texel_dir(row, col, H, W, d);
            for (int k = 0; k < K; ++k) tau[k] = 0.0;
            int64_t j0, j1;
            if (c->culled) { j0 = c->range[item]; j1 = c->range[item + 1]; }
            else { j0 = 0; j1 = c->n; }
            for (int64_t j = j0; j < j1; ++j) {
                int64_t i = c->culled ? (int64_t)c->e_index[j] : j;
                if (!c->culled && c->excluded[(int64_t)l * c->n + i]) continue;
                double mu[3] = {c->means[3 * i], c->means[3 * i + 1], c->means[3 * i + 2]};
                double Ai[3][3];
                memcpy(Ai, c->A + 9 * i, sizeof(Ai));
                double abc[3];
                or_ray_quadratic(Ai, mu, o, d, abc);
                for (int k = klo; k <= khi; ++k)
                    tau[k] += or_segment_depth(abc[0], abc[1], abc[2], c->beta[i],
                                               or_bin_center(k, K, tmax));
            }
            for (int k = klo; k <= khi; ++k)
                *or_T_at(c, q, l, k, row, col) = exp(-tau[k]);
        }
    free(tau);
}

static void* or_build_worker(void* arg)
{
    or_build_ctx* c = (or_build_ctx*)arg;
    int64_t n_items = c->items ? c->n_items_list : (int64_t)c->L * c->n_tiles;
    for (;;) {
        pthread_mutex_lock(&c->lock);
        int64_t q = c->next;
        c->next += 1;
        pthread_mutex_unlock(&c->lock);
        while (!c->items && q < n_items && q % c->tile_stride != 0) {
            pthread_mutex_lock(&c->lock);
            q = c->next;
            c->next += 1;
            pthread_mutex_unlock(&c->lock);
        }
        if (q >= n_items) break;
        int64_t item = c->items ? c->items[q] : q;
        or_build_item(c, item, q);
        int64_t ev = 64 * (c->culled ? (c->range[item + 1] - c->range[item]) : c->n);
        pthread_mutex_lock(&c->lock);
        c->evals += ev;
        pthread_mutex_unlock(&c->lock);
    }
    return NULL;
}

/* Build the atlas.  T_out: [L][K][res][res] doubles; items skipped by
 * tile_stride are set to NaN.  culled=1 uses the R6 tile lists (the GPU
 * parity target), culled=0 sums every non-excluded Gaussian at every texel
 * (the reference for the culling error, P:L335 ablation D).  Returns P (the
 * number of binned entries) in culled mode, 0 otherwise, -1 on bad input. */
int64_t or_build_slab(const float* means, const float* scales, const float* rotations,
                      const float* opacities, int64_t n, const float* light_pos, const float* t_max,
                      int L, int res, int K, double kappa, double k_sigma, double rho_scale,
                      int bin_mode, int culled, int absorption, int64_t tile_stride, int n_threads,
                      const unsigned char* slab_mask, const int32_t* slab_krange,
                      double* T_out, int64_t* evals_out);

int64_t or_build(const float* means, const float* scales, const float* rotations,
                 const float* opacities, int64_t n, const float* light_pos, const float* t_max,
                 int L, int res, int K, double kappa, double k_sigma, double rho_scale,
                 int bin_mode, int culled, int absorption, int64_t tile_stride, int n_threads,
                 double* T_out, int64_t* evals_out /* nullable: (texel, Gaussian) evaluations performed */)
{
    return or_build_slab(means, scales, rotations, opacities, n, light_pos, t_max, L, res, K, kappa,
                         k_sigma, rho_scale, bin_mode, culled, absorption, tile_stride, n_threads,
                         NULL, NULL, T_out, evals_out);
}

/* The build (R8) over all work items (atlas output, `tile_stride` sampling)
 * or over a list of items (compact output).  Shared by or_build_slab and
 * or_build_tiles. */
static int64_t or_build_impl(or_build_ctx* cp, int absorption, int n_threads)
{
    or_build_ctx* c = cp;
    const float *means = c->means, *scales = c->scales, *rotations = c->rotations;
    int64_t n = c->n;
    int L = c->L, res = c->res;
    c->n_tiles = (int64_t)(res / 8) * (res / 8);
    c->A = (double*)malloc(sizeof(double) * 9 * (n > 0 ? n : 1));
    c->beta = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        double Ai[3][3];
        or_precision(scales + 3 * i, rotations + 4 * i, Ai);
        memcpy(c->A + 9 * i, Ai, sizeof(Ai));
        c->beta[i] = or_beta_mode(scales + 3 * i, rotations + 4 * i, c->opacities[i], c->kappa, absorption);
    }
    c->excluded = (unsigned char*)calloc((size_t)L * (n > 0 ? n : 1), 1);
    for (int l = 0; l < L; ++l)
        for (int64_t i = 0; i < n; ++i) {
            double fp[5];
            int64_t rect[4];
            c->excluded[(int64_t)l * n + i] =
                !or_footprint(means + 3 * i, scales + 3 * i, rotations + 4 * i, c->light_pos + 3 * l,
                              res, c->k_sigma, c->rho_scale, fp, rect);
        }

    int64_t P = 0;
    or_entry* e = NULL;
    uint32_t* ei = NULL;
    int64_t* range = NULL;
    if (c->culled) {
        e = or_bin_sorted(means, scales, rotations, n, c->light_pos, L, res, c->k_sigma, c->rho_scale,
                          c->bin_mode, &P);
        ei = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(P > 0 ? P : 1));
        for (int64_t j = 0; j < P; ++j) ei[j] = e[j].index;
        int64_t n_items = (int64_t)L * c->n_tiles;
        range = (int64_t*)malloc(sizeof(int64_t) * (n_items + 1));
        int64_t j = 0;
        for (int64_t it = 0; it <= n_items; ++it) {
            while (j < P && (int64_t)e[j].light * c->n_tiles + e[j].tile < it) ++j;
            range[it] = j;
        }
        c->e_index = ei; c->range = range;
    }

    if (n_threads < 1) n_threads = 1;
    pthread_mutex_init(&c->lock, NULL);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, or_build_worker, c);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&c->lock);
    free(th);

    free(c->A); free(c->beta); free(c->excluded);
    free(e); free(ei); free(range);
    return P;
}

static void or_build_ctx_init(or_build_ctx* c, const float* means, const float* scales,
                              const float* rotations, const float* opacities, int64_t n,
                              const float* light_pos, const float* t_max, int L, int res, int K,
                              double kappa, double k_sigma, double rho_scale, int bin_mode, int culled)
{
    memset(c, 0, sizeof(*c));
    c->means = means; c->scales = scales; c->rotations = rotations; c->opacities = opacities;
    c->n = n; c->light_pos = light_pos; c->t_max = t_max; c->L = L; c->res = res; c->K = K;
    c->kappa = kappa; c->k_sigma = k_sigma; c->rho_scale = rho_scale;
    c->bin_mode = bin_mode; c->culled = culled;
    c->tile_stride = 1;
}

/* As or_build, restricted to the ROI slab (slab_mask [L][res][res], slab_krange
 * [L][2] from or_active_slab); NULL slab_mask = the full atlas. */
int64_t or_build_slab(const float* means, const float* scales, const float* rotations,
                      const float* opacities, int64_t n, const float* light_pos, const float* t_max,
                      int L, int res, int K, double kappa, double k_sigma, double rho_scale,
                      int bin_mode, int culled, int absorption, int64_t tile_stride, int n_threads,
                      const unsigned char* slab_mask, const int32_t* slab_krange,
                      double* T_out, int64_t* evals_out)
{
    if (res < 8 || res % 8 != 0 || K < 1 || L < 1 || n < 0) return -1;
    or_build_ctx c;
    or_build_ctx_init(&c, means, scales, rotations, opacities, n, light_pos, t_max, L, res, K, kappa,
                      k_sigma, rho_scale, bin_mode, culled);
    c.tile_stride = tile_stride < 1 ? 1 : tile_stride;
    c.T = T_out;
    c.slab_mask = slab_mask;
    c.slab_krange = slab_krange;
    int64_t total = (int64_t)L * K * res * res;
    for (int64_t j = 0; j < total; ++j) T_out[j] = NAN;
    int64_t P = or_build_impl(&c, absorption, n_threads);
    if (evals_out) *evals_out = c.evals;
    return P;
}

/* As or_build (culled, full atlas semantics) for the listed work items only:
 * items[q] = l * (res/8)^2 + tile; T_items[q][K][8][8] receives T of the 64
 * texels (row-major within the tile) of item q.  For parity on a sample of
 * tiles of atlases too large to hold in double (2048^2 x 128 x 8 lights). */
int64_t or_build_tiles(const float* means, const float* scales, const float* rotations,
                       const float* opacities, int64_t n, const float* light_pos, const float* t_max,
                       int L, int res, int K, double kappa, double k_sigma, double rho_scale,
                       int bin_mode, int absorption, const int64_t* items, int64_t n_items,
                       int n_threads, double* T_items, int64_t* evals_out)
{
    if (res < 8 || res % 8 != 0 || K < 1 || L < 1 || n < 0 || n_items < 0) return -1;
    int64_t n_all = (int64_t)L * (res / 8) * (res / 8);
    for (int64_t q = 0; q < n_items; ++q)
        if (items[q] < 0 || items[q] >= n_all) return -1;
    or_build_ctx c;
    or_build_ctx_init(&c, means, scales, rotations, opacities, n, light_pos, t_max, L, res, K, kappa,
                      k_sigma, rho_scale, bin_mode, 1);
    c.items = items;
    c.n_items_list = n_items;
    c.T_items = T_items;
    int64_t P = or_build_impl(&c, absorption, n_threads);
    if (evals_out) *evals_out = c.evals;
    return P;
}

/* Optical depth tau(d, t) of the full mixture along one ray (Eq.2), every
 * non-excluded Gaussian, no culling.  Used by the pins (quadrature). */
double or_tau_ray(const float* means, const float* scales, const float* rotations,
                  const float* opacities, int64_t n, const double o[3], const double d_in[3],
                  double t, double kappa)
{
    double nd = sqrt(d_in[0] * d_in[0] + d_in[1] * d_in[1] + d_in[2] * d_in[2]);
    double d[3] = {d_in[0] / nd, d_in[1] / nd, d_in[2] / nd};
    double tau = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double A[3][3], abc[3];
        or_precision(scales + 3 * i, rotations + 4 * i, A);
        double mu[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
        or_ray_quadratic(A, mu, o, d, abc);
        tau += or_segment_depth(abc[0], abc[1], abc[2],
                                or_beta(scales + 3 * i, rotations + 4 * i, opacities[i], kappa), t);
    }
    return tau;
}

/* ------------------------------------------------------------------ */
/* R10-R12  query: trilinear sampling of the atlas at receiver centres   */
/* (P:L185-187), mirror-wrap taps (Q12), t clamped to [t_0, t_{K-1}],    */
/* product over lights (Q13), optional colour multiply.         */
/* ------------------------------------------------------------------ */
double or_sample(const double* atlas_l /* [K][res][res] */, int res, int K, const double o[3],
                 double t_max, const double x[3])
{
    int H = res, W = res;
    double m[3] = {x[0] - o[0], x[1] - o[1], x[2] - o[2]};
    double t = sqrt((m[0] * m[0] + m[1] * m[1]) + m[2] * m[2]);
    if (t == 0.0) return 1.0; /* Q18 */
    double uv[2];
    or_oct_encode(m, uv);
    double fx = (uv[0] + 1.0) * (0.5 * W) - 0.5;
    double fy = (uv[1] + 1.0) * (0.5 * H) - 0.5;
    double x0 = floor(fx), y0 = floor(fy);
    double wx = fx - x0, wy = fy - y0;
    double fk = (t * K) / t_max - 0.5;
    if (fk < 0.0) fk = 0.0;
    if (fk > K - 1) fk = K - 1;
    double k0 = floor(fk);
    double wk = fk - k0;
    int ik0 = (int)k0, ik1 = ik0 + 1 < K ? ik0 + 1 : K - 1;
    double acc = 0.0;
    for (int dk = 0; dk < 2; ++dk)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                int64_t cr[2];
                or_mirror_wrap((int64_t)x0 + dx, (int64_t)y0 + dy, H, W, cr);
                int k = dk ? ik1 : ik0;
                double w = (dx ? wx : 1.0 - wx) * (dy ? wy : 1.0 - wy) * (dk ? wk : 1.0 - wk);
                acc += w * atlas_l[((int64_t)k * H + cr[1]) * W + cr[0]];
            }
    return acc;
}

void or_query(const double* atlas /* [L][K][res][res] */, int L, int K, int res,
              const float* light_pos, const float* t_max, const float* positions, int64_t m,
              double* T_out, double* colors /* nullable [m][3], multiplied in place */)
{
    int64_t per_light = (int64_t)K * res * res;
    for (int64_t q = 0; q < m; ++q) {
        double x[3] = {positions[3 * q], positions[3 * q + 1], positions[3 * q + 2]};
        double T = 1.0;
        for (int l = 0; l < L; ++l) {
            double o[3] = {light_pos[3 * l], light_pos[3 * l + 1], light_pos[3 * l + 2]};
            T *= or_sample(atlas + l * per_light, res, K, o, t_max[l], x);
        }
        T_out[q] = T;
        if (colors) {
            colors[3 * q] *= T;
            colors[3 * q + 1] *= T;
            colors[3 * q + 2] *= T;
        }
    }
}

/* ------------------------------------------------------------------ */
/* NEXT-2: footprint-sampled query ("sampling a small footprint  */
/* around each Gaussian center and averaging deep-shadow lookups";       */
/* P:L308-317 ablation A: x_{g,i} = mu_g + R_g (s_g (.) z_i),            */
/* T_g = sum_i w_i T(x_{g,i}), sum_i w_i = 1).  Per light the footprint   */
/* average, then the product over lights (Q13).  The        */
/* offsets z_i and weights w_i are inputs (stencil or Monte Carlo draws). */
/* ------------------------------------------------------------------ */
void or_query_footprint(const double* atlas, int L, int K, int res, const float* light_pos,
                        const float* t_max, const float* means, const float* scales,
                        const float* rotations, int64_t m, const double* z /* [n][3] */,
                        const double* w /* [n] */, int n, double* T_out)
{
    int64_t per_light = (int64_t)K * res * res;
    for (int64_t g = 0; g < m; ++g) {
        double R[3][3];
        or_rotation(rotations + 4 * g, R);
        double T = 1.0;
        for (int l = 0; l < L; ++l) {
            double o[3] = {light_pos[3 * l], light_pos[3 * l + 1], light_pos[3 * l + 2]};
            double acc = 0.0;
            for (int i = 0; i < n; ++i) {
                double x[3];
                for (int r = 0; r < 3; ++r) {
                    x[r] = means[3 * g + r];
                    for (int c = 0; c < 3; ++c) x[r] += R[r][c] * ((double)scales[3 * g + c] * z[3 * i + c]);
                }
                acc += w[i] * or_sample(atlas + l * per_light, res, K, o, t_max[l], x);
            }
            T *= acc;
        }
        T_out[g] = T;
    }
}

/* ------------------------------------------------------------------ */
/* NEXT-1  receiver-driven ROI and active voxel slab        */
/* ------------------------------------------------------------------ */
/* Receivers x (float [m][3]) inside B = {x : ||(x - c)_xy||_inf <= R,
 * z_min <= x_z <= z_max} are projected per light into atlas pixels
 * (psi: the pixel whose cell holds u, col = floor((u+1) W/2),
 * clamped to W-1) and collected into the set P (mask[L][res][res] = 1); the
 * radial range is their bin floor(t K / t_max) (clamped to [0, K-1]) min/max
 * (P:L159).  Readings (DESIGN.md R-ROI): P is dilated by one pixel, each
 * neighbour mirror-wrapped like the sampler's taps (Q12), and the bin range
 * widened by one each side, so that every trilinear tap of a query
 * at a receiver in B lies in the slab.  A receiver at the light itself is
 * skipped (T = 1 there, Q18).  No receiver: k_min = K, k_max = -1.
 * roi = {c_x, c_y, c_z, R, z_min, z_max}.  Returns the receivers in B. */
int64_t or_active_slab(const float* x, int64_t m, const float* roi, const float* light_pos,
                       const float* t_max, int L, int res, int K, unsigned char* mask,
                       int32_t* krange)
{
    int H = res, W = res;
    memset(mask, 0, (size_t)L * H * W);
    for (int l = 0; l < L; ++l) { krange[2 * l] = K; krange[2 * l + 1] = -1; }
    int64_t inside = 0;
    for (int64_t q = 0; q < m; ++q) {
        double px = x[3 * q], py = x[3 * q + 1], pz = x[3 * q + 2];
        double ex = fabs(px - (double)roi[0]), ey = fabs(py - (double)roi[1]);
        double inf = ex > ey ? ex : ey;
        if (!(inf <= (double)roi[3] && pz >= (double)roi[4] && pz <= (double)roi[5])) continue;
        ++inside;
        for (int l = 0; l < L; ++l) {
            double d[3] = {px - (double)light_pos[3 * l], py - (double)light_pos[3 * l + 1],
                           pz - (double)light_pos[3 * l + 2]};
            double t = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
            if (t == 0.0) continue;
            double uv[2];
            or_oct_encode(d, uv);
            int64_t col = (int64_t)floor((uv[0] + 1.0) * (0.5 * W));
            int64_t row = (int64_t)floor((uv[1] + 1.0) * (0.5 * H));
            if (col > W - 1) col = W - 1;
            if (row > H - 1) row = H - 1;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int64_t cr[2];
                    or_mirror_wrap(col + dx, row + dy, H, W, cr);
                    mask[((int64_t)l * H + cr[1]) * W + cr[0]] = 1;
                }
            double fb = floor((t * K) / (double)t_max[l]);
            int b = fb > K - 1 ? K - 1 : (int)fb;
            int lo = b - 1 < 0 ? 0 : b - 1, hi = b + 1 > K - 1 ? K - 1 : b + 1;
            if (lo < krange[2 * l]) krange[2 * l] = lo;
            if (hi > krange[2 * l + 1]) krange[2 * l + 1] = hi;
        }
    }
    return inside;
}

/* ------------------------------------------------------------------ */
/* NEXT-4  SH lighting transfer (§3.5)             */
/* ------------------------------------------------------------------ */
/* Real spherical-harmonic basis up to degree d ("real spherical-
 * harmonic (SH) basis up to degree d", K = (d+1)^2), orthonormal on the
 * sphere, Condon-Shortley phase, index k = l^2 + l + m (m = -l..l):
 *   Y_l0 = K_l0 P_l^0(cos t),  Y_lm = sqrt2 K_lm P_l^m(cos t) cos(m p)  (m > 0),
 *   Y_l,-m = sqrt2 K_lm P_l^m(cos t) sin(m p),  K_lm = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!),
 * P_l^m by the textbook three-term recurrence (P_m^m = (-1)^m (2m-1)!! (1-z^2)^{m/2}).
 * DESIGN.md reading R-SH. */
void or_sh_basis(int d, const double dir[3], double* out)
{
    double x = dir[0], y = dir[1], z = dir[2];
    double r = sqrt((x * x + y * y) + z * z);
    x /= r; y /= r; z /= r;
    double phi = atan2(y, x);
    double st = sqrt(fmax(0.0, 1.0 - z * z));
    for (int m = 0; m <= d; ++m) {
        /* P_m^m */
        double pmm = 1.0;
        for (int i = 1; i <= m; ++i) pmm *= -(2.0 * i - 1.0) * st;
        double plm2 = 0.0, plm1 = pmm;
        for (int l = m; l <= d; ++l) {
            double p;
            if (l == m) p = pmm;
            else if (l == m + 1) p = z * (2.0 * m + 1.0) * pmm;
            else p = ((2.0 * l - 1.0) * z * plm1 - (double)(l + m - 1) * plm2) / (double)(l - m);
            if (l > m) { plm2 = plm1; plm1 = p; }
            /* K_lm */
            double ratio = 1.0; /* (l-m)!/(l+m)! */
            for (int i = l - m + 1; i <= l + m; ++i) ratio /= (double)i;
            double K = sqrt((2.0 * l + 1.0) / (4.0 * OR_PI) * ratio);
            if (m == 0) out[l * l + l] = K * p;
            else {
                out[l * l + l + m] = sqrt(2.0) * K * p * cos(m * phi);
                out[l * l + l - m] = sqrt(2.0) * K * p * sin(m * phi);
            }
        }
    }
}

/* Lat-long grid point j = i * n_phi + k ("latitude-longitude grid
 * {w_j} with quadrature weights w_j ~ sin theta_j"): theta_i = (i+1/2) pi/n_theta
 * from +z, phi_k = (k+1/2) 2 pi/n_phi, w = sin(theta) (pi/n_theta)(2 pi/n_phi)
 * (reading R-SH: the midpoint-rule weights, sum ~ 4 pi). */
void or_transfer_dir(int n_theta, int n_phi, int64_t j, double dir[3], double* w)
{
    int64_t i = j / n_phi, k = j % n_phi;
    double th = ((double)i + 0.5) * OR_PI / n_theta;
    double ph = ((double)k + 0.5) * 2.0 * OR_PI / n_phi;
    dir[0] = sin(th) * cos(ph);
    dir[1] = sin(th) * sin(ph);
    dir[2] = cos(th);
    *w = sin(th) * (OR_PI / n_theta) * (2.0 * OR_PI / n_phi);
}

/* Per-channel lighting scale and relit colour:
 *   L_c(w_j) = max(0, B(w_j) A_c)          (radiance from the fitted SH, Eq. before
 *                                           P:L209; negative ringing clamped: R-SH)
 *   S(w, n)  = max(0, <w, n>)^q            (S = 0 where <w,n> <= 0)
 *   s_c(n)   = clip_[0, s_max]( sum_j w_j L_c S / (sum_j w_j S + eps) )
 *   c'       = max(0, gamma c (.) s(n))
 * sh: [3][K] coefficients; normals, colors: [n][3] (colors nullable);
 * scales_out [n][3], colors_out [n][3] (nullable). */
void or_sh_transfer(const double* sh, int d, int n_theta, int n_phi, double q, double eps, double s_max,
                    double gamma, const double* normals, const double* colors, int64_t n, double* scales_out,
                    double* colors_out)
{
    int K = (d + 1) * (d + 1);
    int64_t M = (int64_t)n_theta * n_phi;
    double* B = (double*)malloc(sizeof(double) * (size_t)K);
    double* L = (double*)malloc(sizeof(double) * 3 * (size_t)M);
    double* W = (double*)malloc(sizeof(double) * (size_t)M);
    double* Dir = (double*)malloc(sizeof(double) * 3 * (size_t)M);
    for (int64_t j = 0; j < M; ++j) {
        or_transfer_dir(n_theta, n_phi, j, Dir + 3 * j, W + j);
        or_sh_basis(d, Dir + 3 * j, B);
        for (int c = 0; c < 3; ++c) {
            double v = 0.0;
            for (int k = 0; k < K; ++k) v += B[k] * sh[c * K + k];
            L[3 * j + c] = v > 0.0 ? v : 0.0;
        }
    }
    for (int64_t g = 0; g < n; ++g) {
        const double* nn = normals + 3 * g;
        double num[3] = {0.0, 0.0, 0.0}, den = 0.0;
        for (int64_t j = 0; j < M; ++j) {
            double dt = nn[0] * Dir[3 * j] + nn[1] * Dir[3 * j + 1] + nn[2] * Dir[3 * j + 2];
            if (dt <= 0.0) continue;
            double S = pow(dt, q);
            den += W[j] * S;
            for (int c = 0; c < 3; ++c) num[c] += W[j] * L[3 * j + c] * S;
        }
        for (int c = 0; c < 3; ++c) {
            double s = num[c] / (den + eps);
            if (s < 0.0) s = 0.0;
            if (s > s_max) s = s_max;
            if (scales_out) scales_out[3 * g + c] = s;
            if (colors_out && colors) {
                double v = gamma * colors[3 * g + c] * s;
                colors_out[3 * g + c] = v > 0.0 ? v : 0.0;
            }
        }
    }
    free(B); free(L); free(W); free(Dir);
}
