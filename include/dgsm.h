/*
 * dgsm.h — C ABI of libdgsm.so, the B200-native (sm_100a) Deep Gaussian Shadow
 * Map build + query of arXiv 2601.01660.
 *
 * Citations "P:L<n>" are PAPER.md lines (§3.2 build, §3.3 sampling);
 * "Q<n>"/"R<n>" are the readings listed in DESIGN.md.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Device pointers are CUDA global-memory addresses in the caller's current
 *    context; host pointers are plain process memory.  Every buffer is
 *    caller-owned: the library never allocates or frees device memory and keeps
 *    no pointer after the call's stream work has completed.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All work is enqueued on it; only dgsm_build_plan synchronises it (once, to
 *    read the key count P back to the host).
 *  - Functions are re-entrant; concurrent calls on different streams need
 *    different workspaces.
 *  - Return value: DGSM_OK (0) or a positive DGSM_E* code; dgsm_last_error()
 *    returns a thread-local message for the last failure on this thread.
 *    Arguments are validated before any work is enqueued.  A CUDA launch or
 *    runtime error yields DGSM_ECUDA (the stream may then hold partial work).
 *    Data errors (non-finite values, scales <= 0, a zero quaternion: P:L86
 *    needs an SPD Sigma and alpha in (0,1)) are checked on the device with the
 *    DGSM_VALIDATE build flag (dgsm_build_plan then returns DGSM_EDATA; a
 *    sync-free build reports them in its status word); without it the results
 *    for such Gaussians are unspecified.  Opacities outside [1e-4, 1-1e-4] are
 *    clamped (Q16), not rejected.
 */
#ifndef DGSM_H
#define DGSM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define DGSM_OK 0
#define DGSM_EINVAL 1   /* null pointer, n<0, atlas_res%8!=0 or <8 or >2048, n_shells<1 or >DGSM_MAX_SHELLS,
                           n_lights outside [1, DGSM_MAX_LIGHTS], t_max<=0, bad opts, plan/run mismatch */
#define DGSM_ENOSPC 2   /* workspace smaller than required (required size is returned) */
#define DGSM_ECUDA 3    /* CUDA launch/runtime error */
#define DGSM_ERANGE 4   /* problem too large: n >= 2^30 Gaussians or >= 2^30 keys in total */
#define DGSM_EDATA 5    /* DGSM_VALIDATE found invalid Gaussians (see the message) */

#define DGSM_MAX_LIGHTS 64
#define DGSM_MAX_SHELLS 256
#define DGSM_MAX_FOOTPRINT_SAMPLES 64

/* ---- binning mode (R6, Q8) ---------------------------------------------- */
#define DGSM_BIN_WRAP 0   /* default: footprints crossing the atlas border are mirror-wrapped
                             onto the octahedral neighbours (the seam rule of the query, Q12) */
#define DGSM_BIN_CLAMP 1  /* 3DGS getRect semantics: the square is intersected with the grid */

/* ---- build flags --------------------------------------------------------- */
#define DGSM_OUTPUT_TAU 1u /* write optical depth tau (Eq.2) instead of T = exp(-tau) (Eq.4);
                              used by Gaussian-sharded multi-GPU builds before the reduce-scatter */
#define DGSM_COLLECT_STATS 2u /* count the accumulation work into the run workspace (read it with
                                 dgsm_build_stats); instrumented kernel variant, for roofline accounting */
#define DGSM_NO_TILE_CULL 4u  /* ablation D: bin every non-excluded Gaussian into every
                                 tile (no light-space culling); P = L * n * (res/8)^2 keys */
#define DGSM_VALIDATE 8u      /* check every Gaussian on the device: finite mean, finite scales > 0,
                                 finite non-zero quaternion, finite opacity (SPD Sigma) */

/* Work counted by a DGSM_COLLECT_STATS build. */
typedef struct dgsm_build_stats {
    uint64_t pairs;         /* (texel, listed Gaussian) evaluations = 64 * P */
    uint64_t pairs_live;    /* pairs whose Eq.3 prefactor is non-zero in fp32 (r <= 180, x0 < 3.92) */
    uint64_t window_shells; /* shells evaluated with an erf (|x_k| < 3.92) */
    uint64_t steps;         /* saturated tails added as one step */
    uint64_t warp_records;  /* (warp, listed Gaussian) iterations = 2 * P (two warps per tile) */
    uint64_t warp_live_any; /* of those, with at least one live lane (the warp runs the live path) */
    uint64_t warp_live_max; /* sum over (warp, stage) of the max live count of one lane */
    uint64_t band_records;  /* records run through the pair tests, summed over the shell bands
                               (K > 64: a record meeting two bands counts twice; else = P) */
} dgsm_build_stats_t;

/* Occluder Gaussians, structure of arrays, DEVICE pointers (mean mu_i,
 * covariance Sigma_i = R diag(s^2) R^T, precision A_i = Sigma_i^-1, opacity alpha_i). */
typedef struct dgsm_gaussians {
    const float* means;     /* [n][3] world metres */
    const float* scales;    /* [n][3] per-axis standard deviations s (activated, > 0) */
    const float* rotations; /* [n][4] quaternion (w, x, y, z), any norm > 0 (normalised in fp64) */
    const float* opacities; /* [n] alpha in (0,1), clamped to [1e-4, 1-1e-4] */
    int64_t n;              /* number of Gaussians, >= 0 (n = 0 gives T == 1 exactly) */
} dgsm_gaussians_t;

/* Point light o_L and the radial range of its atlas: shells
 * t_k = (k + 1/2) t_max / K.  HOST memory. */
typedef struct dgsm_light {
    float position[3]; /* o_L, world metres */
    float t_max;       /* > 0, metres (Q2) */
} dgsm_light_t;

/* Build options.  dgsm_default_opts() gives the paper's setting. */
typedef struct dgsm_build_opts {
    float kappa;       /* Eq.5 global strength knob, default 1 (Q15); > 0 */
    float k_sigma;     /* footprint k_sigma rule, default 3 (Q6); > 0 */
    float rho_scale;   /* multiplies rho = (H+W)/(2 pi) pixels per radian, default 1 (Q5); > 0 */
    int32_t bin_mode;  /* DGSM_BIN_WRAP (default) or DGSM_BIN_CLAMP */
    uint32_t flags;    /* DGSM_OUTPUT_TAU | DGSM_COLLECT_STATS | DGSM_NO_TILE_CULL | DGSM_VALIDATE, or 0 */
    int32_t absorption; /* DGSM_ABS_* alpha -> beta mapping (ablation B), default TRACEAVG */
    const void* slab;   /* NULL (default): the full atlas.  Else a device slab written by
                           dgsm_active_slab for the same n_lights, atlas_res and n_shells: only
                           the voxel slab R = P x {k_min..k_max} is accumulated and T = 1 (tau = 0
                           with DGSM_OUTPUT_TAU) everywhere else; tiles without a
                           texel of P are not binned at all.  8-B aligned, read-only; like the
                           Gaussian arrays it must not change between dgsm_build_plan and
                           dgsm_build_run and must stay valid until the run has completed. */
} dgsm_build_opts_t;

/* ---- alpha -> beta mappings, tau* = -ln(1 - alpha) ----------- */
#define DGSM_ABS_TRACEAVG 0 /* kappa tau* sqrt(tr A / 3) / sqrt(2 pi)       (Eq.5, default)      */
#define DGSM_ABS_SIMPLE 1   /* kappa tau*                                   (mapping 1)          */
#define DGSM_ABS_MASS 2     /* kappa tau* / ((2 pi)^{3/2} sqrt(det Sigma))  (mapping 3, Q14)     */
#define DGSM_ABS_DIAG 3     /* kappa tau* / ((2 pi)^{3/2} s_x s_y s_z)      (mapping 4)          */

/* Host-side plan: filled by dgsm_build_plan, consumed by dgsm_build_run.
 * Caller-owned plain struct; treat the fields as read-only. */
typedef struct dgsm_plan {
    int64_t n;
    int32_t n_lights, atlas_res, n_shells, chunk;
    int64_t n_keys;                                /* P = total (light, Gaussian, tile) keys */
    int64_t light_key_begin[DGSM_MAX_LIGHTS + 1];  /* per-light key segment [begin, begin') */
    uint32_t depth_min[DGSM_MAX_LIGHTS];           /* fp32 bit patterns of min/max D per light */
    uint32_t depth_max[DGSM_MAX_LIGHTS];
    int32_t depth_bits[DGSM_MAX_LIGHTS];           /* key bits used for (D bits - depth_min) */
    int32_t tile_bits;
    size_t run_workspace_bytes;                    /* size dgsm_build_run needs */
    uint64_t signature;                            /* ties a plan to its arguments */
} dgsm_plan_t;

/* Fill opts with the defaults: kappa=1, k_sigma=3, rho_scale=1, WRAP, flags=0. */
void dgsm_default_opts(dgsm_build_opts_t* opts);

/* Size in bytes of the plan workspace for n Gaussians and n_lights lights
 * (per-(light, Gaussian) footprint records, tile counts and their scan). */
size_t dgsm_plan_workspace_bytes(int64_t n, int n_lights);

/* DGSM build, step 1: per (light, Gaussian) calibration (Eq.5,
 * P:L128-136), light-space footprint and its 8x8 tile count;
 * exclusive scan of the counts.  Synchronises `stream` once to read P back.
 *   g, lights[n_lights]   occluders (device) and lights (host)
 *   atlas_res             H = W = atlas_res texels, multiple of 8, 8..2048
 *   n_shells              K radial shells, 1..DGSM_MAX_SHELLS
 *   opts                  NULL = defaults
 *   plan_ws               device, >= dgsm_plan_workspace_bytes(n, n_lights) bytes, 256-B aligned;
 *                         must stay untouched until dgsm_build_run has been enqueued
 *   plan                  host, filled on success (plan->run_workspace_bytes is the run size) */
int dgsm_build_plan(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights,
                    int atlas_res, int n_shells, const dgsm_build_opts_t* opts, void* plan_ws,
                    size_t plan_ws_bytes, dgsm_plan_t* plan, void* stream);

/* DGSM build, step 2 (Eq.2-4): key duplication into (tile, light
 * distance) pairs, onesweep radix sort, per-tile ranges, per-tile accumulation
 * of Eq.3 over K shells and T = exp(-tau).  Same g/lights/opts as the plan.
 *   run_ws     device, >= plan->run_workspace_bytes, 256-B aligned, scratch
 *   atlas_out  device float [n_lights][n_shells][atlas_res][atlas_res], k-major then
 *              row-major (row = v, col = u; Q3); fully overwritten with T (or tau). */
int dgsm_build_run(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights,
                   const dgsm_build_opts_t* opts, const dgsm_plan_t* plan, void* plan_ws,
                   size_t plan_ws_bytes, void* run_ws, size_t run_ws_bytes, float* atlas_out,
                   void* stream);

/* Binning only (a3-a5 of the build, for inspection and tests): runs the key
 * duplication, the onesweep sort and the tile ranges of dgsm_build_run, then
 * decodes the sorted keys.  Outputs (device, caller-owned):
 *   light_out, tile_out, depth_bits_out, index_out   uint32 [plan->n_keys]: entry j of the
 *       ascending (light, tile, fp32 bits of D, Gaussian index) order (R7); tile = row-major
 *       8x8 tile index ty*(res/8)+tx
 *   tile_start_out, tile_end_out   uint32 [n_lights*(res/8)^2] or NULL: [start, end) of each
 *       (light, tile) in that order (0, 0 for an empty tile) */
int dgsm_build_bins(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights,
                    const dgsm_build_opts_t* opts, const dgsm_plan_t* plan, void* plan_ws,
                    size_t plan_ws_bytes, void* run_ws, size_t run_ws_bytes, uint32_t* light_out,
                    uint32_t* tile_out, uint32_t* depth_bits_out, uint32_t* index_out,
                    uint32_t* tile_start_out, uint32_t* tile_end_out, void* stream);

/* Convenience: plan + run with one caller workspace `ws` laid out as
 * [plan workspace | run workspace].  If ws_bytes is too small, returns
 * DGSM_ENOSPC and stores the required size in *ws_required (after the plan
 * step, so the call synchronises the stream either way). */
int dgsm_build(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights,
               int atlas_res, int n_shells, const dgsm_build_opts_t* opts, void* ws,
               size_t ws_bytes, size_t* ws_required, float* atlas_out, void* stream);

/* ------------------------------------------------------------------
 * Sync-free build (no host synchronisation, capturable in a CUDA graph):
 * plan + run with the key arrays sized for a caller-chosen capacity instead
 * of the key count P (which dgsm_build_plan reads back).  Every launch size
 * is a function of (n, n_lights, atlas_res, n_shells, key_capacity); the
 * kernels read P and the per-light key segments on the device.
 * ------------------------------------------------------------------ */
typedef struct dgsm_build_status {
    uint64_t n_keys;    /* P of the build */
    uint32_t overflow;  /* 1: P > key_capacity — the atlas is NOT valid (all 1): rebuild with
                           key_capacity >= n_keys (dgsm_async_workspace_bytes grows with it) */
    uint32_t n_invalid; /* DGSM_VALIDATE: invalid Gaussians found (0 without the flag) */
} dgsm_build_status_t;

/* Device workspace bytes of dgsm_build_async (0 on bad input). */
size_t dgsm_async_workspace_bytes(int64_t n, int n_lights, int atlas_res, int n_shells, int64_t key_capacity);

/* As dgsm_build (Eq.2-4), enqueued on `stream`
 * without any host synchronisation.  key_capacity: 1 .. 2^30-1 keys;
 * ws: DEVICE, >= dgsm_async_workspace_bytes(...), 256-B aligned;
 * status: DEVICE dgsm_build_status_t written by the build (read it after the
 * stream has passed the build: overflow == 1 means the atlas is invalid).
 * The chunking of the accumulation follows key_capacity (the count the host
 * knows), so the result equals dgsm_build's up to fp32 summation order when
 * key_capacity differs from P, and bit for bit when key_capacity == P.
 * DGSM_COLLECT_STATS is not available here.
 * Errors: as dgsm_build_plan, DGSM_ENOSPC (workspace), DGSM_EINVAL (null status). */
int dgsm_build_async(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights, int atlas_res,
                     int n_shells, const dgsm_build_opts_t* opts, int64_t key_capacity, void* ws,
                     size_t ws_bytes, float* atlas_out, dgsm_build_status_t* status, void* stream);

/* T = exp(-tau) elementwise (Eq.4), in place allowed (tau == T). Device pointers.
 * Computed as 2^(-tau log2 e) with the hardware ex2 (relative error ~2^-22, T = 1
 * exactly at tau = 0), the same form as the build's own epilogue, so a sharded
 * build's tau -> T equals a single-GPU build's T up to the summation order of tau. */
int dgsm_exp_epilogue(const float* tau, float* T, int64_t count, void* stream);

/* DGSM sampling: for each receiver x_q (device [m][3]),
 *   T_out[q] = prod_l trilinear(atlas_l, psi(x_q - o_l), |x_q - o_l|)
 * octahedral bilinear with mirror-wrapped taps (Q12) x radial linear with t
 * clamped to [t_0, t_{K-1}]; T_l = 1 at the light itself (Q18); product over
 * lights (Q13).  If colors_inout (device [m][3]) is not NULL it is multiplied
 * by T_out in place ("multiply the direct term").
 *   atlas  device float [n_lights][n_shells][atlas_res][atlas_res] (as written by dgsm_build_run)
 *   T_out  device float [m] */
int dgsm_query(const float* atlas, const dgsm_light_t* lights, int n_lights, int atlas_res,
               int n_shells, const float* positions, int64_t m, float* T_out, float* colors_inout,
               void* stream);

/* ------------------------------------------------------------------
 * Receiver access order for the query (not in the paper: a B200 memory-
 * access choice, DESIGN.md §6 a8).  A query gathers 8 taps per light from a
 * [K][H][W] atlas of up to 2 GiB per light; receivers in arbitrary order make
 * every lane of a warp a random DRAM access.  Sorting the receivers by a
 * Morton code of their position makes neighbouring threads neighbours in
 * space, hence in every light's atlas.  The receivers of P:L185-187 are the
 * static scene Gaussians, so the order can be computed once per scene and
 * reused every frame (or per call: dgsm_query_ordered's cost then includes it).
 * ------------------------------------------------------------------ */
/* Device workspace bytes of dgsm_receiver_order for m receivers. */
size_t dgsm_order_workspace_bytes(int64_t m);

/* order_out (DEVICE uint32 [m]) = the permutation of 0..m-1 sorting the
 * receivers (DEVICE float [m][3]) by the 30-bit Morton code (10 bits per
 * axis) of their position in the receivers' own bounding box (stable: equal
 * codes keep index order).  ws: DEVICE, >= dgsm_order_workspace_bytes(m),
 * 256-B aligned.  Errors: DGSM_EINVAL, DGSM_ENOSPC, DGSM_ERANGE (m >= 2^30). */
int dgsm_receiver_order(const float* positions, int64_t m, uint32_t* order_out, void* ws, size_t ws_bytes,
                        void* stream);

/* dgsm_query visiting the receivers in the given order: thread j serves
 * receiver order[j] (position gathered, T_out[order[j]] and colours written
 * in place).  Every receiver's arithmetic is that of dgsm_query, so the result
 * is bit-identical to dgsm_query for any permutation `order` (DEVICE uint32
 * [m]); only the memory-access pattern changes.  order must be a permutation
 * of 0..m-1 (not checked: a repeated index races on its outputs). */
int dgsm_query_ordered(const float* atlas, const dgsm_light_t* lights, int n_lights, int atlas_res,
                       int n_shells, const float* positions, const uint32_t* order, int64_t m, float* T_out,
                       float* colors_inout, void* stream);

/* ------------------------------------------------------------------
 * Multi-GPU query of sharded atlases (the product over lights
 * Q13 and the linearity of the trilinear sample in the atlas values).  After
 * a reduce-scatter of the partial optical depth a rank holds, per light, a
 * chunk of shells [k_begin, k_end) of T.  dgsm_query_chunks samples each held
 * chunk at the receivers with the taps of dgsm_query, counting taps on shells
 * outside the chunk as 0:
 *   split[l] == 0 (the chunk holds every shell, k_begin = 0, k_end = K):
 *       T_out[q] = prod of T_l(x_q) over these lights (1 if none); an empty
 *       chunk (k_begin == k_end) with split[l] == 0 is skipped;
 *   split[l] != 0: partial_out[j][q] = the chunk's share of T_l(x_q), j = the
 *       rank of l among the split lights; summing partial_out over the ranks
 *       holding the light's other shells (all-reduce SUM) gives T_l(x_q).
 * dgsm_query_combine then folds the summed split lights in:
 *   T_inout[q] *= prod_j partial[j][q].
 *   chunks, k_begin, k_end, split: HOST arrays [n_lights]; chunks[l] is a DEVICE
 *       pointer to float [k_end - k_begin][res][res] (unused, may be NULL, when
 *       k_begin == k_end); 0 <= k_begin <= k_end <= n_shells.
 *   T_out: DEVICE float [m] (may be NULL when every light is split);
 *   partial_out: DEVICE float [n_split][m] (may be NULL when none is split).
 * Errors: DGSM_EINVAL (bad ranges, null pointers, a complete light whose
 * chunk is not [0, K)). */
int dgsm_query_chunks(const float* const* chunks, const int32_t* k_begin, const int32_t* k_end,
                      const int32_t* split, const dgsm_light_t* lights, int n_lights, int atlas_res, int n_shells,
                      const float* positions, int64_t m, float* T_out, float* partial_out, void* stream);
int dgsm_query_combine(const float* partial, int n_split, int64_t m, float* T_inout, void* stream);

/* One frame end to end from HOST memory (the benchmark's e2e path): upload the
 * occluder Gaussians (g_host: HOST arrays, pinned for copy/compute overlap) in
 * chunks, each projected as soon as it lands; build the atlas (plan + run, as
 * dgsm_build) into atlas_out (DEVICE, [L][K][H][W]); upload the receivers
 * (receivers_host, HOST float [m][3]) on a side stream while the atlas is
 * built; query them (dgsm_query) and return T (HOST float [m]): a page-locked
 * T_host is written directly by the query kernel over the bus, a pageable one
 * through a device buffer and a copy.  Stream-ordered on `stream`: T_host is
 * valid once `stream` has completed.
 *   ws, ws_bytes  caller-owned DEVICE workspace (256-B aligned).  *ws_required
 *                 receives the bytes needed: the plan part is known up front,
 *                 the run part after the plan — a call that returns
 *                 DGSM_ENOSPC has done no device work beyond the plan; grow the
 *                 workspace to *ws_required and call again.
 * Pipelining: the uploads of a frame wait only for the end of the previous frame
 * that used the SAME workspace (tracked per workspace address, 4 most recent),
 * not for work queued on `stream` in general: a caller alternating two
 * workspaces overlaps frame i+1's uploads with frame i's build.  The host
 * arrays must stay valid and unmodified until `stream` has passed the frame.
 * Errors: as dgsm_build_plan / dgsm_build_run / dgsm_query; DGSM_EINVAL for null
 * host arrays, DGSM_ENOSPC as above.  One host synchronisation (the plan). */
int dgsm_frame_host(const dgsm_gaussians_t* g_host, const dgsm_light_t* lights, int n_lights, int atlas_res,
                    int n_shells, const dgsm_build_opts_t* opts, const float* receivers_host, int64_t m,
                    float* T_host, void* ws, size_t ws_bytes, size_t* ws_required, float* atlas_out,
                    void* stream);

/* Footprint-sampled query ("rather than
 * integrating over each receiver's footprint", "sampling only the
 * Gaussian center ... tends to underestimate soft shadowing").  For receiver
 * Gaussian g (mean mu_g, scales s_g, quaternion q_g = (w, x, y, z), normalised
 * here, R_g its rotation):
 *   T_out[g] = prod_l sum_i weights[i] * T_l(mu_g + R_g (s_g . offsets[i]))
 * with T_l the trilinear sample of dgsm_query.  offsets are standard-normal
 * points z_i (e.g. a 7-point stencil {0, +-delta e_j} or Monte Carlo draws),
 * weights w_i (normally summing to 1); both are HOST arrays copied into the
 * kernel parameters, 1 <= n_samples <= DGSM_MAX_FOOTPRINT_SAMPLES.
 * offsets = {0,0,0}, weights = {1}, n_samples = 1 equals dgsm_query at mu_g.
 *   means/scales device float [m][3], rotations device float [m][4],
 *   T_out device float [m], colors_inout as in dgsm_query.
 * Errors: DGSM_EINVAL as dgsm_query, plus null offsets/weights or n_samples
 * outside [1, DGSM_MAX_FOOTPRINT_SAMPLES]. */
int dgsm_query_footprint(const float* atlas, const dgsm_light_t* lights, int n_lights, int atlas_res,
                         int n_shells, const float* means, const float* scales, const float* rotations,
                         int64_t m, const float* offsets, const float* weights, int n_samples,
                         float* T_out, float* colors_inout, void* stream);

/* Footprint sample sets for dgsm_query_footprint (host arithmetic, no device
 * work).  kind DGSM_STENCIL_CENTER: the single point z = 0, weight 1 (equals
 * dgsm_query at the means).  kind DGSM_STENCIL_7: the deterministic 7-point
 * stencil {0, +-delta e_1, +-delta e_2, +-delta e_3} in the receiver's
 * principal-axes frame with weights proportional to the standard normal
 * density exp(-|z|^2 / 2), normalised to sum 1 ("7-point";
 * centre weight 1 / (1 + 6 e^{-delta^2/2}) = 0.2156 at delta = 1).
 *   offsets_out HOST float [7][3], weights_out HOST float [7]; *n_out = the
 *   number of samples written (1 or 7).  Errors: DGSM_EINVAL (null pointers,
 *   unknown kind, delta not finite or <= 0 for the stencil). */
#define DGSM_STENCIL_CENTER 0
#define DGSM_STENCIL_7 1
int dgsm_footprint_stencil(int kind, float delta, float* offsets_out, float* weights_out, int* n_out);

/* ------------------------------------------------------------------
 * Receiver-driven region of interest and active voxel slab (SURVEY §8(f)
 * NEXT-1; §3.2).
 * ------------------------------------------------------------------ */
/* B = {x : ||(x - center)_xy||_inf <= radius, z_min <= x_z <= z_max}.
 * The paper leaves the centre (alpha-weighted avatar centroid) and the "robust
 * height bounds" to the caller; so does this ABI. */
typedef struct {
    float center[3];
    float radius;      /* R > 0 (the paper's example: 2 m) */
    float z_min, z_max;
} dgsm_roi_t;

/* Bytes of a slab buffer for n_lights lights at atlas_res (0 on bad input).
 * Layout (device, caller-owned, 256-B aligned sections):
 *   uint64_t texel_mask[n_lights][(atlas_res/8)^2]  bit (row%8)*8 + col%8 of
 *            word tile = (row/8)*(atlas_res/8) + col/8 is set iff texel
 *            (row, col) is in the pixel set P;
 *   int32_t  k_range[n_lights][2]                   k_min, k_max (k_min > k_max:
 *            no receiver for that light, the light's atlas stays 1). */
size_t dgsm_slab_bytes(int n_lights, int atlas_res);

/* Write the slab of the receivers x (device float [m][3], e.g. scene Gaussian
 * centres) for the lights: "For scene Gaussians whose centers lie in B, we
 * project their light rays into atlas pixels, collect the unique set P, and
 * infer a tight radial range k in [k_min, k_max] from their light-space
 * distances".  Pixel of a receiver = the texel whose cell holds
 * psi(x - o_L) (col = floor((u+1) W/2), clamped to W-1); its bin =
 * floor(|x - o_L| K / t_max), clamped to [0, K-1].  DESIGN.md reading R-ROI:
 * P is dilated by one pixel (neighbours mirror-wrapped like the sampler's
 * taps) and the bin range widened by one each side, so every trilinear tap
 * of a dgsm_query at a receiver in B lies in the slab and reads the value
 * the full build would have written.  A receiver exactly at a light is
 * skipped for that light.  fp64 decisions, bit-exact with the oracle.
 * Errors: DGSM_EINVAL (null/invalid arguments, radius <= 0, z_min > z_max),
 * DGSM_ENOSPC (slab_bytes < dgsm_slab_bytes). */
int dgsm_active_slab(const float* receivers, int64_t m, const dgsm_roi_t* roi, const dgsm_light_t* lights,
                     int n_lights, int atlas_res, int n_shells, void* slab, size_t slab_bytes,
                     void* stream);

/* ------------------------------------------------------------------
 * SH lighting transfer (§3.5)
 * ------------------------------------------------------------------ */
#define DGSM_MAX_SH_DEGREE 3

typedef struct dgsm_transfer_opts {
    int32_t grid_theta, grid_phi;  /* lat-long grid, M = grid_theta * grid_phi (default 64 x 128) */
    float q;                       /* cosine-lobe exponent >= 0 (default 1: Lambertian) */
    float eps;                     /* denominator guard (default 1e-6) */
    float s_max;                   /* clip bound, the paper's second "t_max" (default 4) */
    float gamma;                   /* global intensity (default 1) */
} dgsm_transfer_opts_t;

void dgsm_default_transfer_opts(dgsm_transfer_opts_t* opts);

/* Device workspace bytes of dgsm_sh_transfer for n Gaussians (0 on bad input). */
size_t dgsm_transfer_workspace_bytes(const dgsm_transfer_opts_t* opts, int64_t n);

/* Per-channel lighting scale of each Gaussian from an SH environment probe
 * and, if colors_in/colors_out are given, the relit colour:
 *   L_c(w_j) = max(0, sum_k Y_k(w_j) sh[c][k])    (negative ringing clamped: reading R-SH)
 *   S(w, n)  = max(0, <w, n>)^q
 *   s_c(n)   = clip_[0, s_max]( sum_j w_j L_c(w_j) S(w_j, n) / (sum_j w_j S(w_j, n) + eps) )
 *   c'       = max(0, gamma c (.) s(n))
 * over the lat-long grid theta_i = (i + 1/2) pi / grid_theta (from +z),
 * phi_k = (k + 1/2) 2 pi / grid_phi, w = sin(theta) (pi/grid_theta)(2 pi/grid_phi).
 *   sh        HOST float [3][(sh_degree+1)^2]: real orthonormal SH with the
 *             Condon-Shortley phase, index l^2 + l + m (the 3DGS convention)
 *   normals   DEVICE float [n][3], unit; colors_in / colors_out DEVICE [n][3] or NULL;
 *   scales_out DEVICE float [n][3] or NULL.
 * Errors: DGSM_EINVAL (sh_degree outside [0, DGSM_MAX_SH_DEGREE], grid < 1,
 * q < 0, eps < 0, s_max <= 0, null arrays), DGSM_ENOSPC (workspace). */
int dgsm_sh_transfer(const float* sh, int sh_degree, const float* normals, const float* colors_in, int64_t n,
                     const dgsm_transfer_opts_t* opts, float* scales_out, float* colors_out, void* ws,
                     size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------
 * The sort primitive of step a4 (the (tile, light-distance)
 * order of R7 — the paper itself never names a sort, P:L173 only buckets).
 * ------------------------------------------------------------------ */
/* Device scratch bytes for sorting up to n pairs (0 for n < 0). */
size_t dgsm_sort_temp_bytes(int64_t n);

/* Stable LSD onesweep radix sort of (key, value) pairs by key bits [0, nbits)
 * (higher key bits are ignored by the order and carried along).  keys/vals
 * and keys_alt/vals_alt are DEVICE uint32 [n] ping-pong buffers; the sorted
 * pairs end in (keys, vals) if *result_in_alt == 0 on return, else in
 * (keys_alt, vals_alt).  temp: DEVICE, >= dgsm_sort_temp_bytes(n), 256-B aligned.
 * Errors: DGSM_EINVAL (null buffers, nbits outside [0, 32]), DGSM_ENOSPC,
 * DGSM_ERANGE (n >= 2^30: the look-back status words hold 30-bit counts). */
int dgsm_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                        int nbits, void* temp, size_t temp_bytes, int* result_in_alt, void* stream);

/* Read the counters of the last DGSM_COLLECT_STATS dgsm_build_run that used
 * this run workspace (synchronises `stream`). */
int dgsm_build_stats(const dgsm_plan_t* plan, void* run_ws, size_t run_ws_bytes,
                     dgsm_build_stats_t* out, void* stream);

/* Benchmark instrumentation: caller-owned cudaEvent_t handles (as void*) that
 * subsequent dgsm_build_run calls on this thread record on their stream
 * immediately before and after the accumulation kernel (a6).  NULL, NULL
 * disables.  Always returns DGSM_OK. */
int dgsm_set_accumulate_events(void* before, void* after);

/* Frame pipelining: a caller-owned cudaEvent_t (as void*) that subsequent builds on
 * this thread record on their stream right before the work units and the
 * accumulation (a5/a6), with cudaEventRecordExternal: captured in a CUDA graph it is
 * an event-record node, so a copy stream can start the next frame's uploads when this
 * frame's FP32-bound accumulation starts (dgsm.FrameStream).  NULL disables.  Always
 * returns DGSM_OK. */
int dgsm_set_frame_event(void* ev);

/* Message for a status code / for the last failure on the calling thread. */
const char* dgsm_strerror(int code);
const char* dgsm_last_error(void);

/* Number of kernel launches enqueued by the last dgsm_build_run / dgsm_query /
 * dgsm_exp_epilogue on the calling thread (for the benchmark's gpu_launches). */
int dgsm_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* DGSM_H */
