// dgsm_internal.cuh — internal layouts and launch helpers of libdgsm.so.
// Nothing here is shared with oracle/ (which has its own independent code).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dgsm.h"

namespace dgsm {

constexpr int kTile = 8;             // 8x8 atlas tiles
constexpr int kTexels = kTile * kTile;
constexpr int kTileSplit = 1;         // accumulation work units per (tile, chunk) (2 = one warp per half tile: measured slower)

// Per-(light, Gaussian) footprint record written by the projection kernel and
// gathered (by TMA bulk copy) into shared memory by the accumulation kernel.
// 96 B = 6 x 16 B; array base is 256-B aligned so every record is 32-B aligned.
struct __align__(16) PairRec {
    double di[3];     // d_i = (mu - o)/D in fp64: the delta-formulation anchor (R9)
    float g[3];       // g = W d_i, W = diag(1/s) R^T (whitening: A = W^T W)
    float W[9];       // row-major W
    float D;          // |mu - o| (its fp32 bits are the depth key)
    float eD;         // t_{kD} - D (fp64 -> fp32), anchors the shell arguments
    int32_t kD;       // anchor shell
    float betap;      // beta * sqrt(pi/2) = kappa tau* sqrt(tr A / 3) / 2  (Eq.3 x Eq.5)
    float rcut_D2;    // negligible-pair bound r_cut / D^2 (R8', per Gaussian-light)
    uint32_t shells;  // lo | hi << 16: conservative bounds of the shells any live pair of this
                      // record writes (window rows and step row, hi inclusive, <= K): the
                      // accumulation's shell bands (accumulate.cu, DESIGN.md §6 a6)
};
static_assert(sizeof(PairRec) == 96, "PairRec must be 96 B");
// field offsets the accumulation kernel's register staging reads by word (accumulate.cu)
static_assert(offsetof(PairRec, g) == 24 && offsetof(PairRec, W) == 36 && offsetof(PairRec, D) == 72 &&
                  offsetof(PairRec, eD) == 76 && offsetof(PairRec, kD) == 80 && offsetof(PairRec, betap) == 84 &&
                  offsetof(PairRec, rcut_D2) == 88 && offsetof(PairRec, shells) == 92,
              "PairRec layout");

struct LightsParam {
    float4 l[DGSM_MAX_LIGHTS];  // xyz = o_L, w = t_max
};

// Footprint-query samples (NEXT-2): xyz = standard-normal offset z_i, w = weight.
struct FootprintParam {
    int n;
    float4 zw[DGSM_MAX_FOOTPRINT_SAMPLES];
};

// SH probe coefficients of the transfer (NEXT-4): [channel][l^2 + l + m], degree <= 3.
struct ShParam {
    float a[3][16];
    int d;
};

// Digit plan of an onesweep sort: pass p sorts key bits [shift[p], shift[p] + bits[p]).
constexpr int kSortRadix = 256;
constexpr int kSortMaxPasses = 8;
struct PassDigits {
    int shift[kSortMaxPasses], bits[kSortMaxPasses];
    int passes;
};

// Device-side statistics of a plan, copied back to the host once.
struct PlanStats {
    uint32_t depth_min[DGSM_MAX_LIGHTS];
    uint32_t depth_max[DGSM_MAX_LIGHTS];
    uint64_t light_key_begin[DGSM_MAX_LIGHTS + 1];
    uint32_t n_invalid, first_invalid;  // DGSM_VALIDATE: invalid Gaussians, the smallest invalid index
    PassDigits depth_pd[DGSM_MAX_LIGHTS];  // sync-free build: the depth sort's digits (k_run_setup)
};

// Work unit of the accumulation kernel: one chunk of one (light, tile) list.
struct __align__(16) WorkUnit {
    uint32_t tile;      // l * n_tiles + tile
    uint32_t jbeg, jend;  // [jbeg, jend) into the sorted (key, value) arrays
    uint32_t chunk;     // chunk index within the tile
    uint32_t nchunks;   // chunks of this tile (1 = write T directly)
    uint32_t slot;      // scratch slot of chunk 0 (multi-chunk tiles only)
    uint32_t part;      // which kTexels / kTileSplit texels of the tile (0 .. kTileSplit-1)
    uint32_t pad1;
};

// Region decomposition of the clamped footprint square on the extended lattice
// [-W, 2W-1]^2 into at most 9 pieces, each mapped by the mirror-wrap rule
// (R6/R10) onto a rectangle of tiles.  Integer-only: shared by the projection
// (tile count) and duplication (key emission) kernels so both enumerate the
// same tile set in the same order.
struct TileRects {
    int n;
    int tx0[9], tx1[9], ty0[9], ty1[9];
};

__host__ __device__ inline void make_tile_rects(int c0, int c1, int r0, int r1, int res, int bin_mode,
                                                TileRects& R) {
    R.n = 0;
    if (c0 > c1 || r0 > r1) return;
    const int W = res, H = res;
    if (bin_mode == DGSM_BIN_CLAMP) {
        int a = c0 < 0 ? 0 : c0, b = c1 > W - 1 ? W - 1 : c1;
        int c = r0 < 0 ? 0 : r0, d = r1 > H - 1 ? H - 1 : r1;
        if (a > b || c > d) return;
        R.tx0[0] = a >> 3; R.tx1[0] = b >> 3; R.ty0[0] = c >> 3; R.ty1[0] = d >> 3;
        R.n = 1;
        return;
    }
    // column regions: 0 = in-grid, 1 = left (<0), 2 = right (>W-1); rows: 0 in, 1 top (<0), 2 bottom (>H-1)
    int xa[3], xb[3], ya[3], yb[3];
    xa[0] = c0 < 0 ? 0 : c0;       xb[0] = c1 > W - 1 ? W - 1 : c1;
    xa[1] = c0;                    xb[1] = c1 < -1 ? c1 : -1;
    xa[2] = c0 > W ? c0 : W;       xb[2] = c1;
    ya[0] = r0 < 0 ? 0 : r0;       yb[0] = r1 > H - 1 ? H - 1 : r1;
    ya[1] = r0;                    yb[1] = r1 < -1 ? r1 : -1;
    ya[2] = r0 > H ? r0 : H;       yb[2] = r1;
    // fixed order: (in,in), then (x-overflow, in), (in, y-overflow), then corners
    const int order[9][2] = {{0, 0}, {1, 0}, {2, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 1}, {2, 2}};
    for (int o = 0; o < 9; ++o) {
        int rx = order[o][0], ry = order[o][1];
        int a = xa[rx], b = xb[rx], c = ya[ry], d = yb[ry];
        if (a > b || c > d) continue;
        int ma, mb, mc, md;  // mapped texel rectangle (inclusive)
        if (rx == 0 && ry == 0) { ma = a; mb = b; mc = c; md = d; }
        else if (ry == 0) {  // x overflow: col reflects, row flips
            if (rx == 1) { ma = -1 - b; mb = -1 - a; } else { ma = 2 * W - 1 - b; mb = 2 * W - 1 - a; }
            mc = H - 1 - d; md = H - 1 - c;
        } else if (rx == 0) {  // y overflow: row reflects, col flips
            if (ry == 1) { mc = -1 - d; md = -1 - c; } else { mc = 2 * H - 1 - d; md = 2 * H - 1 - c; }
            ma = W - 1 - b; mb = W - 1 - a;
        } else {  // corners: translation by (+-W, +-H)
            int sx = rx == 1 ? W : -W, sy = ry == 1 ? H : -H;
            ma = a + sx; mb = b + sx; mc = c + sy; md = d + sy;
        }
        R.tx0[R.n] = ma >> 3; R.tx1[R.n] = mb >> 3; R.ty0[R.n] = mc >> 3; R.ty1[R.n] = md >> 3;
        R.n++;
    }
}

__host__ __device__ inline bool in_earlier_rect(const TileRects& R, int j, int tx, int ty) {
    for (int q = 0; q < j; ++q)
        if (tx >= R.tx0[q] && tx <= R.tx1[q] && ty >= R.ty0[q] && ty <= R.ty1[q]) return true;
    return false;
}

// Number of distinct tiles in the union of the rectangles.
__host__ __device__ inline uint32_t count_tiles(const TileRects& R) {
    if (R.n == 0) return 0;
    uint32_t cnt = (uint32_t)(R.tx1[0] - R.tx0[0] + 1) * (uint32_t)(R.ty1[0] - R.ty0[0] + 1);
    for (int j = 1; j < R.n; ++j)
        for (int ty = R.ty0[j]; ty <= R.ty1[j]; ++ty)
            for (int tx = R.tx0[j]; tx <= R.tx1[j]; ++tx)
                if (!in_earlier_rect(R, j, tx, ty)) ++cnt;
    return cnt;
}

// Paired FP32 (sm_100 FFMA2 / FADD2 / FMUL2): a packed value holds two fp32
// operands (low, high); one f32x2 instruction does both.
// ---- programmatic dependent launch (PDL) -------------------------------------
// Every kernel of the library starts with pdl_begin(): it waits for the grid it
// depends on (griddepcontrol.wait: that grid has completed and its memory is
// visible; a no-op when the kernel was not launched as a dependent) and lets the
// next grid in the stream launch now (griddepcontrol.launch_dependents: its CTAs
// take SM slots as this grid's retire and wait there, hiding the launch gap).
// pdl_launch() launches with cudaLaunchAttributeProgrammaticStreamSerialization;
// captured in a CUDA graph these become programmatic dependency edges.
#ifndef DGSM_PDL
#define DGSM_PDL 1
#endif
__device__ __forceinline__ void pdl_begin() {
#if DGSM_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
#if DGSM_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
#else
    kernel<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
#endif
}

typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2add(f2_t a, f2_t b) { f2_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2_t f2sub(f2_t a, f2_t b) { f2_t d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2_t f2mul(f2_t a, f2_t b) { f2_t d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2_t f2fma(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t f2pack(float lo, float hi) { f2_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float f2lo(f2_t r) { float lo; asm("mov.b64 {%0, _}, %1;" : "=f"(lo) : "l"(r)); return lo; }
__device__ __forceinline__ float f2hi(f2_t r) { float hi; asm("mov.b64 {_, %0}, %1;" : "=f"(hi) : "l"(r)); return hi; }
__device__ __forceinline__ f2_t f2bc(float x) { return f2pack(x, x); }

// ROI slab buffer (include/dgsm.h dgsm_slab_bytes): per-tile texel masks, then k ranges.
inline size_t slab_mask_bytes(int n_lights, int res) {
    const size_t b = sizeof(uint64_t) * (size_t)n_lights * (res / kTile) * (res / kTile);
    return (b + 255) / 256 * 256;
}
inline const uint64_t* slab_mask_ptr(const void* slab) { return (const uint64_t*)slab; }
inline const int2* slab_k_ptr(const void* slab, int n_lights, int res) {
    return slab ? (const int2*)((const char*)slab + slab_mask_bytes(n_lights, res)) : nullptr;
}

// Number of distinct tiles of the footprint that are active in the ROI slab
// (tm = the light's per-tile texel masks, nonzero = active, NEXT-1); the same
// enumeration order as the key duplication.
__device__ inline uint32_t count_active_tiles(int c0, int c1, int r0, int r1, int res, int bin_mode,
                                              const uint64_t* __restrict__ tm) {
    const int TW = res / kTile;
    uint32_t cnt = 0;
    if (c0 > c1 || r0 > r1) return 0;
    if (c0 >= 0 && c1 <= res - 1 && r0 >= 0 && r1 <= res - 1) {
        for (int ty = r0 >> 3; ty <= (r1 >> 3); ++ty)
            for (int tx = c0 >> 3; tx <= (c1 >> 3); ++tx) cnt += tm[ty * TW + tx] != 0ull;
        return cnt;
    }
    TileRects TR;
    make_tile_rects(c0, c1, r0, r1, res, bin_mode, TR);
    for (int q = 0; q < TR.n; ++q)
        for (int ty = TR.ty0[q]; ty <= TR.ty1[q]; ++ty)
            for (int tx = TR.tx0[q]; tx <= TR.tx1[q]; ++tx) {
                if (q > 0 && in_earlier_rect(TR, q, tx, ty)) continue;
                cnt += tm[ty * TW + tx] != 0ull;
            }
    return cnt;
}

}  // namespace dgsm

// ---------------------------------------------------------------- kernels
// (declared here, defined in the .cu files, launched from dgsm_api.cu)
namespace dgsm {
void launch_project_init(PlanStats* stats, cudaStream_t s);
// Gaussians [i0, i0 + cnt) of every light (after launch_project_init)
void launch_project(const dgsm_gaussians_t& g, const LightsParam& lp, int n_lights, int res, int K,
                    const dgsm_build_opts_t& o, int64_t i0, int64_t cnt, PairRec* recs, uint32_t* counts,
                    uint4* dup, PlanStats* stats, cudaStream_t s);
size_t scan_u32_to_u64_temp_bytes(int64_t n);
constexpr int kScanLaunches = 2;  // kernels per launch_scan_* call
void launch_scan_u32_to_u64(const uint32_t* in, uint64_t* out, int64_t n, void* temp, cudaStream_t s);
void launch_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, void* temp, cudaStream_t s);
// the plan's light segment begins: begin[l + 1] += the key counts of lights <= l
void launch_light_begin(const uint32_t* counts, int64_t n, int n_lights, uint64_t* begin, cudaStream_t s);
// dup[l*n + i] = {fp32 bits of D, c0 | c1 << 16, r0 | r1 << 16, tile count} (16 B per (light, Gaussian))

void launch_gather_counts(const uint32_t* counts, const uint32_t* perm, int64_t n, uint32_t* cperm,
                          cudaStream_t s);
// keys written from base = *base_dev (the light's first key), none at or past *n_keys_dev;
// key = key_hi | tile (key_hi = light << tile_bits)
void launch_duplicate_ranked(const uint4* dup, const uint32_t* perm, const uint64_t* offs, int64_t n, int res,
                             int bin_mode, const uint64_t* base_dev, const uint64_t* n_keys_dev, uint32_t key_hi,
                             const uint64_t* tile_mask, uint32_t* keys, uint32_t* vals, cudaStream_t s);
size_t onesweep_temp_bytes(int64_t n_max);
// returns 1 if the sorted result ended in the *_alt buffers
int launch_onesweep(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int64_t n,
                    int nbits, void* temp, cudaStream_t s, int* launches);
// Onesweep digits: pass p sorts bits [shift[p], shift[p] + bits[p]) of the key,
// bits <= 8; the passes split the key's significant bits evenly (a 12-bit tile
// key: 6 + 6).  onesweep_prepare clears the sort's histograms, partition
// counters and first status buffer and returns the histograms [passes][256]; a
// key producer may fill them (hist_ready) instead of the sort's own k_hist.
PassDigits onesweep_digits(int nbits);
uint32_t* onesweep_prepare(void* temp, int64_t n, cudaStream_t s);
// depth keys (fp32 bits of D - the light's minimum, read on the device) of one light's
// Gaussians + their digit histograms into hist (pd.passes = 0: none)
void launch_depth_keys(const uint4* dup, int64_t n, const uint32_t* dmin_dev, uint32_t* keys, uint32_t* vals,
                       const PassDigits& pd, uint32_t* hist, cudaStream_t s, const PassDigits* pd_dev = nullptr);
// n_keys = P (light_key_begin[n_lights], device) or 0 + overflow when P > capacity
void launch_run_setup(PlanStats* ps, int n_lights, uint64_t capacity, uint64_t* n_keys,
                      dgsm_build_status_t* status, cudaStream_t s, int depth_passes = 0);
// (gsrc/gdst optional: the last pass also writes gdst[o] = gsrc[value] at each output
// position o, i.e. a gather by the sorted permutation; only when nbits > 0 and n > 1.
// top_match: rank the top pass with match.any (few distinct digits per warp, as in
// tile keys); false: ballots on every pass (random top digits, e.g. Morton codes))
int launch_onesweep_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                        int nbits, void* temp, cudaStream_t s, int* launches, const uint32_t* gsrc = nullptr,
                        uint32_t* gdst = nullptr, bool hist_ready = false, bool top_match = true,
                        const uint64_t* n_dev = nullptr, const PassDigits* pd_dev = nullptr);
void launch_decode_keys(const uint32_t* keys, const uint32_t* vals, const uint4* dup, const dgsm_plan_t& plan,
                        uint32_t* light_out, uint32_t* tile_out, uint32_t* depth_out, uint32_t* index_out,
                        cudaStream_t s);
// tile ranges of all lights' sorted keys (*n_dev keys, grid for `capacity`)
void launch_ranges(const uint32_t* keys, const uint64_t* n_dev, int64_t capacity, int tile_bits, uint32_t n_tiles,
                   uint32_t* tile_start, uint32_t* tile_end, cudaStream_t s);
// Multi-chunk tiles with at most this many chunks are combined by the
// accumulation CTA that finishes their last chunk; the others (listed by the
// unit builder) by k_combine_deferred after it (accumulate.cu).
constexpr uint32_t kInlineCombine = 16;
constexpr int kUnitClasses = 128;  // work-unit size classes (LPT dispatch order, binning.cu unit_class)
void launch_units(const uint32_t* tile_start, const uint32_t* tile_end, int64_t n_tiles_total, int chunk,
                  uint64_t* unit_counts, uint64_t* unit_offsets, void* scan_temp, WorkUnit* units_tmp,
                  WorkUnit* units, uint32_t max_units, uint32_t* n_units_dev, uint32_t* class_hist,
                  uint32_t* class_fill, uint32_t* deferred, uint32_t* deferred_count, cudaStream_t s,
                  int* launches);
size_t accumulate_smem_bytes(int K, bool tma);
bool accumulate_last_used_tma();  // staging of the last launch on this thread (benchmark info)
void launch_accumulate(const WorkUnit* units, const uint32_t* n_units_dev, uint32_t max_units,
                       const uint32_t* vals, const PairRec* recs, int64_t n, const LightsParam& lp,
                       int n_lights, int res, int K, uint32_t flags, float* scratch, uint32_t* tile_arrive,
                       uint32_t* unit_counter, float* atlas, unsigned long long* stats,
                       const uint64_t* slab_mask, const int2* slab_k, const uint32_t* deferred,
                       const uint32_t* deferred_count, cudaEvent_t ev_before, cudaEvent_t ev_after, cudaStream_t s);
int transfer_chunks(int64_t n, int64_t M);
size_t transfer_workspace_bytes(int n_theta, int n_phi, int64_t n);
void launch_transfer(const ShParam& sp, int n_theta, int n_phi, float q, float eps, float s_max, float gamma,
                     const float* normals, const float* colors, int64_t n, float* scales_out, float* colors_out,
                     void* ws, cudaStream_t s, int* launches);
void launch_active_slab(const float* x, int64_t m, const dgsm_roi_t& roi, const LightsParam& lp, int n_lights,
                        int res, int K, uint64_t* mask, int2* kr, cudaStream_t s, int* launches);
void launch_exp(const float* tau, float* T, int64_t count, cudaStream_t s);
void launch_query(const float* atlas, const LightsParam& lp, int n_lights, int res, int K,
                  const float* positions, int64_t m, float* T_out, float* colors, cudaStream_t s);
void launch_query_ordered(const float* atlas, const LightsParam& lp, int n_lights, int res, int K,
                          const float* positions, const uint32_t* order, int64_t m, float* T_out, float* colors,
                          cudaStream_t s);
// receivers' bounding box (box: 6 device words) + Morton keys, vals = index, and
// their onesweep digit histograms into hist (from onesweep_prepare) (2 kernels)
void launch_morton(const float* positions, int64_t m, uint32_t* box, uint32_t* keys, uint32_t* vals,
                   const PassDigits& pd, uint32_t* hist, cudaStream_t s);
void launch_query_chunks(const float* const* chunks, const int* kb, const int* ke, const int* split,
                         const LightsParam& lp, int n_lights, int res, int K, const float* positions, int64_t m,
                         float* T_out, float* partial_out, cudaStream_t s);
void launch_query_combine(const float* partial, int n, int64_t m, float* T, cudaStream_t s);
void launch_query_footprint(const float* atlas, const LightsParam& lp, const FootprintParam& fp, int n_lights,
                            int res, int K, const float* means, const float* scales, const float* rotations,
                            int64_t m, float* T_out, float* colors, cudaStream_t s);
}  // namespace dgsm
