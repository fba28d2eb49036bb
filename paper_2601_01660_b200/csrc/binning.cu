// binning.cu — key duplication (a3), per-tile ranges (a5) and the work units of
// the accumulation kernel.  "We bucket occluders into 8x8 atlas tiles using
// these rectangles"; the (tile, light-distance) key order is
// DESIGN.md reading Q10/R7.
#include "dgsm_internal.cuh"

namespace dgsm {

namespace {

struct DupParams {
    uint32_t depth_min[DGSM_MAX_LIGHTS];
    int32_t depth_bits[DGSM_MAX_LIGHTS];
};

// One thread per (light, Gaussian): emit its tiles in the fixed rectangle order
// (the same enumeration that produced its count).  Key (per light segment):
//   (tile << depth_bits) | (fp32 bits of D - depth_min)     value: Gaussian index
__global__ void __launch_bounds__(256) k_duplicate(const PairRec* __restrict__ recs,
                                                   const uint32_t* __restrict__ counts,
                                                   const uint64_t* __restrict__ offsets, int64_t n,
                                                   int n_lights, int res, int bin_mode, DupParams dp,
                                                   uint64_t* __restrict__ keys,
                                                   uint32_t* __restrict__ vals) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n_lights * n) return;
    const uint32_t cnt = counts[idx];
    if (cnt == 0) return;
    const int l = (int)(idx / n);
    const uint32_t i = (uint32_t)(idx - (int64_t)l * n);
    const PairRec& r = recs[idx];
    const uint64_t depth = (uint64_t)(__float_as_uint(r.D) - dp.depth_min[l]);
    const int db = dp.depth_bits[l];
    const int TW = res / kTile;
    uint64_t o = offsets[idx];
    const int c0 = r.c0, c1 = r.c1, r0 = r.r0, r1 = r.r1;
    if (c0 >= 0 && c1 <= res - 1 && r0 >= 0 && r1 <= res - 1) {  // common case: inside the grid
        for (int ty = r0 >> 3; ty <= (r1 >> 3); ++ty)
            for (int tx = c0 >> 3; tx <= (c1 >> 3); ++tx) {
                keys[o] = ((uint64_t)(ty * TW + tx) << db) | depth;
                vals[o] = i;
                ++o;
            }
        return;
    }
    TileRects TR;
    make_tile_rects(c0, c1, r0, r1, res, bin_mode, TR);
    for (int j = 0; j < TR.n; ++j)
        for (int ty = TR.ty0[j]; ty <= TR.ty1[j]; ++ty)
            for (int tx = TR.tx0[j]; tx <= TR.tx1[j]; ++tx) {
                if (j > 0 && in_earlier_rect(TR, j, tx, ty)) continue;
                const uint64_t tile = (uint64_t)(ty * TW + tx);
                keys[o] = (tile << db) | depth;
                vals[o] = i;
                ++o;
            }
}

// Tile ranges over one light's sorted segment [begin, end): absolute positions.
__global__ void __launch_bounds__(256) k_ranges(const uint64_t* __restrict__ keys, int64_t begin,
                                                int64_t end, int db, uint32_t tile_base,
                                                uint32_t* __restrict__ tile_start,
                                                uint32_t* __restrict__ tile_end) {
    const int64_t j = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= end) return;
    const uint32_t t = (uint32_t)(keys[j] >> db);
    if (j == begin || (uint32_t)(keys[j - 1] >> db) != t) tile_start[tile_base + t] = (uint32_t)j;
    if (j == end - 1 || (uint32_t)(keys[j + 1] >> db) != t) tile_end[tile_base + t] = (uint32_t)(j + 1);
}

// Per (light, tile): number of chunks (>= 1, an empty tile still writes T = 1)
// in the low 32 bits, scratch slots (chunks of multi-chunk tiles) in the high.
__global__ void __launch_bounds__(256) k_unit_counts(const uint32_t* __restrict__ ts,
                                                     const uint32_t* __restrict__ te, int64_t nt,
                                                     int chunk, uint64_t* __restrict__ cnt) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint32_t len = te[t] - ts[t];
    uint32_t c = (len + chunk - 1) / chunk;
    if (c == 0) c = 1;
    cnt[t] = (uint64_t)c | ((uint64_t)(c > 1 ? c : 0) << 32);
}

__global__ void __launch_bounds__(256) k_units(const uint32_t* __restrict__ ts,
                                               const uint32_t* __restrict__ te,
                                               const uint64_t* __restrict__ off, int64_t nt, int chunk,
                                               WorkUnit* __restrict__ units, uint32_t* n_units) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) *n_units = (uint32_t)(off[nt] & 0xffffffffu);
    if (t >= nt) return;
    const uint32_t s = ts[t], e = te[t];
    const uint64_t o = off[t];
    const uint32_t u0 = (uint32_t)(o & 0xffffffffu), slot = (uint32_t)(o >> 32);
    const uint32_t nc = (uint32_t)((off[t + 1] & 0xffffffffu) - u0);
    for (uint32_t c = 0; c < nc; ++c) {
        WorkUnit w;
        w.tile = (uint32_t)t;
        w.jbeg = s + c * (uint32_t)chunk;
        w.jend = min(e, w.jbeg + (uint32_t)chunk);
        if (w.jbeg > e) w.jbeg = e;
        w.chunk = c;
        w.nchunks = nc;
        w.slot = slot;
        w.pad0 = w.pad1 = 0;
        units[u0 + c] = w;
    }
}
struct DecodeParams {
    int64_t begin[DGSM_MAX_LIGHTS + 1];
    uint32_t depth_min[DGSM_MAX_LIGHTS];
    int32_t depth_bits[DGSM_MAX_LIGHTS];
    int n_lights;
};

__global__ void __launch_bounds__(256) k_decode(const uint64_t* __restrict__ keys,
                                                const uint32_t* __restrict__ vals, int64_t P, DecodeParams dp,
                                                uint32_t* lo, uint32_t* to, uint32_t* dout, uint32_t* io) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= P) return;
    int l = 0;
    while (l + 1 < dp.n_lights && j >= dp.begin[l + 1]) ++l;
    const uint64_t k = keys[j];
    const int db = dp.depth_bits[l];
    lo[j] = (uint32_t)l;
    to[j] = (uint32_t)(k >> db);
    dout[j] = (uint32_t)(k & ((db ? (~0ull >> (64 - db)) : 0ull))) + dp.depth_min[l];
    io[j] = vals[j];
}
}  // namespace

void launch_decode_keys(const uint64_t* keys, const uint32_t* vals, const dgsm_plan_t& plan, uint32_t* light_out,
                        uint32_t* tile_out, uint32_t* depth_out, uint32_t* index_out, cudaStream_t s) {
    if (plan.n_keys <= 0) return;
    DecodeParams dp;
    dp.n_lights = plan.n_lights;
    for (int l = 0; l <= DGSM_MAX_LIGHTS; ++l) dp.begin[l] = l <= plan.n_lights ? plan.light_key_begin[l] : 0;
    for (int l = 0; l < DGSM_MAX_LIGHTS; ++l) {
        dp.depth_min[l] = plan.depth_min[l];
        dp.depth_bits[l] = plan.depth_bits[l];
    }
    k_decode<<<(unsigned)((plan.n_keys + 255) / 256), 256, 0, s>>>(keys, vals, plan.n_keys, dp, light_out, tile_out,
                                                                  depth_out, index_out);
}

void launch_duplicate(const PairRec* recs, const uint32_t* counts, const uint64_t* offsets, int64_t n,
                      int n_lights, int res, int bin_mode, const dgsm_plan_t& plan, uint64_t* keys,
                      uint32_t* vals, cudaStream_t s) {
    const int64_t total = (int64_t)n_lights * n;
    if (total == 0 || plan.n_keys == 0) return;
    DupParams dp;
    for (int l = 0; l < DGSM_MAX_LIGHTS; ++l) {
        dp.depth_min[l] = l < n_lights ? plan.depth_min[l] : 0;
        dp.depth_bits[l] = l < n_lights ? plan.depth_bits[l] : 0;
    }
    k_duplicate<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(recs, counts, offsets, n, n_lights, res,
                                                                  bin_mode, dp, keys, vals);
}

void launch_ranges(const uint64_t* keys, int64_t begin, int64_t end, int depth_bits, uint32_t tile_base,
                   uint32_t* tile_start, uint32_t* tile_end, cudaStream_t s) {
    if (end <= begin) return;
    k_ranges<<<(unsigned)((end - begin + 255) / 256), 256, 0, s>>>(keys, begin, end, depth_bits,
                                                                    tile_base, tile_start, tile_end);
}

void launch_units(const uint32_t* tile_start, const uint32_t* tile_end, int64_t n_tiles_total, int chunk,
                  uint64_t* unit_counts, uint64_t* unit_offsets, void* scan_temp, WorkUnit* units,
                  uint32_t* n_units_dev, cudaStream_t s, int* launches) {
    uint64_t* cnt = unit_counts;
    const unsigned g = (unsigned)((n_tiles_total + 255) / 256);
    k_unit_counts<<<g, 256, 0, s>>>(tile_start, tile_end, n_tiles_total, chunk, cnt);
    launch_scan_u64(cnt, unit_offsets, n_tiles_total, scan_temp, s);
    k_units<<<g, 256, 0, s>>>(tile_start, tile_end, unit_offsets, n_tiles_total, chunk, units, n_units_dev);
    *launches += 5;
}

}  // namespace dgsm
