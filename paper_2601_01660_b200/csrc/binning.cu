// binning.cu — key duplication (a3), per-tile ranges (a5) and the work units of
// the accumulation kernel.  "We bucket occluders into 8x8 atlas tiles using
// these rectangles"; the (tile, light-distance) key order is
// DESIGN.md reading Q10/R7.
//
// Per light the order (tile, D bits, Gaussian index) is produced by an LSD
// radix sort whose low digits run on the un-duplicated Gaussians:
//   1. k_depth_keys + onesweep on N (D bits - D_min, index)  -> depth rank order
//   2. k_gather_counts + scan                                 -> emission offsets in that order
//   3. k_duplicate_ranked: each Gaussian, in depth-rank order, emits (tile, index)
//   4. onesweep (stable) on the P tile keys                   -> (tile, D bits, index)
#include <algorithm>
#include <cstdlib>

#include "dgsm_internal.cuh"

namespace dgsm {

namespace {

__device__ __forceinline__ void unpack_rect(const uint4& r, int& c0, int& c1, int& r0, int& r1) {
    c0 = (int16_t)(r.y & 0xffffu); c1 = (int16_t)(r.y >> 16);
    r0 = (int16_t)(r.z & 0xffffu); r1 = (int16_t)(r.z >> 16);
}

// Depth key of each Gaussian of one light (0 for Gaussians that bin no tile:
// they emit nothing, their position in the order is irrelevant), and the
// onesweep digit histograms of those keys (the sort's own histogram pass is
// skipped): grid-stride, per-CTA shared histograms, one global add per bin.
__global__ void __launch_bounds__(256) k_depth_keys(const uint4* __restrict__ dup, int64_t n,
                                                    const uint32_t* __restrict__ dmin_dev,
                                                    uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                    PassDigits pd, uint32_t* __restrict__ hist,
                                                    const PassDigits* __restrict__ pd_dev) {
    pdl_begin();
    if (pd_dev)  // the device's digit plan (same pass count)
        for (int p = 0; p < pd.passes; ++p) {
            pd.shift[p] = pd_dev->shift[p];
            pd.bits[p] = pd_dev->bits[p];
        }
    __shared__ uint32_t sh[kSortMaxPasses][kSortRadix];
    const uint32_t dmin = *dmin_dev;  // the light's smallest depth key (the plan's reduction, on the device)
    for (int t = threadIdx.x; t < pd.passes * kSortRadix; t += blockDim.x) (&sh[0][0])[t] = 0u;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 r = dup[i];
        const uint32_t k = r.w ? r.x - dmin : 0u;
        keys[i] = k;
        vals[i] = (uint32_t)i;
        for (int p = 0; p < pd.passes; ++p) atomicAdd(&sh[p][(k >> pd.shift[p]) & ((1u << pd.bits[p]) - 1u)], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < pd.passes * kSortRadix; t += blockDim.x) {
        const uint32_t c = (&sh[0][0])[t];
        if (c) atomicAdd(&hist[t], c);
    }
}

// key counts in depth-rank order (a 4-B gather from the count array, which
// stays L2-resident, rather than from the 16-B dup records)
__global__ void __launch_bounds__(256) k_gather_counts(const uint32_t* __restrict__ counts,
                                                       const uint32_t* __restrict__ perm, int64_t n,
                                                       uint32_t* __restrict__ cperm) {
    pdl_begin();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    cperm[j] = counts[perm[j]];
}

// One warp per 32 consecutive Gaussians in depth-rank order.  Their outputs
// are one contiguous segment [offs[j0], offs[j0 + 32]) (offs is the exclusive
// scan in this order), so the warp writes it cooperatively, 32 consecutive
// keys per store: lane l takes segment position p + l, finds the Gaussian that
// owns it (binary search over the lanes' offsets) and the k-th tile of that
// Gaussian's in-grid tile rectangle (row-major, the counting order).
// Gaussians whose footprint wraps across the atlas border, or any Gaussian when
// a ROI slab masks tiles, emit their own run in the fixed rectangle order
// (the enumeration that produced their count), as before.
__global__ void __launch_bounds__(256) k_duplicate_ranked(const uint4* __restrict__ dup,
                                                          const uint32_t* __restrict__ perm,
                                                          const uint64_t* __restrict__ offs, int64_t n,
                                                          int res, int bin_mode,
                                                          const uint64_t* __restrict__ base_dev,
                                                          const uint64_t* __restrict__ n_keys_dev,
                                                          uint32_t key_hi,
                                                          const uint64_t* __restrict__ tm,
                                                          uint32_t* __restrict__ keys,
                                                          uint32_t* __restrict__ vals) {
    pdl_begin();
    // keys of this light start at base = the plan's light_key_begin[l] (device);
    // nothing is written at or past n_keys (0 when the keys overflowed the
    // workspace capacity of a sync-free build).  key = light << tile_bits | tile.
    const uint64_t base = *base_dev, kcap = *n_keys_dev;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t j0 = j - lane;
    if (j0 >= n) return;  // whole warp past the end (warp-uniform)
    const bool valid = j < n;
    const uint32_t i = valid ? perm[j] : 0u;
    const uint4 r = valid ? dup[i] : make_uint4(0u, 0u, 0u, 0u);
    const int TW = res / kTile;
    int c0, c1, r0, r1;
    unpack_rect(r, c0, c1, r0, r1);
    const bool in_grid = c0 >= 0 && c1 <= res - 1 && r0 >= 0 && r1 <= res - 1;
    // a footprint covering the whole texel grid bins every tile once (its wrapped
    // rectangles only repeat tiles): the full grid as one cooperative rectangle
    const bool full = c0 <= 0 && c1 >= res - 1 && r0 <= 0 && r1 >= res - 1;
    const bool coop = r.w > 0 && (in_grid || full) && tm == nullptr;
    // segment of this warp and each lane's start within it
    const uint64_t seg0 = offs[j0];
    const uint32_t excl = (uint32_t)((valid ? offs[j] : offs[n]) - seg0);
    const uint32_t seg_len = __shfl_sync(0xffffffffu, excl + (valid ? r.w : 0u), 31);
    // the owner's rectangle packed in one word (tx0 | ty0 << 11 | wt << 22, wt = 0:
    // not cooperative) and 1/wt for the row split (exact: (k + 1/2)/wt is at least
    // 1/(2 wt) from an integer, far above fp32 rounding for k, wt < 2^11)
    const uint32_t tx0 = full ? 0u : (uint32_t)(c0 >> 3), ty0 = full ? 0u : (uint32_t)(r0 >> 3);
    const uint32_t wt = !coop ? 0u : (full ? (uint32_t)TW : (uint32_t)((c1 >> 3) - (c0 >> 3) + 1));
    const uint32_t rect = tx0 | (ty0 << 11) | (wt << 22);
    const float iwt = coop ? 1.0f / (float)wt : 0.0f;
    for (uint32_t p = 0; p < seg_len; p += 32) {
        const uint32_t q = p + (uint32_t)lane;
        int lo = 0;  // owner: the last lane whose start is <= q
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t e = __shfl_sync(0xffffffffu, excl, lo + step < 32 ? lo + step : 31);
            if (lo + step < 32 && e <= q) lo += step;
        }
        const uint32_t ek = __shfl_sync(0xffffffffu, excl, lo);
        const uint32_t o_rect = __shfl_sync(0xffffffffu, rect, lo);
        const float o_iwt = __shfl_sync(0xffffffffu, iwt, lo);
        const uint32_t o_i = __shfl_sync(0xffffffffu, i, lo);
        const uint32_t o_wt = o_rect >> 22;
        if (q < seg_len && o_wt && base + seg0 + q < kcap) {
            const uint32_t k = q - ek;
            const uint32_t dy = (uint32_t)(((float)k + 0.5f) * o_iwt), dx = k - dy * o_wt;
            keys[base + seg0 + q] =
                key_hi | (((o_rect >> 11) & 2047u) * (uint32_t)TW + dy * (uint32_t)TW + (o_rect & 2047u) + dx);
            vals[base + seg0 + q] = o_i;
        }
    }
    // The rest (Gaussians whose footprint wraps across the atlas border, or any
    // Gaussian under a ROI slab mask) one Gaussian at a time by the whole warp:
    // the lanes walk its tile rectangles 32 tiles per round and place the kept
    // tiles by ballot prefix.  A Gaussian's tiles are distinct, so the order
    // inside its run does not change the sorted result (the tile sort is stable
    // across Gaussians only).
    uint32_t pend = __ballot_sync(0xffffffffu, valid && r.w > 0 && !coop);
    const uint64_t my_o = valid ? offs[j] : 0ull;
    const uint32_t lt = (1u << lane) - 1u;
    while (pend) {
        const int L = __ffs(pend) - 1;
        pend &= pend - 1u;
        const int Lc0 = __shfl_sync(0xffffffffu, c0, L), Lc1 = __shfl_sync(0xffffffffu, c1, L);
        const int Lr0 = __shfl_sync(0xffffffffu, r0, L), Lr1 = __shfl_sync(0xffffffffu, r1, L);
        const uint32_t Li = __shfl_sync(0xffffffffu, i, L), Lw = __shfl_sync(0xffffffffu, r.w, L);
        uint64_t o = base + __shfl_sync(0xffffffffu, my_o, L);
        uint64_t end = o + Lw;  // never more keys than the plan counted (a slab changed since the plan)
        if (end > kcap) end = kcap;
        TileRects TR;
        make_tile_rects(Lc0, Lc1, Lr0, Lr1, res, Lc0 >= 0 && Lc1 <= res - 1 && Lr0 >= 0 && Lr1 <= res - 1
                                                     ? DGSM_BIN_CLAMP : bin_mode, TR);
#pragma unroll 1
        for (int q = 0; q < TR.n; ++q) {
            const int w = TR.tx1[q] - TR.tx0[q] + 1;
            const int cnt = w * (TR.ty1[q] - TR.ty0[q] + 1);
            for (int b0 = 0; b0 < cnt; b0 += 32) {
                const int idx = b0 + lane;
                const int ty = TR.ty0[q] + idx / w, tx = TR.tx0[q] + idx % w;
                bool ok = idx < cnt;
                if (ok && q > 0) ok = !in_earlier_rect(TR, q, tx, ty);
                if (ok && tm) ok = tm[ty * TW + tx] != 0ull;
                const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                const uint64_t at = o + __popc(bal & lt);
                if (ok && at < end) {
                    keys[at] = key_hi | (uint32_t)(ty * TW + tx);
                    vals[at] = Li;
                }
                o += __popc(bal);
            }
        }
    }
}

// Tile ranges over the sorted keys of all lights: [start, end) of each (light,
// tile) = l * n_tiles + tile, absolute positions; key = l << tile_bits | tile.
// The key count is read on the device (the grid covers the capacity).
__global__ void __launch_bounds__(256) k_ranges(const uint32_t* __restrict__ keys,
                                                const uint64_t* __restrict__ n_dev, int tile_bits,
                                                uint32_t n_tiles, uint32_t* __restrict__ tile_start,
                                                uint32_t* __restrict__ tile_end) {
    pdl_begin();
    const int64_t end = (int64_t)*n_dev;
    // four consecutive keys per thread (loads issued together), neighbours through L1
    const int64_t j0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (j0 >= end) return;
    uint32_t k[6];
#pragma unroll
    for (int u = 0; u < 6; ++u) {
        const int64_t j = j0 - 1 + u;
        k[u] = (j >= 0 && j < end) ? keys[j] : 0xffffffffu;
    }
    const uint32_t tmask = (1u << tile_bits) - 1u;
#pragma unroll
    for (int u = 1; u <= 4; ++u) {
        const int64_t j = j0 - 1 + u;
        if (j >= end) break;
        const uint32_t gt = (k[u] >> tile_bits) * n_tiles + (k[u] & tmask);
        if (k[u - 1] != k[u]) tile_start[gt] = (uint32_t)j;
        if (k[u + 1] != k[u]) tile_end[gt] = (uint32_t)(j + 1);
    }
}

// Sync-free run setup (one thread): the plan's key count P (on the device)
// against the workspace capacity; n_keys = P, or 0 with the overflow flag set
// when P exceeds it (the atlas is then all 1 and must be rebuilt with a larger
// workspace); the caller's status word receives both.
__global__ void k_run_setup(PlanStats* __restrict__ ps, int n_lights, uint64_t capacity,
                            uint64_t* __restrict__ n_keys, dgsm_build_status_t* status, int depth_passes) {
    pdl_begin();
    // sync-free build (depth_passes > 0): each light's depth keys (D bits - the
    // light's minimum) have bits(max - min) significant bits, known only here; they
    // are split evenly over the passes the host launched, as the planned build
    // splits them (digits that cannot occur stay out of the look-back)
    for (int l = 0; l < (depth_passes ? n_lights : 0); ++l) {
        const uint32_t lo = ps->depth_min[l], hi = ps->depth_max[l];
        const int db = hi > lo ? 32 - __clz(hi - lo) : 0;
        PassDigits& pd = ps->depth_pd[l];
        pd.passes = depth_passes;
        for (int p = 0, sh = 0; p < kSortMaxPasses; ++p) {
            const int b = p < depth_passes ? db / depth_passes + (p < db % depth_passes ? 1 : 0) : 0;
            pd.shift[p] = sh;
            pd.bits[p] = b;
            sh += b;
        }
    }
    const uint64_t P = ps->light_key_begin[n_lights];
    const bool over = P > capacity;
    *n_keys = over ? 0ull : P;
    if (status) {
        status->n_keys = P;
        status->overflow = over ? 1u : 0u;
        status->n_invalid = ps->n_invalid;
    }
}

// Per (light, tile): number of chunks (>= 1, an empty tile still writes T = 1)
// in the low 32 bits, scratch slots (chunks of multi-chunk tiles) in the high.
__global__ void __launch_bounds__(256) k_unit_counts(const uint32_t* __restrict__ ts,
                                                     const uint32_t* __restrict__ te, int64_t nt,
                                                     int chunk, uint64_t* __restrict__ cnt) {
    pdl_begin();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const uint32_t len = te[t] - ts[t];
    uint32_t c = (len + chunk - 1) / chunk;
    if (c == 0) c = 1;
    cnt[t] = (uint64_t)(c * kTileSplit) | ((uint64_t)(c > 1 ? c * kTileSplit : 0) << 32);
}

// Size class of a work unit for the longest-first dispatch order, monotone in
// its length: four classes per octave (len < 4: len itself).  Measured on cfg2:
// a6 1.05 -> 1.01 ms against one class per octave (a tail of same-class units
// that differ up to 2x in length).
__device__ __forceinline__ int unit_class(uint32_t len) {
    if (len < 4u) return (int)len;
    const int msb = 31 - __clz(len);
    const int c = 4 * (msb - 1) + (int)((len >> (msb - 2)) & 3u);
    return c < kUnitClasses ? c : kUnitClasses - 1;
}

__global__ void __launch_bounds__(256) k_units(const uint32_t* __restrict__ ts,
                                               const uint32_t* __restrict__ te,
                                               const uint64_t* __restrict__ off, int64_t nt, int chunk,
                                               WorkUnit* __restrict__ units, uint32_t* n_units,
                                               uint32_t* __restrict__ class_hist) {
    pdl_begin();
    __shared__ uint32_t s_hist[kUnitClasses];
    if (threadIdx.x < kUnitClasses) s_hist[threadIdx.x] = 0u;
    __syncthreads();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) *n_units = (uint32_t)(off[nt] & 0xffffffffu);
    if (t < nt) {
    const uint32_t s = ts[t], e = te[t];
    const uint64_t o = off[t];
    const uint32_t u0 = (uint32_t)(o & 0xffffffffu), slot = (uint32_t)(o >> 32);
    const uint32_t nc = (uint32_t)((off[t + 1] & 0xffffffffu) - u0) / kTileSplit;
    for (uint32_t part = 0; part < (uint32_t)kTileSplit; ++part)
    for (uint32_t c = 0; c < nc; ++c) {
        WorkUnit w;
        w.tile = (uint32_t)t;
        w.jbeg = s + c * (uint32_t)chunk;
        w.jend = min(e, w.jbeg + (uint32_t)chunk);
        if (w.jbeg > e) w.jbeg = e;
        w.chunk = c;
        w.nchunks = nc;
        w.slot = slot + part * nc;
        w.part = part;
        w.pad1 = 0;
        units[u0 + part * nc + c] = w;
        atomicAdd(&s_hist[unit_class(w.jend - w.jbeg)], 1u);
    }
    }
    __syncthreads();
    if (threadIdx.x < kUnitClasses && s_hist[threadIdx.x]) atomicAdd(&class_hist[threadIdx.x], s_hist[threadIdx.x]);
}

// Longest-processing-time-first order of the persistent accumulation grid:
// units are scattered by size class, largest class first, so the tail of the
// grid is made of the smallest units (results do not depend on this order:
// every unit writes its own tile or its own scratch slot).
__global__ void __launch_bounds__(256) k_units_lpt(const WorkUnit* __restrict__ in, const uint32_t* n_units,
                                                   const uint32_t* __restrict__ class_hist,
                                                   uint32_t* __restrict__ class_fill,
                                                   WorkUnit* __restrict__ out, uint32_t* __restrict__ deferred,
                                                   uint32_t* deferred_count) {
    pdl_begin();
    __shared__ uint32_t s_base[kUnitClasses];
    if (threadIdx.x == 0) {
        uint32_t b = 0;
        for (int c = kUnitClasses - 1; c >= 0; --c) { s_base[c] = b; b += class_hist[c]; }
    }
    __syncthreads();
    const uint32_t n = *n_units;
    // warp-aggregated class counters: most units share one class (full chunks), and one
    // global atomic per unit on its counter serialised (cfg5: 174 us for ~200 K units)
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
    for (uint32_t j0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); j0 < n; j0 += stride) {  // warp-uniform
        const uint32_t j = j0 + lane;
        WorkUnit w;
        int c = -1;
        if (j < n) {
            w = in[j];
            c = unit_class(w.jend - w.jbeg);
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, c);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0u;
        if ((int)lane == leader && c >= 0) base = atomicAdd(&class_fill[c], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (c >= 0) {
            const uint32_t pos = s_base[c] + base + (uint32_t)__popc(peers & lt);
            out[pos] = w;
            if (w.chunk == 0 && w.part == 0 && w.nchunks > kInlineCombine) deferred[atomicAdd(deferred_count, 1u)] = pos;
        }
    }
}

// sorted (light|tile key, Gaussian index) -> (light, tile, fp32 bits of D, index)
__global__ void __launch_bounds__(256) k_decode(const uint32_t* __restrict__ keys,
                                                const uint32_t* __restrict__ vals,
                                                const uint4* __restrict__ dup, int64_t n, int64_t P,
                                                int tile_bits, uint32_t* lo, uint32_t* to, uint32_t* dout,
                                                uint32_t* io) {
    pdl_begin();
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= P) return;
    const uint32_t l = keys[j] >> tile_bits;
    const uint32_t i = vals[j];
    lo[j] = l;
    to[j] = keys[j] & ((1u << tile_bits) - 1u);
    dout[j] = dup[(int64_t)l * n + i].x;
    io[j] = i;
}

// All of the above in one CTA for up to kFusedTiles (light, tile) pairs: pass 1
// counts the units per size class, pass 2 writes each unit at its class's next
// position (longest first) and gives multi-chunk tiles their scratch slots from
// a shared counter (slot positions are free: a tile's partials are combined in
// chunk order from its own slots).  One launch instead of five.
constexpr int kFusedThreads = 1024;
// single-CTA builder up to 16 K (light, tile) pairs (cfg2/cfg4: 4 K); above, the
// multi-kernel path: cfg3 (64 K) 9.14 -> 9.00 ms per step against the single CTA
#ifndef DGSM_FUSED_TILES
#define DGSM_FUSED_TILES (16 * 1024)
#endif
constexpr int64_t kFusedTiles = DGSM_FUSED_TILES;

__global__ void __launch_bounds__(kFusedThreads) k_units_fused(const uint32_t* __restrict__ ts,
                                                               const uint32_t* __restrict__ te, int64_t nt,
                                                               int chunk, WorkUnit* __restrict__ units,
                                                               uint32_t* n_units, uint32_t* __restrict__ deferred,
                                                               uint32_t* deferred_count) {
    pdl_begin();
    __shared__ uint32_t s_class[kUnitClasses], s_fill[kUnitClasses], s_slots;
    const int tid = threadIdx.x;
    if (tid < kUnitClasses) { s_class[tid] = 0u; s_fill[tid] = 0u; }
    if (tid == 0) s_slots = 0u;
    __syncthreads();
    // A tile's units: nfull full chunks (one size class) and, when the length is not a
    // multiple of the chunk (or the tile is empty: one empty unit, T = 1), a last one.
    // Each class counter takes one atomic per tile and kind, not one per unit (a dense
    // tile of an avatar close to the light has ~30 units of one class).
    const uint32_t cls_full = (uint32_t)unit_class((uint32_t)chunk);
    for (int64_t t = tid; t < nt; t += kFusedThreads) {
        const uint32_t len = te[t] - ts[t];
        const uint32_t nfull = len / (uint32_t)chunk, rem = len - nfull * (uint32_t)chunk;
        if (nfull) atomicAdd(&s_class[cls_full], nfull * (uint32_t)kTileSplit);
        if (rem || len == 0) atomicAdd(&s_class[unit_class(rem)], (uint32_t)kTileSplit);
    }
    __syncthreads();
    if (tid == 0) {  // class bases, largest class first: s_class becomes the base
        uint32_t base = 0;
        for (int c = kUnitClasses - 1; c >= 0; --c) { const uint32_t k = s_class[c]; s_class[c] = base; base += k; }
        *n_units = base;
    }
    __syncthreads();
    for (int64_t t = tid; t < nt; t += kFusedThreads) {
        const uint32_t s = ts[t], e = te[t], len = e - s;
        const uint32_t nfull = len / (uint32_t)chunk, rem = len - nfull * (uint32_t)chunk;
        const bool last = rem || len == 0;
        const uint32_t nc = nfull + (last ? 1u : 0u);
        const uint32_t slot = nc > 1 ? atomicAdd(&s_slots, nc * kTileSplit) : 0u;
        const uint32_t pos_full = nfull ? s_class[cls_full] + atomicAdd(&s_fill[cls_full], nfull * (uint32_t)kTileSplit) : 0u;
        const int cls_last = unit_class(rem);
        const uint32_t pos_last = last ? s_class[cls_last] + atomicAdd(&s_fill[cls_last], (uint32_t)kTileSplit) : 0u;
        for (uint32_t part = 0; part < (uint32_t)kTileSplit; ++part)
            for (uint32_t c = 0; c < nc; ++c) {
                WorkUnit w;
                w.tile = (uint32_t)t;
                w.jbeg = s + c * (uint32_t)chunk;
                w.jend = min(e, w.jbeg + (uint32_t)chunk);
                if (w.jbeg > e) w.jbeg = e;
                w.chunk = c;
                w.nchunks = nc;
                w.slot = slot + part * nc;
                w.part = part;
                w.pad1 = 0;
                const uint32_t pos = c < nfull ? pos_full + part * nfull + c : pos_last + part;
                units[pos] = w;
                if (c == 0 && part == 0 && nc > kInlineCombine) deferred[atomicAdd(deferred_count, 1u)] = pos;
            }
    }
}
}  // namespace

void launch_depth_keys(const uint4* dup, int64_t n, const uint32_t* dmin_dev, uint32_t* keys, uint32_t* vals,
                       const PassDigits& pd, uint32_t* hist, cudaStream_t s, const PassDigits* pd_dev) {
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 4);
    pdl_launch(k_depth_keys, (unsigned)blocks, 256, 0, s, dup, n, dmin_dev, keys, vals, pd, hist, pd_dev);
}

void launch_run_setup(PlanStats* ps, int n_lights, uint64_t capacity, uint64_t* n_keys,
                      dgsm_build_status_t* status, cudaStream_t s, int depth_passes) {
    pdl_launch(k_run_setup, 1, 1, 0, s, ps, n_lights, capacity, n_keys, status, depth_passes);
}

void launch_gather_counts(const uint32_t* counts, const uint32_t* perm, int64_t n, uint32_t* cperm,
                          cudaStream_t s) {
    if (n <= 0) return;
    pdl_launch(k_gather_counts, (unsigned)((n + 255) / 256), 256, 0, s, counts, perm, n, cperm);
}

void launch_duplicate_ranked(const uint4* dup, const uint32_t* perm, const uint64_t* offs, int64_t n, int res,
                             int bin_mode, const uint64_t* base_dev, const uint64_t* n_keys_dev, uint32_t key_hi,
                             const uint64_t* tile_mask, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    if (n <= 0) return;
    pdl_launch(k_duplicate_ranked, (unsigned)((n + 255) / 256), 256, 0, s, dup, perm, offs, n, res, bin_mode, base_dev,
                                                                    n_keys_dev, key_hi, tile_mask, keys, vals);
}

void launch_decode_keys(const uint32_t* keys, const uint32_t* vals, const uint4* dup, const dgsm_plan_t& plan,
                        uint32_t* light_out, uint32_t* tile_out, uint32_t* depth_out, uint32_t* index_out,
                        cudaStream_t s) {
    if (plan.n_keys <= 0) return;
    pdl_launch(k_decode, (unsigned)((plan.n_keys + 255) / 256), 256, 0, s, keys, vals, dup, plan.n, plan.n_keys,
                                                                  plan.tile_bits, light_out, tile_out, depth_out,
                                                                  index_out);
}

void launch_ranges(const uint32_t* keys, const uint64_t* n_dev, int64_t capacity, int tile_bits, uint32_t n_tiles,
                   uint32_t* tile_start, uint32_t* tile_end, cudaStream_t s) {
    if (capacity <= 0) return;
    pdl_launch(k_ranges, (unsigned)((capacity + 1023) / 1024), 256, 0, s, keys, n_dev, tile_bits, n_tiles, tile_start,
                                                                 tile_end);
}

void launch_units(const uint32_t* tile_start, const uint32_t* tile_end, int64_t n_tiles_total, int chunk,
                  uint64_t* unit_counts, uint64_t* unit_offsets, void* scan_temp, WorkUnit* units_tmp,
                  WorkUnit* units, uint32_t max_units, uint32_t* n_units_dev, uint32_t* class_hist,
                  uint32_t* class_fill, uint32_t* deferred, uint32_t* deferred_count, cudaStream_t s,
                  int* launches) {
    const bool force_multi = getenv("DGSM_UNITS_MULTI") != nullptr;  // tests: the > 64K-tile path
    if (n_tiles_total <= kFusedTiles && !force_multi) {
        pdl_launch(k_units_fused, 1, kFusedThreads, 0, s, tile_start, tile_end, n_tiles_total, chunk, units, n_units_dev,
                                                  deferred, deferred_count);
        *launches += 1;
        return;
    }
    const unsigned g = (unsigned)((n_tiles_total + 255) / 256);
    pdl_launch(k_unit_counts, g, 256, 0, s, tile_start, tile_end, n_tiles_total, chunk, unit_counts);
    launch_scan_u64(unit_counts, unit_offsets, n_tiles_total, scan_temp, s);
    pdl_launch(k_units, g, 256, 0, s, tile_start, tile_end, unit_offsets, n_tiles_total, chunk, units_tmp, n_units_dev,
                              class_hist);
    const unsigned gl = (unsigned)std::min<uint32_t>((max_units + 255) / 256, 148u * 8u);
    pdl_launch(k_units_lpt, gl, 256, 0, s, units_tmp, n_units_dev, class_hist, class_fill, units, deferred, deferred_count);
    *launches += 3 + kScanLaunches;
}

}  // namespace dgsm
