// scan.cu — exclusive prefix sums (reduce-then-scan, 2 launches) used for the
// per-Gaussian key offsets in depth-rank order and the per-tile work-unit
// offsets; the plan's per-light key totals (a segmented reduction).
#include <algorithm>

#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096 elements per block

__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Block-wide exclusive scan of one value per thread; returns the block total in *total.
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t x, uint64_t* total) {
    __shared__ uint64_t warp_sums[kScanThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t inc = warp_incl_scan(x);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint64_t v = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
        v = warp_incl_scan(v);
        if (lane < kScanThreads / 32) warp_sums[lane] = v;
    }
    __syncthreads();
    const uint64_t warp_prefix = wid ? warp_sums[wid - 1] : 0;
    *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads();
    return warp_prefix + inc - x;
}

// Two launches: k_reduce sums each block's contiguous run of 4096-element tiles;
// k_downsweep adds the partials of the blocks before it (<= kMaxBlocks values,
// L2-resident) and scans its run tile by tile, storing coalesced through shared
// memory.  The grid is capped at kMaxBlocks so that prefix read stays small.
constexpr int64_t kMaxBlocks = 1024;

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_reduce(const T* __restrict__ in, int64_t n, int64_t tpb,
                                                         uint64_t* __restrict__ partials) {
    pdl_begin();
    const int64_t t0 = (int64_t)blockIdx.x * tpb;
    uint64_t s = 0;
    for (int64_t t = t0; t < t0 + tpb; ++t) {
        const int64_t base = t * kScanTile;
        if (base >= n) break;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            const int64_t k = base + (int64_t)j * kScanThreads + threadIdx.x;
            if (k < n) s += in[k];
        }
    }
    uint64_t total;
    block_excl_scan(s, &total);
    if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

template <typename T, typename O>
__global__ void __launch_bounds__(kScanThreads) k_downsweep(const T* __restrict__ in, int64_t n, int64_t tpb,
                                                            const uint64_t* __restrict__ partials,
                                                            O* __restrict__ out) {
    pdl_begin();
    // padded: element e at e + e/16, so the blocked accesses (stride 16) spread over banks
    __shared__ uint64_t tile[kScanTile + kScanTile / kScanItems];
    auto at = [](int e) { return e + (e >> 4); };
    // exclusive prefix of this block: the partials of the blocks before it
    uint64_t pre = 0;
    for (int64_t b = threadIdx.x; b < (int64_t)blockIdx.x; b += kScanThreads) pre += partials[b];
    uint64_t carry;
    block_excl_scan(pre, &carry);
    const int64_t t0 = (int64_t)blockIdx.x * tpb;
    for (int64_t t = t0; t < t0 + tpb; ++t) {
        const int64_t base = t * kScanTile;
        if (base >= n) break;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {  // coalesced load
            const int64_t k = base + (int64_t)j * kScanThreads + threadIdx.x;
            tile[at(j * kScanThreads + threadIdx.x)] = k < n ? (uint64_t)in[k] : 0ull;
        }
        __syncthreads();
        uint64_t v[kScanItems];
        uint64_t s = 0;
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {  // blocked: thread t owns items [16 t, 16 t + 16)
            v[j] = tile[at(threadIdx.x * kScanItems + j)];
            s += v[j];
        }
        uint64_t total;
        uint64_t run = carry + block_excl_scan(s, &total);  // (its barriers also order the tile reads)
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {
            tile[at(threadIdx.x * kScanItems + j)] = run;
            run += v[j];
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kScanItems; ++j) {  // coalesced store
            const int64_t k = base + (int64_t)j * kScanThreads + threadIdx.x;
            if (k < n) out[k] = (O)tile[at(j * kScanThreads + threadIdx.x)];
        }
        carry += total;
        if (base + kScanTile >= n && threadIdx.x == 0) out[n] = (O)carry;
        __syncthreads();
    }
}

template <typename T, typename O>
void scan_impl(const T* in, O* out, int64_t n, void* temp, cudaStream_t s) {
    uint64_t* partials = (uint64_t*)temp;
    if (n == 0) {
        cudaMemsetAsync(out, 0, sizeof(O), s);
        return;
    }
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    const int64_t tpb = (tiles + kMaxBlocks - 1) / kMaxBlocks;
    const int64_t nb = (tiles + tpb - 1) / tpb;
    pdl_launch(k_reduce<T>, (unsigned)nb, kScanThreads, 0, s, in, n, tpb, partials);
    pdl_launch(k_downsweep<T, O>, (unsigned)nb, kScanThreads, 0, s, in, n, tpb, partials, out);
}

// Per-light key totals of the plan: only the light segments' begins are used
// downstream (the per-Gaussian offsets are scanned in depth-rank order by the
// run), so a reduction replaces the full scan.  Each block sums a contiguous
// range of counts per light segment, then thread t adds the block's total of
// the lights < t + 1 to begin[t + 1] (begin zeroed by the plan's init kernel).
__global__ void __launch_bounds__(kScanThreads) k_light_begin(const uint32_t* __restrict__ counts, int64_t n,
                                                              int n_lights, uint64_t* begin) {
    pdl_begin();
    __shared__ unsigned long long s_tot[DGSM_MAX_LIGHTS];
    if (threadIdx.x < DGSM_MAX_LIGHTS) s_tot[threadIdx.x] = 0ull;
    __syncthreads();
    const int64_t m = n * n_lights;
    const int64_t per = (m + gridDim.x - 1) / gridDim.x;
    const int64_t a = (int64_t)blockIdx.x * per, e = a + per < m ? a + per : m;
    for (int64_t seg = a; seg < e;) {  // block-uniform loop over the light segments of [a, e)
        const int l = (int)(seg / n);
        const int64_t se = (int64_t)(l + 1) * n < e ? (int64_t)(l + 1) * n : e;
        uint64_t t = 0;
#pragma unroll 4
        for (int64_t j = seg + threadIdx.x; j < se; j += kScanThreads) t += counts[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if ((threadIdx.x & 31) == 0 && t) atomicAdd(&s_tot[l], (unsigned long long)t);
        seg = se;
    }
    __syncthreads();
    if ((int)threadIdx.x < n_lights) {
        unsigned long long pre = 0ull;
        for (int l = 0; l <= (int)threadIdx.x; ++l) pre += s_tot[l];
        if (pre) atomicAdd(reinterpret_cast<unsigned long long*>(begin + threadIdx.x + 1), pre);
    }
}

}  // namespace

void launch_light_begin(const uint32_t* counts, int64_t n, int n_lights, uint64_t* begin, cudaStream_t s) {
    const int64_t m = n * n_lights;
    if (m <= 0) return;
    const int64_t blocks = std::min<int64_t>((m + kScanThreads * 8 - 1) / (kScanThreads * 8), 148 * 8);
    pdl_launch(k_light_begin, (unsigned)blocks, kScanThreads, 0, s, counts, n, n_lights, begin);
}

size_t scan_u32_to_u64_temp_bytes(int64_t n) {
    return sizeof(uint64_t) * (size_t)((n + kScanTile - 1) / kScanTile + 2);
}

void launch_scan_u32_to_u64(const uint32_t* in, uint64_t* out, int64_t n, void* temp, cudaStream_t s) {
    scan_impl<uint32_t, uint64_t>(in, out, n, temp, s);
}

void launch_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, void* temp, cudaStream_t s) {
    scan_impl<uint64_t, uint64_t>(in, out, n, temp, s);
}

}  // namespace dgsm
