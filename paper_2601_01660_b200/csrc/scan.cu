// scan.cu — exclusive prefix sums (reduce-then-scan, 2 launches) used for the
// per-(light, Gaussian) key offsets and the per-tile work-unit offsets.
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
                                                            O* __restrict__ out, uint64_t* __restrict__ marks,
                                                            int64_t mark_stride, int n_marks) {
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
        // marks[i] = out[i * mark_stride] (i <= n_marks; the plan's per-light key begins)
        if (marks && threadIdx.x <= (unsigned)n_marks) {
            const int64_t k = (int64_t)threadIdx.x * mark_stride;
            if (k >= base && k < base + kScanTile && k < n) marks[threadIdx.x] = tile[at((int)(k - base))];
        }
        carry += total;
        if (base + kScanTile >= n && threadIdx.x == 0) out[n] = (O)carry;
        if (base + kScanTile >= n && marks && threadIdx.x <= (unsigned)n_marks &&
            (int64_t)threadIdx.x * mark_stride >= n)
            marks[threadIdx.x] = carry;
        __syncthreads();
    }
}

template <typename T, typename O>
void scan_impl(const T* in, O* out, int64_t n, void* temp, cudaStream_t s, uint64_t* marks = nullptr,
               int64_t mark_stride = 1, int n_marks = 0) {
    uint64_t* partials = (uint64_t*)temp;
    if (n == 0) {
        cudaMemsetAsync(out, 0, sizeof(O), s);
        if (marks) cudaMemsetAsync(marks, 0, sizeof(uint64_t) * (n_marks + 1), s);
        return;
    }
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    const int64_t tpb = (tiles + kMaxBlocks - 1) / kMaxBlocks;
    const int64_t nb = (tiles + tpb - 1) / tpb;
    pdl_launch(k_reduce<T>, (unsigned)nb, kScanThreads, 0, s, in, n, tpb, partials);
    pdl_launch(k_downsweep<T, O>, (unsigned)nb, kScanThreads, 0, s, in, n, tpb, partials, out, marks, mark_stride,
                                                            n_marks);
}

}  // namespace

size_t scan_u32_to_u64_temp_bytes(int64_t n) {
    return sizeof(uint64_t) * (size_t)((n + kScanTile - 1) / kScanTile + 2);
}

void launch_scan_u32_to_u64(const uint32_t* in, uint64_t* out, int64_t n, void* temp, cudaStream_t s) {
    scan_impl<uint32_t, uint64_t>(in, out, n, temp, s);
}

void launch_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, void* temp, cudaStream_t s) {
    scan_impl<uint64_t, uint64_t>(in, out, n, temp, s);
}

void launch_scan_u32_to_u64_marks(const uint32_t* in, uint64_t* out, int64_t n, void* temp, uint64_t* marks,
                                  int64_t mark_stride, int n_marks, cudaStream_t s) {
    scan_impl<uint32_t, uint64_t>(in, out, n, temp, s, marks, mark_stride, n_marks);
}

}  // namespace dgsm
