// scan.cu — exclusive prefix sums (reduce-then-scan, 3 launches) used for the
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

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_reduce(const T* __restrict__ in, int64_t n,
                                                         uint64_t* __restrict__ partials) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t k = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (k < n) s += in[k];
    }
    uint64_t total;
    block_excl_scan(s, &total);
    if (threadIdx.x == 0) partials[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(uint64_t* partials, int64_t nb) {
    uint64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
        int64_t k = b0 + threadIdx.x;
        uint64_t v = k < nb ? partials[k] : 0;
        uint64_t total;
        uint64_t ex = block_excl_scan(v, &total);
        if (k < nb) partials[k] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) partials[nb] = carry;
}

template <typename T, typename O>
__global__ void __launch_bounds__(kScanThreads) k_downsweep(const T* __restrict__ in, int64_t n,
                                                            const uint64_t* __restrict__ partials,
                                                            int64_t nb, O* __restrict__ out) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    // blocked arrangement: thread t owns items [base + t*16, base + t*16 + 16)
    __shared__ T tile[kScanTile];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t k = base + (int64_t)j * kScanThreads + threadIdx.x;
        tile[j * kScanThreads + threadIdx.x] = k < n ? in[k] : T(0);
    }
    __syncthreads();
    uint64_t v[kScanItems];
    uint64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = tile[threadIdx.x * kScanItems + j];
        s += v[j];
    }
    uint64_t total;
    uint64_t run = block_excl_scan(s, &total) + partials[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t k = base + (int64_t)threadIdx.x * kScanItems + j;
        if (k < n) out[k] = (O)run;
        run += v[j];
    }
    if (blockIdx.x == nb - 1 && threadIdx.x == 0) out[n] = (O)partials[nb];
}

template <typename T, typename O>
void scan_impl(const T* in, O* out, int64_t n, void* temp, cudaStream_t s) {
    uint64_t* partials = (uint64_t*)temp;
    if (n == 0) {
        cudaMemsetAsync(out, 0, sizeof(O), s);
        return;
    }
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    k_reduce<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partials);
    k_scan_partials<<<1, kScanThreads, 0, s>>>(partials, nb);
    k_downsweep<T, O><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partials, nb, out);
}

__global__ void k_plan_stats(const uint64_t* __restrict__ offsets, int64_t n, int n_lights,
                             PlanStats* stats) {
    int l = threadIdx.x;
    if (l <= n_lights) stats->light_key_begin[l] = offsets[(int64_t)l * n];
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

void launch_plan_stats(const uint64_t* offsets, int64_t n, int n_lights, PlanStats* stats,
                       cudaStream_t s) {
    k_plan_stats<<<1, DGSM_MAX_LIGHTS + 1, 0, s>>>(offsets, n, n_lights, stats);
}

}  // namespace dgsm
