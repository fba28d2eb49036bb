// onesweep.cu — stable LSD radix sort of (key, u32 value) pairs, key = u32 or
// u64, in the "onesweep" style: one histogram pass over all digits, then ONE
// kernel per digit (<= 8 bits) that ranks a 4096-key partition in shared memory (warp
// multi-split by ballots, or match.any on a narrow top digit), obtains its global digit offsets by decoupled
// look-back over earlier partitions (8 predecessors per round trip), and
// scatters through shared memory for coalesced writes.  Partition ids come from
// an atomic counter, so a CTA only ever waits on partitions that are already
// running (forward progress without co-residency).
//
// The build uses it twice per light (binning.cu / dgsm_api.cu): the low digits
// (fp32 bits of the light distance D) are sorted on the N Gaussians before key
// duplication, the high digits (tile index) on the P duplicated keys emitted in
// that depth order — an LSD radix sort whose low passes run on the
// un-duplicated array.  Stability gives the order (tile, D bits, Gaussian index)
// of DESIGN.md R7.
#include <atomic>

#include "dgsm_internal.cuh"

namespace dgsm {

namespace {
constexpr int kThreads = 256;
// tuning knobs: an 8-wide look-back window (tools/ab_sort.sh; 16/32-wide slower);
// 16 keys per thread at 2 CTAs/SM (tools/ab_os16.sh, whole steps: cfg2 -5 us,
// cfg5 -0.13 ms, cfg3 +0.02 ms against 8 keys at 4 CTAs/SM; 12 keys at 3 CTAs/SM:
// cfg5 -0.27 ms but cfg2 +4 us; 12 or 16 under the 4-CTA bound spill)
#ifndef DGSM_OS_ITEMS
#define DGSM_OS_ITEMS 16
#endif
constexpr int kItems = DGSM_OS_ITEMS;
#ifndef DGSM_OS_MINB
#define DGSM_OS_MINB 2  // CTAs per SM the pass kernel is register-bounded for (126 registers)
#endif
constexpr int kTileKeys = kThreads * kItems;  // 4096 keys per partition (126 regs: 2 CTAs/SM)
constexpr int kRadix = kSortRadix;
constexpr int kMaxPasses = kSortMaxPasses;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;


template <typename KeyT>
__global__ void __launch_bounds__(256) k_hist(const KeyT* __restrict__ keys, int64_t n, int passes,
                                              PassDigits pd, uint32_t* __restrict__ hist,
                                              const uint64_t* __restrict__ n_dev) {
    pdl_begin();
    if (n_dev) n = (int64_t)*n_dev;  // device-side count (<= the launch capacity)
    __shared__ uint32_t sh[kMaxPasses][kRadix];
    for (int t = threadIdx.x; t < kMaxPasses * kRadix; t += blockDim.x) (&sh[0][0])[t] = 0;
    __syncthreads();
    // 8 keys per thread per round, loads issued together (memory-level parallelism)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < n; j0 += 8 * stride) {
        KeyT k[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t j = j0 + u * stride;
            k[u] = j < n ? keys[j] : (KeyT)0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (j0 + u * stride >= n) break;
            for (int p = 0; p < passes; ++p)
                atomicAdd(&sh[p][(uint32_t)(k[u] >> pd.shift[p]) & ((1u << pd.bits[p]) - 1u)], 1u);
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < passes * kRadix; t += blockDim.x) {
        const uint32_t c = (&sh[0][0])[t];
        if (c) atomicAdd(&hist[t], c);
    }
}

__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t x, uint32_t* warp_sums) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t v = lane < kThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane < kThreads / 32) warp_sums[lane] = v;
    }
    __syncthreads();
    const uint32_t r = (wid ? warp_sums[wid - 1] : 0) + inc - x;
    __syncthreads();
    return r;
}

#ifndef DGSM_OS_WIN_NARROW
#define DGSM_OS_WIN_NARROW 8
#endif
#ifndef DGSM_OS_NARROW_BITS
#define DGSM_OS_NARROW_BITS 6
#endif
// Decoupled look-back of digit d for partition `part`: sum the aggregates of the
// predecessors, kWin per round trip, until an inclusive prefix is found;
// re-poll from the first predecessor that has not published yet.
template <int kWin>
__device__ __forceinline__ uint32_t look_back(volatile uint32_t* st, uint32_t part, uint32_t d) {
    uint32_t excl = 0;
    int64_t q = (int64_t)part - 1;
    while (true) {
        uint32_t s[kWin];
#pragma unroll
        for (int i = 0; i < kWin; ++i) s[i] = (q - i >= 0) ? st[(size_t)(q - i) * kRadix + d] : 0u;
        int i = 0;
        bool done = false;
#pragma unroll
        for (int w = 0; w < kWin; ++w) {
            if (done || w != i) continue;
            const uint32_t f = s[w] & ~kValMask;
            if (f == 0) continue;  // not ready: stop consuming this window
            excl += s[w] & kValMask;
            if (f == kFlagInc) done = true;
            ++i;
        }
        if (done) return excl;
        q -= i;
    }
}

template <typename KeyT>
__global__ void __launch_bounds__(kThreads, DGSM_OS_MINB) k_pass(const KeyT* __restrict__ kin,
                                                      const uint32_t* __restrict__ vin,
                                                      KeyT* __restrict__ kout, uint32_t* __restrict__ vout,
                                                      int64_t n, int shift, int bits, bool top,
                                                      const uint32_t* __restrict__ hist,
                                                      uint32_t* status, uint32_t* status_next,
                                                      uint32_t* part_ctr, const uint32_t* __restrict__ gsrc,
                                                      uint32_t* __restrict__ gdst,
                                                      const uint64_t* __restrict__ n_dev,
                                                      const PassDigits* __restrict__ pd_dev, int pass) {
    pdl_begin();
    if (pd_dev) {  // the digit plan made on the device (sync-free build: the depth range)
        shift = pd_dev->shift[pass];
        bits = pd_dev->bits[pass];
    }
    extern __shared__ __align__(16) unsigned char os_smem[];
    KeyT* s_keys = reinterpret_cast<KeyT*>(os_smem);
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(os_smem + sizeof(KeyT) * kTileKeys);
    __shared__ uint32_t s_warp_hist[kThreads / 32][kRadix];
    __shared__ uint32_t s_tile_start[kRadix];
    __shared__ uint32_t s_global[kRadix];
    __shared__ uint32_t s_ws[kThreads / 32];
    __shared__ uint32_t s_part;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_part = atomicAdd(part_ctr, 1u);
    for (int t = tid; t < (kThreads / 32) * kRadix; t += kThreads) (&s_warp_hist[0][0])[t] = 0;
    __syncthreads();
    const uint32_t part = s_part;
    // device-side count: the grid is sized for a capacity, partitions past the
    // keys present exit (partition ids are handed out in order: the CTAs that
    // stay are exactly partitions 0 .. parts(n) - 1)
    if (n_dev) {
        n = (int64_t)*n_dev;
        if ((int64_t)part * kTileKeys >= n) return;
    }
    // clear this partition's row of the next pass's status buffer (double
    // buffered: no memset between passes; kernel boundaries order it)
    status_next[(size_t)part * kRadix + tid] = 0u;
    const int64_t base = (int64_t)part * kTileKeys + warp * (32 * kItems);

    KeyT k[kItems];
    uint32_t v[kItems], dig[kItems], rank[kItems];
    const uint32_t dmask = (1u << bits) - 1u;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const int64_t idx = base + j * 32 + lane;
        const bool valid = idx < n;
        k[j] = valid ? kin[idx] : (KeyT)0;
        v[j] = valid ? vin[idx] : 0u;
        dig[j] = valid ? ((uint32_t)(k[j] >> shift) & dmask) : 256u;
    }
    // global digit offsets: exclusive scan of this pass's histogram (every CTA
    // redoes it, 256 values from L2, instead of a separate scan launch)
    const uint32_t gofs_d = block_excl_scan_u32(hist[tid], s_ws);
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const uint32_t d = dig[j];
        // warp multi-split (lanes holding the same digit, or 256 = invalid): one ballot
        // per digit bit, except on the key's top pass, whose digits are few within a
        // warp (light distance and tile row are coherent there): match.any, measured
        // faster there and slower on the low digits
        uint32_t peers;
        if (top) {  // uniform
            peers = __match_any_sync(0xffffffffu, d);
        } else {
            const bool inv = d >> 8;
            const uint32_t bv = __ballot_sync(0xffffffffu, inv);
            peers = inv ? bv : ~bv;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (b < bits) {  // uniform
                    const bool bit = (d >> b) & 1u;
                    const uint32_t bb = __ballot_sync(0xffffffffu, bit);
                    peers &= bit ? bb : ~bb;
                }
            }
        }
        uint32_t cnt = 0;
        if (d < 256u) cnt = s_warp_hist[warp][d];
        rank[j] = cnt + __popc(peers & lt);
        __syncwarp();
        if (d < 256u && lane == (__ffs(peers) - 1)) s_warp_hist[warp][d] = cnt + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // per digit: exclusive prefix over warps, partition total
    const uint32_t d = tid;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const uint32_t c = s_warp_hist[w][d];
        s_warp_hist[w][d] = run;
        run += c;
    }
    const uint32_t tile_count = run;

    // decoupled look-back (one thread per digit; digits >= 2^bits never occur)
    volatile uint32_t* st = status;
    if (d > dmask) {
        s_global[d] = 0u;
    } else if (part == 0) {
        st[d] = kFlagInc | tile_count;
        s_global[d] = gofs_d;
    } else {
        st[(size_t)part * kRadix + d] = kFlagAgg | tile_count;
        // look back through a window of predecessors per round trip (wider when
        // the pass has few digits: fewer look-back requests in flight per CTA)
        const uint32_t excl = bits <= DGSM_OS_NARROW_BITS ? look_back<DGSM_OS_WIN_NARROW>(st, part, d)
                                                          : look_back<8>(st, part, d);
        st[(size_t)part * kRadix + d] = kFlagInc | (excl + tile_count);
        s_global[d] = gofs_d + excl;
    }
    s_tile_start[d] = block_excl_scan_u32(tile_count, s_ws);
    __syncthreads();

#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        if (dig[j] < 256u) {
            const uint32_t pos = s_tile_start[dig[j]] + s_warp_hist[warp][dig[j]] + rank[j];
            s_keys[pos] = k[j];
            s_vals[pos] = v[j];
        }
    }
    __syncthreads();
    const int64_t rem = n - (int64_t)part * kTileKeys;
    const int n_valid = rem < kTileKeys ? (int)rem : kTileKeys;
    for (int x = tid; x < n_valid; x += kThreads) {
        const KeyT key = s_keys[x];
        const uint32_t dd = (uint32_t)(key >> shift) & dmask;
        const uint32_t o = s_global[dd] + (uint32_t)x - s_tile_start[dd];
        kout[o] = key;
        vout[o] = s_vals[x];
        if (gdst) gdst[o] = gsrc[s_vals[x]];  // optional gather by the sorted values (last pass)
    }
}

struct OnesweepTemp {
    uint32_t* hist;       // [kMaxPasses][256]
    uint32_t* part_ctr;   // [kMaxPasses]
    uint32_t* status[2];  // [parts][256] each, by pass parity
};

OnesweepTemp carve(void* temp, int64_t parts) {
    OnesweepTemp t;
    char* p = (char*)temp;
    t.hist = (uint32_t*)p; p += sizeof(uint32_t) * kMaxPasses * kRadix;
    t.part_ctr = (uint32_t*)p; p += 256;
    t.status[0] = (uint32_t*)p; p += sizeof(uint32_t) * kRadix * (size_t)parts;
    t.status[1] = (uint32_t*)p;
    return t;
}

template <typename KeyT>
int onesweep_impl(KeyT* keys, uint32_t* vals, KeyT* keys_alt, uint32_t* vals_alt, int64_t n, int nbits,
                  void* temp, cudaStream_t s, int* launches, const uint32_t* gsrc = nullptr,
                  uint32_t* gdst = nullptr, bool hist_ready = false, bool top_match = true,
                  const uint64_t* n_dev = nullptr, const PassDigits* pd_dev = nullptr) {
    // n: the key count, or (n_dev != NULL) the capacity the grid is sized for while
    // the kernels read the count from n_dev (no host synchronisation)
    if (n <= 1 || nbits <= 0) return 0;
    const int passes = (nbits + 7) / 8;
    const int64_t parts = (n + kTileKeys - 1) / kTileKeys;
    OnesweepTemp t = carve(temp, parts);
    // the dynamic shared-memory opt-in is per device: set once for each device used
    static std::atomic<unsigned long long> attr_set{0ull};
    const int dyn = (int)(sizeof(KeyT) + sizeof(uint32_t)) * kTileKeys;
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_set.load() & bit)) {
        cudaFuncSetAttribute(k_pass<KeyT>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        attr_set.fetch_or(bit);
    }
    const PassDigits pd = onesweep_digits(nbits);
    if (!hist_ready) {
        // histograms, partition counters and the first pass's status in one memset
        onesweep_prepare(temp, n, s);
        const int hist_grid = (int)std::min<int64_t>(148 * 4, (n + 2047) / 2048);
        pdl_launch(k_hist<KeyT>, hist_grid, 256, 0, s, keys, n, passes, pd, t.hist, n_dev);
        *launches += 1;
    }
    KeyT *ki = keys, *ko = keys_alt;
    uint32_t *vi = vals, *vo = vals_alt;
    int flipped = 0;
    for (int p = 0; p < passes; ++p) {
        pdl_launch(k_pass<KeyT>, (unsigned)parts, kThreads, dyn, s, ki, vi, ko, vo, n, pd.shift[p], pd.bits[p],
                                                           top_match && p == passes - 1, t.hist + p * kRadix,
                                                           t.status[p & 1], t.status[(p + 1) & 1],
                                                           t.part_ctr + p, gsrc, p == passes - 1 ? gdst : nullptr,
                                                           n_dev, pd_dev, p);
        *launches += 1;
        KeyT* tk = ki; ki = ko; ko = tk;
        uint32_t* tv = vi; vi = vo; vo = tv;
        flipped ^= 1;
    }
    return flipped;
}
}  // namespace

size_t onesweep_temp_bytes(int64_t n_max) {
    const int64_t parts = (n_max + kTileKeys - 1) / kTileKeys;
    return sizeof(uint32_t) * kMaxPasses * kRadix + 256 + 2 * sizeof(uint32_t) * kRadix * (size_t)(parts + 1);
}

int launch_onesweep(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, int64_t n,
                    int nbits, void* temp, cudaStream_t s, int* launches) {
    return onesweep_impl<uint64_t>(keys, vals, keys_alt, vals_alt, n, nbits, temp, s, launches);
}

int launch_onesweep_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                        int nbits, void* temp, cudaStream_t s, int* launches, const uint32_t* gsrc,
                        uint32_t* gdst, bool hist_ready, bool top_match, const uint64_t* n_dev,
                        const PassDigits* pd_dev) {
    return onesweep_impl<uint32_t>(keys, vals, keys_alt, vals_alt, n, nbits, temp, s, launches, gsrc, gdst,
                                   hist_ready, top_match, n_dev, pd_dev);
}

PassDigits onesweep_digits(int nbits) {
    PassDigits pd{};
    pd.passes = nbits > 0 ? (nbits + 7) / 8 : 0;
    for (int p = 0, sh = 0; p < pd.passes; ++p) {
        pd.bits[p] = nbits / pd.passes + (p < nbits % pd.passes ? 1 : 0);
        pd.shift[p] = sh;
        sh += pd.bits[p];
    }
    return pd;
}

uint32_t* onesweep_prepare(void* temp, int64_t n, cudaStream_t s) {
    const int64_t parts = (n + kTileKeys - 1) / kTileKeys;
    OnesweepTemp t = carve(temp, parts);
    cudaMemsetAsync(t.hist, 0, sizeof(uint32_t) * kMaxPasses * kRadix + 256 + sizeof(uint32_t) * kRadix * (size_t)parts,
                    s);
    return t.hist;
}

}  // namespace dgsm
