// dgsm_api.cu — the C ABI of include/dgsm.h: argument validation, workspace
// layout (caller-owned memory only), stream-ordered launches, error strings.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "dgsm_internal.cuh"

using namespace dgsm;

namespace {
thread_local char g_err[512] = "";
thread_local int g_launches = 0;
thread_local cudaEvent_t g_ev_before = nullptr, g_ev_after = nullptr;
// dgsm_frame_host: recorded on the build stream right before the accumulation
// (a5/a6) of the frame being enqueued (nullptr: not recorded)
thread_local cudaEvent_t g_ev_frame_acc = nullptr;
// dgsm_set_frame_event: a caller event recorded (as an external event: a record node
// when the build is captured in a CUDA graph) right before the accumulation
thread_local cudaEvent_t g_ev_frame_ext = nullptr;

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_check(const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(DGSM_ECUDA, "%s: %s", where, cudaGetErrorString(e));
    return DGSM_OK;
}

constexpr size_t kAlign = 256;
constexpr int kChunk = 1024;  // Gaussians per accumulation work unit (512, 768, 1536, 2048 measured slower on cfg2)
#ifndef DGSM_MIN_CHUNK
#define DGSM_MIN_CHUNK 128
#endif
#ifndef DGSM_MIN_UNITS
#define DGSM_MIN_UNITS 2048
#endif
constexpr int kMinChunk = DGSM_MIN_CHUNK;
constexpr int64_t kMinUnits = DGSM_MIN_UNITS;
constexpr int kCounterWords = 8 + 2 * kUnitClasses;  // n_units, unit counter, class histogram + fill

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Carver {
    char* base;
    size_t off = 0;
    explicit Carver(void* b) : base((char*)b) {}
    template <typename T>
    T* take(size_t count) {
        T* p = base ? (T*)(base + off) : nullptr;
        off += align_up(sizeof(T) * (count ? count : 1));
        return p;
    }
};

struct PlanLayout {
    PairRec* recs;
    uint32_t* counts;
    uint4* dup;
    PlanStats* stats;
    size_t bytes;
};

PlanLayout plan_layout(void* ws, int64_t n, int L) {
    Carver c(ws);
    PlanLayout p;
    const int64_t m = (int64_t)L * n;
    p.recs = c.take<PairRec>(m);
    p.counts = c.take<uint32_t>(m);
    p.dup = c.take<uint4>(m);
    p.stats = c.take<PlanStats>(1);
    p.bytes = c.off;
    return p;
}

// What the run's launch sizes and workspace depend on: host-known quantities
// only (the key count P enters as a capacity: P itself for dgsm_build_run,
// the caller's bound for dgsm_build_async).
struct RunShape {
    int64_t n;
    int n_lights, res, K, chunk, tile_bits, light_bits;
    int64_t cap;  // key capacity (>= P for a valid build)
    int depth_bits[DGSM_MAX_LIGHTS];  // significant bits of (D bits - the light's minimum); 32 when unknown
};

// keys per accumulation work unit: kChunk, halved (down to kMinChunk) while the
// build would have fewer than kMinUnits full chunks, so that a small key set (an
// avatar's occluders) still spreads over the ~1600 resident CTAs
int chunk_for(int64_t P) {
    int c = kChunk;
    while (c > kMinChunk && P / c < kMinUnits) c /= 2;
    return c;
}

int bits_for(uint64_t v);

RunShape make_shape(int64_t n, int L, int res, int K, int64_t cap) {
    RunShape sh;
    sh.n = n; sh.n_lights = L; sh.res = res; sh.K = K; sh.cap = cap;
    sh.chunk = chunk_for(cap);
    const int64_t n_tiles = (int64_t)(res / kTile) * (res / kTile);
    sh.tile_bits = bits_for((uint64_t)(n_tiles - 1));
    sh.light_bits = bits_for((uint64_t)(L - 1));
    for (int l = 0; l < DGSM_MAX_LIGHTS; ++l) sh.depth_bits[l] = 32;
    return sh;
}

// The per-light chains before the tile sort (depth keys, depth sort, emission
// offsets, key duplication) are independent: up to kLanes of them run at once on
// side streams (fork / join by events; light l on lane l % kLanes), each lane
// with its own buffers.  One light: lane 0 is the caller's stream itself.
constexpr int kLanes = 4;
struct LaneBufs {
    uint32_t *gkeys_a, *gkeys_b; // per-light depth keys of the N Gaussians, ping-pong
    uint32_t *gvals_a, *gvals_b; // Gaussian indices -> depth-rank permutation
    uint32_t* cperm;             // tile counts in depth-rank order (N)
    uint64_t* offs_perm;         // their exclusive scan (N + 1)
    void* gscan_temp;
    void* sort_temp;             // the depth sort's histograms / partition status (N keys)
};
struct RunLayout {
    uint32_t *keys_a, *keys_b;   // (light | tile) keys (capacity), ping-pong
    uint32_t *vals_a, *vals_b;   // Gaussian indices (capacity)
    LaneBufs lane[kLanes];
    int n_lanes;
    void* sort_temp;             // the tile sort's (capacity keys)
    uint32_t *tile_start, *tile_end;
    uint64_t *unit_cnt, *unit_off;
    void* unit_scan_temp;
    WorkUnit *units, *units_tmp;
    uint32_t* deferred;  // see dgsm_internal.cuh kInlineCombine; count in counters[2]
    uint32_t* counters;  // [0] n_units, [1] unit counter, then the unit class histogram and class fill (kUnitClasses each)
    int64_t zero_words;  // counters .. tile_end, cleared by one memset per run
    uint32_t* tile_arrive;
    uint64_t* n_keys;    // device: the run's key count (P, or 0 on overflow)
    unsigned long long* stats;  // [8] dgsm_build_stats_t words (DGSM_COLLECT_STATS)
    float* scratch;
    size_t bytes;
    uint32_t max_units;
};

RunLayout run_layout(void* ws, const RunShape& sh) {
    Carver c(ws);
    RunLayout r;
    const int64_t P = sh.cap;
    const int64_t nt = (int64_t)sh.n_lights * (sh.res / kTile) * (sh.res / kTile);
    const int64_t n = sh.n;
    r.keys_a = c.take<uint32_t>(P);
    r.keys_b = c.take<uint32_t>(P);
    r.vals_a = c.take<uint32_t>(P);
    r.vals_b = c.take<uint32_t>(P);
    r.n_lanes = std::max(1, std::min(sh.n_lights, kLanes));
    // a lane also runs its lights' tile sorts (planned multi-light builds, run_binning):
    // its sort temp then covers a light's key segment (<= capacity)
    const bool lane_tile_sort = sh.n_lights > 1;
    for (int j = 0; j < r.n_lanes; ++j) {
        LaneBufs& b = r.lane[j];
        b.gkeys_a = c.take<uint32_t>(n);
        b.gkeys_b = c.take<uint32_t>(n);
        b.gvals_a = c.take<uint32_t>(n);
        b.gvals_b = c.take<uint32_t>(n);
        b.cperm = c.take<uint32_t>(n);
        b.offs_perm = c.take<uint64_t>(n + 1);
        b.gscan_temp = c.take<char>(scan_u32_to_u64_temp_bytes(n));
        b.sort_temp = c.take<char>(onesweep_temp_bytes(lane_tile_sort ? std::max<int64_t>(P, n) : n));
    }
    r.sort_temp = c.take<char>(onesweep_temp_bytes(std::max<int64_t>(P, n)));

    r.unit_cnt = c.take<uint64_t>(nt);
    r.unit_off = c.take<uint64_t>(nt + 1);
    r.unit_scan_temp = c.take<char>(scan_u32_to_u64_temp_bytes(nt));
    const int64_t max_units = kTileSplit * (nt + P / sh.chunk + 1);
    r.max_units = (uint32_t)max_units;
    r.units = c.take<WorkUnit>(max_units);
    r.units_tmp = c.take<WorkUnit>(max_units);
    r.deferred = c.take<uint32_t>(nt);  // units[] positions of the tiles k_combine_deferred sums
    // zeroed together at the start of a run: counters, arrival counters, tile ranges
    r.counters = c.take<uint32_t>(kCounterWords + kTileSplit * nt + 2 * nt);
    r.tile_arrive = r.counters + kCounterWords;
    r.tile_start = r.tile_arrive + kTileSplit * nt;
    r.tile_end = r.tile_start + nt;
    r.zero_words = kCounterWords + (kTileSplit + 2) * nt;
    r.n_keys = c.take<uint64_t>(2);
    r.stats = c.take<unsigned long long>(8);
    const int64_t max_slots = kTileSplit * (2 * (P / sh.chunk) + 1);
    r.scratch = c.take<float>((size_t)max_slots * sh.K * (kTexels / kTileSplit));
    r.bytes = c.off;
    return r;
}

RunShape plan_shape(const dgsm_plan_t& pl) {
    RunShape sh = make_shape(pl.n, pl.n_lights, pl.atlas_res, pl.n_shells, pl.n_keys);
    sh.chunk = pl.chunk;
    // the plan read the depth range back: sort only its significant bits (fewer digits per pass)
    for (int l = 0; l < pl.n_lights; ++l) sh.depth_bits[l] = pl.depth_bits[l];
    return sh;
}

int bits_for(uint64_t v) {  // bits needed to represent 0..v
    int b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

uint64_t signature(const dgsm_gaussians_t* g, int L, int res, int K, const dgsm_build_opts_t& o,
                   const dgsm_light_t* lights) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* p, size_t n) {
        const unsigned char* b = (const unsigned char*)p;
        for (size_t i = 0; i < n; ++i) { h ^= b[i]; h *= 1099511628211ull; }
    };
    mix(&g->n, sizeof(g->n));
    mix(&g->means, sizeof(void*) * 4);
    mix(&L, sizeof(L)); mix(&res, sizeof(res)); mix(&K, sizeof(K));
    mix(&o, sizeof(o));
    mix(lights, sizeof(dgsm_light_t) * (size_t)L);
    return h;
}

int validate(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int L, int res, int K,
             const dgsm_build_opts_t& o) {
    if (!g || !lights) return fail(DGSM_EINVAL, "null gaussians or lights");
    if (g->n < 0) return fail(DGSM_EINVAL, "n < 0");
    if (g->n > 0 && (!g->means || !g->scales || !g->rotations || !g->opacities))
        return fail(DGSM_EINVAL, "null Gaussian array");
    // the depth sort runs over all n Gaussians of a light: its look-back status
    // words hold 30-bit counts (onesweep.cu)
    if (g->n >= (int64_t)1 << 30) return fail(DGSM_ERANGE, "n >= 2^30");
    if (L < 1 || L > DGSM_MAX_LIGHTS) return fail(DGSM_EINVAL, "n_lights %d outside [1, %d]", L, DGSM_MAX_LIGHTS);
    if (res < 8 || res % 8 != 0 || res > 2048) return fail(DGSM_EINVAL, "atlas_res %d: need 8..2048, multiple of 8", res);
    if (K < 1 || K > DGSM_MAX_SHELLS) return fail(DGSM_EINVAL, "n_shells %d outside [1, %d]", K, DGSM_MAX_SHELLS);
    for (int l = 0; l < L; ++l)
        if (!(lights[l].t_max > 0.0f)) return fail(DGSM_EINVAL, "light %d: t_max <= 0", l);
    if (!(o.kappa > 0.0f) || !(o.k_sigma > 0.0f) || !(o.rho_scale > 0.0f))
        return fail(DGSM_EINVAL, "kappa, k_sigma, rho_scale must be > 0");
    if (o.bin_mode != DGSM_BIN_WRAP && o.bin_mode != DGSM_BIN_CLAMP) return fail(DGSM_EINVAL, "bad bin_mode");
    if (o.flags & ~(DGSM_OUTPUT_TAU | DGSM_COLLECT_STATS | DGSM_NO_TILE_CULL | DGSM_VALIDATE))
        return fail(DGSM_EINVAL, "unknown flags");
    if (o.absorption < DGSM_ABS_TRACEAVG || o.absorption > DGSM_ABS_DIAG) return fail(DGSM_EINVAL, "bad absorption");
    if ((uintptr_t)o.slab % 8) return fail(DGSM_EINVAL, "slab not 8-B aligned");
    return DGSM_OK;
}

LightsParam lights_param(const dgsm_light_t* lights, int L) {
    LightsParam lp;
    memset(&lp, 0, sizeof(lp));
    for (int l = 0; l < L; ++l)
        lp.l[l] = make_float4(lights[l].position[0], lights[l].position[1], lights[l].position[2],
                              lights[l].t_max);
    return lp;
}
}  // namespace

extern "C" {

void dgsm_default_opts(dgsm_build_opts_t* o) {
    if (!o) return;
    o->kappa = 1.0f;
    o->k_sigma = 3.0f;
    o->rho_scale = 1.0f;
    o->bin_mode = DGSM_BIN_WRAP;
    o->flags = 0u;
    o->absorption = DGSM_ABS_TRACEAVG;
    o->slab = nullptr;
}

size_t dgsm_slab_bytes(int n_lights, int atlas_res) {
    if (n_lights < 1 || n_lights > DGSM_MAX_LIGHTS || atlas_res < 8 || atlas_res % 8 || atlas_res > 2048) return 0;
    return slab_mask_bytes(n_lights, atlas_res) + sizeof(int2) * (size_t)n_lights;
}

int dgsm_active_slab(const float* receivers, int64_t m, const dgsm_roi_t* roi, const dgsm_light_t* lights,
                     int n_lights, int atlas_res, int n_shells, void* slab, size_t slab_bytes, void* stream) {
    g_launches = 0;
    if (!roi || !lights || !slab) return fail(DGSM_EINVAL, "null roi, lights or slab");
    if (n_lights < 1 || n_lights > DGSM_MAX_LIGHTS) return fail(DGSM_EINVAL, "n_lights %d outside [1, %d]", n_lights, DGSM_MAX_LIGHTS);
    if (atlas_res < 8 || atlas_res % 8 != 0 || atlas_res > 2048) return fail(DGSM_EINVAL, "bad atlas_res %d", atlas_res);
    if (n_shells < 1 || n_shells > DGSM_MAX_SHELLS) return fail(DGSM_EINVAL, "bad n_shells %d", n_shells);
    if (m < 0 || (m > 0 && !receivers)) return fail(DGSM_EINVAL, "bad receivers");
    if (!(roi->radius > 0.0f) || !(roi->z_min <= roi->z_max)) return fail(DGSM_EINVAL, "roi: need radius > 0, z_min <= z_max");
    for (int l = 0; l < n_lights; ++l)
        if (!(lights[l].t_max > 0.0f)) return fail(DGSM_EINVAL, "light %d: t_max <= 0", l);
    if ((uintptr_t)slab % 256) return fail(DGSM_EINVAL, "slab not 256-B aligned");
    const size_t need = dgsm_slab_bytes(n_lights, atlas_res);
    if (slab_bytes < need) return fail(DGSM_ENOSPC, "slab %zu < %zu bytes", slab_bytes, need);
    const LightsParam lp = lights_param(lights, n_lights);
    launch_active_slab(receivers, m, *roi, lp, n_lights, atlas_res, n_shells, (uint64_t*)slab,
                       (int2*)((char*)slab + slab_mask_bytes(n_lights, atlas_res)), (cudaStream_t)stream,
                       &g_launches);
    return cuda_check("active slab");
}

size_t dgsm_plan_workspace_bytes(int64_t n, int n_lights) {
    if (n < 0 || n_lights < 1) return 0;
    return plan_layout(nullptr, n, n_lights).bytes;
}

// Upload pipeline depth of dgsm_frame_host (chunks of the Gaussian arrays): the
// projection of chunk c starts when it has landed.  Frames back to back (each
// frame's uploads overlapping the previous build) measured 1.50 / 1.51 / 1.53
// ms per frame with 1 / 2 / 4 chunks; 2 keeps an isolated frame's upload and
// projection overlapped.
#ifndef DGSM_UPLOAD_CHUNKS
#define DGSM_UPLOAD_CHUNKS 2
#endif
constexpr int kUploadChunks = DGSM_UPLOAD_CHUNKS;

// A copy stream + events per (thread, device) for the host-buffer entry point.
struct CopyStream {
    cudaStream_t st = nullptr;
    cudaEvent_t start = nullptr, done = nullptr;
    // end of the last frame that used a workspace (by workspace address): a
    // frame's uploads wait only for the previous frame in the SAME workspace, so
    // a caller alternating two workspaces overlaps frame i+1's uploads with
    // frame i's build (the layout may shift with n, m: the whole frame must be done)
    void* slot_ws[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t slot_ev[4];
    int slot_next = 0;
    cudaEvent_t chunk[kUploadChunks];
    // the accumulation of the last frame enqueued: the next frame's uploads start
    // there (overlapping the FP32-bound a6 kernel, not the L2-resident sorts, which a
    // concurrent 60 MB upload slowed by 28 %: tools/e2e_probe3.py).  cfg2 frames back
    // to back: 1.51-1.65 -> 1.50-1.51 ms (recording it before the tile sort instead: same)
    cudaEvent_t acc = nullptr;
    bool acc_valid = false;
    int dev = -1;
};
static CopyStream& copy_stream() {
    thread_local CopyStream cs;
    int dev = 0;
    cudaGetDevice(&dev);
    if (cs.dev != dev) {
        cudaStreamCreateWithFlags(&cs.st, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&cs.start, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&cs.done, cudaEventDisableTiming);
        for (int i = 0; i < 4; ++i) {
            cudaEventCreateWithFlags(&cs.slot_ev[i], cudaEventDisableTiming);
            cs.slot_ws[i] = nullptr;
        }
        for (int i = 0; i < kUploadChunks; ++i) cudaEventCreateWithFlags(&cs.chunk[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&cs.acc, cudaEventDisableTiming);
        cs.acc_valid = false;
        cs.dev = dev;
    }
    return cs;
}

// The plan's kernels (a1, a2 and the key-count scan) on stream s, no
// synchronisation; with g_host != NULL the Gaussian arrays are first uploaded
// from host memory into the device arrays of g in n_chunks pieces, each
// projected as soon as it has landed (copy engine and SMs overlap).
static void enqueue_plan(const dgsm_gaussians_t* g, const dgsm_gaussians_t* g_host, int n_chunks,
                         cudaEvent_t upload_after, const dgsm_light_t* lights, int n_lights, int atlas_res,
                         int n_shells, const dgsm_build_opts_t& o, const PlanLayout& p, cudaStream_t s) {
    const LightsParam lp = lights_param(lights, n_lights);

    launch_project_init(p.stats, s);
    if (g_host && g->n > 0) {
        // chunks are copied on the copy stream, each projected on `s` as soon as it
        // has landed (copy engine and SMs overlap); the copy stream first waits for
        // the work already queued on `s` (the device arrays may still be in use)
        CopyStream& cs = copy_stream();
        if (upload_after) cudaStreamWaitEvent(cs.st, upload_after, 0);  // the workspace's previous frame is done
        if (cs.acc_valid) cudaStreamWaitEvent(cs.st, cs.acc, 0);       // the previous frame's a6 has started
        const int64_t n = g->n, per = (n + n_chunks - 1) / n_chunks;
        int c = 0;
        for (int64_t i0 = 0; i0 < n; i0 += per, ++c) {
            const int64_t cnt = std::min<int64_t>(per, n - i0);
            cudaMemcpyAsync((float*)g->means + 3 * i0, g_host->means + 3 * i0, 12 * cnt, cudaMemcpyHostToDevice, cs.st);
            cudaMemcpyAsync((float*)g->scales + 3 * i0, g_host->scales + 3 * i0, 12 * cnt, cudaMemcpyHostToDevice, cs.st);
            cudaMemcpyAsync((float*)g->rotations + 4 * i0, g_host->rotations + 4 * i0, 16 * cnt,
                            cudaMemcpyHostToDevice, cs.st);
            cudaMemcpyAsync((float*)g->opacities + i0, g_host->opacities + i0, 4 * cnt, cudaMemcpyHostToDevice, cs.st);
            cudaEventRecord(cs.chunk[c], cs.st);
            cudaStreamWaitEvent(s, cs.chunk[c], 0);
            launch_project(*g, lp, n_lights, atlas_res, n_shells, o, i0, cnt, p.recs, p.counts, p.dup, p.stats, s);
            g_launches += 1;
        }
    } else {
        launch_project(*g, lp, n_lights, atlas_res, n_shells, o, 0, g->n, p.recs, p.counts, p.dup, p.stats, s);
        g_launches += 1;
    }
    // the light segments' key begins (per-light totals of the counts) into the plan stats
    launch_light_begin(p.counts, g->n, n_lights, p.stats->light_key_begin, s);
    g_launches += 2;  // init, totals
}

// The plan; with g_host != NULL the Gaussian arrays are first uploaded from
// host memory into the device arrays of g in n_chunks pieces, each projected
// as soon as it has landed (copy engine and SMs overlap).
static int plan_impl(const dgsm_gaussians_t* g, const dgsm_gaussians_t* g_host, int n_chunks,
                     cudaEvent_t upload_after, const dgsm_light_t* lights, int n_lights, int atlas_res,
                     int n_shells, const dgsm_build_opts_t* opts, void* plan_ws, size_t plan_ws_bytes,
                     dgsm_plan_t* plan, void* stream);

int dgsm_build_plan(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights, int atlas_res,
                    int n_shells, const dgsm_build_opts_t* opts, void* plan_ws, size_t plan_ws_bytes,
                    dgsm_plan_t* plan, void* stream) {
    return plan_impl(g, nullptr, 1, nullptr, lights, n_lights, atlas_res, n_shells, opts, plan_ws, plan_ws_bytes,
                     plan, stream);
}

static int plan_impl(const dgsm_gaussians_t* g, const dgsm_gaussians_t* g_host, int n_chunks,
                     cudaEvent_t upload_after, const dgsm_light_t* lights, int n_lights, int atlas_res,
                     int n_shells, const dgsm_build_opts_t* opts, void* plan_ws, size_t plan_ws_bytes,
                     dgsm_plan_t* plan, void* stream) {
    g_launches = 0;
    dgsm_build_opts_t o;
    if (opts) o = *opts; else dgsm_default_opts(&o);
    int rc = validate(g, lights, n_lights, atlas_res, n_shells, o);
    if (rc) return rc;
    if (!plan || !plan_ws) return fail(DGSM_EINVAL, "null plan or plan workspace");
    if ((uintptr_t)plan_ws % kAlign) return fail(DGSM_EINVAL, "plan workspace not 256-B aligned");
    const size_t need = plan_layout(nullptr, g->n, n_lights).bytes;
    if (plan_ws_bytes < need) return fail(DGSM_ENOSPC, "plan workspace %zu < %zu bytes", plan_ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    PlanLayout p = plan_layout(plan_ws, g->n, n_lights);
    enqueue_plan(g, g_host, n_chunks, upload_after, lights, n_lights, atlas_res, n_shells, o, p, s);
    if ((rc = cuda_check("plan launch"))) return rc;
    PlanStats hs;
    cudaMemcpyAsync(&hs, p.stats, sizeof(PlanStats), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_check("plan sync");

    if (hs.n_invalid)
        return fail(DGSM_EDATA, "%u invalid Gaussians (non-finite mean / scale / rotation / opacity, scale <= 0 "
                                "or zero quaternion), the first at index %u", hs.n_invalid, hs.first_invalid);
    memset(plan, 0, sizeof(*plan));
    plan->n = g->n;
    plan->n_lights = n_lights;
    plan->atlas_res = atlas_res;
    plan->n_shells = n_shells;
    plan->n_keys = (int64_t)hs.light_key_begin[n_lights];
    // keys per accumulation work unit: kChunk, halved (down to kMinChunk) while
    // the build would have fewer than kMinUnits full chunks, so that a small key
    // set (an avatar's occluders) still spreads over the ~1600 resident CTAs
    plan->chunk = chunk_for(plan->n_keys);
    const int64_t n_tiles = (int64_t)(atlas_res / kTile) * (atlas_res / kTile);
    plan->tile_bits = bits_for((uint64_t)(n_tiles - 1));
    for (int l = 0; l <= n_lights; ++l) plan->light_key_begin[l] = (int64_t)hs.light_key_begin[l];
    for (int l = 0; l < n_lights; ++l) {
        const int64_t pl = plan->light_key_begin[l + 1] - plan->light_key_begin[l];
        plan->depth_min[l] = pl ? hs.depth_min[l] : 0u;
        plan->depth_max[l] = pl ? hs.depth_max[l] : 0u;
        plan->depth_bits[l] = pl ? bits_for((uint64_t)(hs.depth_max[l] - hs.depth_min[l])) : 0;
    }
    // one onesweep sorts all lights' keys: its look-back status words hold 30-bit counts
    if (plan->n_keys >= ((int64_t)1 << 30)) return fail(DGSM_ERANGE, "%lld keys (>= 2^30)", (long long)plan->n_keys);
    plan->run_workspace_bytes = run_layout(nullptr, plan_shape(*plan)).bytes;
    plan->signature = signature(g, n_lights, atlas_res, n_shells, o, lights);
    return DGSM_OK;
}

static int check_run_args(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights,
                          const dgsm_build_opts_t& o, const dgsm_plan_t* plan, void* plan_ws,
                          size_t plan_ws_bytes, void* run_ws, size_t run_ws_bytes) {
    if (!plan) return fail(DGSM_EINVAL, "null plan");
    int rc = validate(g, lights, n_lights, plan->atlas_res, plan->n_shells, o);
    if (rc) return rc;
    if (plan->signature != signature(g, n_lights, plan->atlas_res, plan->n_shells, o, lights))
        return fail(DGSM_EINVAL, "plan does not match these arguments");
    if (!plan_ws) return fail(DGSM_EINVAL, "null plan workspace");
    if (plan_ws_bytes < plan_layout(nullptr, g->n, n_lights).bytes) return fail(DGSM_ENOSPC, "plan workspace too small");
    if (plan->run_workspace_bytes > 0 && (!run_ws || run_ws_bytes < plan->run_workspace_bytes))
        return fail(DGSM_ENOSPC, "run workspace %zu < %zu bytes", run_ws_bytes, plan->run_workspace_bytes);
    if ((uintptr_t)run_ws % kAlign) return fail(DGSM_EINVAL, "run workspace not 256-B aligned");
    return DGSM_OK;
}

// a3-a5: per light, the depth sort of its N Gaussians (low LSD digits: fp32 bits
// of D) and the key duplication in depth-rank order into the light's key
// segment; then ONE stable onesweep of all lights' (light | tile) keys and the
// tile ranges.  Every count that depends on the build (P, the per-light key
// segments, the depth minimum) is read on the device: no host synchronisation.
// Returns the sorted (key, Gaussian index) arrays.
struct Sorted {
    const uint32_t *keys, *vals;
};

// Side streams + events of the per-light lanes, per (thread, device).
struct LaneStreams {
    cudaStream_t st[kLanes];
    cudaEvent_t fork, done[kLanes];
    int dev = -1;
};
static LaneStreams& lane_streams() {
    thread_local LaneStreams ls;
    int dev = 0;
    cudaGetDevice(&dev);
    if (ls.dev != dev) {
        for (int j = 0; j < kLanes; ++j) {
            cudaStreamCreateWithFlags(&ls.st[j], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&ls.done[j], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&ls.fork, cudaEventDisableTiming);
        ls.dev = dev;
    }
    return ls;
}

static Sorted run_binning(const dgsm_gaussians_t* g, const dgsm_build_opts_t& o, const RunShape& sh,
                          const PlanLayout& p, const RunLayout& r, dgsm_build_status_t* status, cudaStream_t s,
                          const int64_t* key_begin_host = nullptr) {
    const int res = sh.res;
    const int64_t n = g->n;
    const int64_t n_tiles = (int64_t)(res / kTile) * (res / kTile);
    // (tile ranges zeroed by the caller's run memset)
    // (sync-free builds: the depth digits are planned on the device from the plan's depth range)
    bool dev_digits = false;
    for (int l = 0; l < sh.n_lights; ++l) dev_digits |= sh.depth_bits[l] == 32;
    launch_run_setup(p.stats, sh.n_lights, (uint64_t)sh.cap, r.n_keys, status, s,
                     dev_digits ? onesweep_digits(32).passes : 0);
    g_launches += 1;
    PassDigits pd0 = onesweep_digits(32);
    pd0.passes = 0;
    // the tile sort per light segment when the host knows the segments (the planned
    // build; the keys are emitted grouped by light): in the light's lane, right after
    // its duplication.  cfg5: 3 + 16 bits = 3 passes over all keys, 16 bits = 2 per light
    const int tb = sh.tile_bits;
    // (also when it saves no pass: cfg3's 2 + 14 bits, 2 passes either way, 8.58 -> 8.47 ms
    // from the lanes' overlap)
    const bool per_light_sort = key_begin_host && sh.n_lights > 1;
    const int target = onesweep_digits(tb).passes & 1;  // where a sorted segment of > 1 key ends
    LaneStreams* ls = nullptr;
    if (r.n_lanes > 1) {  // fork: the lanes start after everything queued on s
        ls = &lane_streams();
        cudaEventRecord(ls->fork, s);
        for (int j = 0; j < r.n_lanes; ++j) cudaStreamWaitEvent(ls->st[j], ls->fork, 0);
    }
    for (int l = 0; l < sh.n_lights; ++l) {
        const LaneBufs& lb = r.lane[l % r.n_lanes];
        const cudaStream_t ss = ls ? ls->st[l % r.n_lanes] : s;
        const uint4* dup = p.dup + (int64_t)l * n;
        const uint32_t* counts_l = p.counts + (int64_t)l * n;
        const uint32_t* perm = lb.gvals_a;
        const int db = sh.depth_bits[l];
        if (n > 1 && db > 0) {
            const PassDigits pd = onesweep_digits(db);
            // 1. light-distance digits on the Gaussians (the key kernel fills the sort's
            //    digit histograms; the sort's last pass gathers the key counts into
            //    depth-rank order)
            uint32_t* hist = onesweep_prepare(lb.sort_temp, n, ss);
            const PassDigits* pd_dev = db == 32 ? p.stats->depth_pd + l : nullptr;
            launch_depth_keys(dup, n, p.stats->depth_min + l, lb.gkeys_a, lb.gvals_a, pd, hist, ss, pd_dev);
            const int fl = launch_onesweep_u32(lb.gkeys_a, lb.gvals_a, lb.gkeys_b, lb.gvals_b, n, db, lb.sort_temp, ss,
                                               &g_launches, counts_l, lb.cperm, true, true, nullptr, pd_dev);
            perm = fl ? lb.gvals_b : lb.gvals_a;
            g_launches += 1;
        } else {
            launch_depth_keys(dup, n, p.stats->depth_min + l, lb.gkeys_a, lb.gvals_a, pd0, nullptr, ss);
            launch_gather_counts(counts_l, lb.gvals_a, n, lb.cperm, ss);
            g_launches += 2;
        }
        // 2. emission offsets in depth-rank order
        launch_scan_u32_to_u64(lb.cperm, lb.offs_perm, n, lb.gscan_temp, ss);
        // 3. key duplication (key = light | tile, value = Gaussian index) into the light's segment
        const uint64_t* tm = o.slab ? slab_mask_ptr(o.slab) + (int64_t)l * n_tiles : nullptr;
        launch_duplicate_ranked(dup, perm, lb.offs_perm, n, res, o.bin_mode, p.stats->light_key_begin + l, r.n_keys,
                                (uint32_t)l << sh.tile_bits, tm, r.keys_a, r.vals_a, ss);
        g_launches += kScanLaunches + 1;
        if (per_light_sort) {
            const int64_t b = key_begin_host[l], nl = key_begin_host[l + 1] - key_begin_host[l];
            if (nl > 0) {
                const int fl = launch_onesweep_u32(r.keys_a + b, r.vals_a + b, r.keys_b + b, r.vals_b + b, nl, tb,
                                                   lb.sort_temp, ss, &g_launches);
                if (fl != target) {  // (a segment of one key: no pass ran)
                    cudaMemcpyAsync((target ? r.keys_b : r.keys_a) + b, (fl ? r.keys_b : r.keys_a) + b, 4 * nl,
                                    cudaMemcpyDeviceToDevice, ss);
                    cudaMemcpyAsync((target ? r.vals_b : r.vals_a) + b, (fl ? r.vals_b : r.vals_a) + b, 4 * nl,
                                    cudaMemcpyDeviceToDevice, ss);
                }
            }
        }
    }
    if (ls) {  // join
        for (int j = 0; j < r.n_lanes; ++j) {
            cudaEventRecord(ls->done[j], ls->st[j]);
            cudaStreamWaitEvent(s, ls->done[j], 0);
        }
    }
    // 4. one stable sort of the (light | tile) digits of all keys (grid: the capacity),
    //    unless the lanes sorted each light's segment above
    int ft = target;
    if (!per_light_sort)
        ft = launch_onesweep_u32(r.keys_a, r.vals_a, r.keys_b, r.vals_b, sh.cap, sh.light_bits + tb, r.sort_temp, s,
                                 &g_launches, nullptr, nullptr, false, true, r.n_keys);
    Sorted out{ft ? r.keys_b : r.keys_a, ft ? r.vals_b : r.vals_a};
    // 5. tile ranges
    launch_ranges(out.keys, r.n_keys, sh.cap, sh.tile_bits, (uint32_t)n_tiles, r.tile_start, r.tile_end, s);
    g_launches += 1;
    return out;
}

// a5 work units + a6 accumulation (+ Eq.4) of a run whose binning is done.
static void run_accumulate(const dgsm_gaussians_t* g, const dgsm_light_t* lights, const dgsm_build_opts_t& o,
                           const RunShape& sh, const PlanLayout& p, const RunLayout& r, const Sorted& so,
                           float* atlas_out, cudaStream_t s) {
    const LightsParam lp = lights_param(lights, sh.n_lights);
    const int64_t nt = sh.n_lights * (int64_t)(sh.res / kTile) * (sh.res / kTile);
    if (g_ev_frame_acc) cudaEventRecord(g_ev_frame_acc, s);
    if (g_ev_frame_ext) cudaEventRecordWithFlags(g_ev_frame_ext, s, cudaEventRecordExternal);
    launch_units(r.tile_start, r.tile_end, nt, sh.chunk, r.unit_cnt, r.unit_off, r.unit_scan_temp, r.units_tmp,
                 r.units, r.max_units, r.counters, r.counters + 8, r.counters + 8 + kUnitClasses, r.deferred,
                 r.counters + 2, s, &g_launches);
    if (o.flags & DGSM_COLLECT_STATS) cudaMemsetAsync(r.stats, 0, sizeof(unsigned long long) * 8, s);
    launch_accumulate(r.units, r.counters, r.max_units, so.vals, p.recs, g->n, lp, sh.n_lights, sh.res, sh.K,
                      o.flags, r.scratch, r.tile_arrive, r.counters + 1, atlas_out, r.stats, slab_mask_ptr(o.slab),
                      slab_k_ptr(o.slab, sh.n_lights, sh.res), r.deferred, r.counters + 2, g_ev_before, g_ev_after, s);
    g_launches += 2;  // accumulate + deferred combine
}

int dgsm_build_run(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights,
                   const dgsm_build_opts_t* opts, const dgsm_plan_t* plan, void* plan_ws,
                   size_t plan_ws_bytes, void* run_ws, size_t run_ws_bytes, float* atlas_out, void* stream) {
    g_launches = 0;
    dgsm_build_opts_t o;
    if (opts) o = *opts; else dgsm_default_opts(&o);
    int rc = check_run_args(g, lights, n_lights, o, plan, plan_ws, plan_ws_bytes, run_ws, run_ws_bytes);
    if (rc) return rc;
    if (!atlas_out) return fail(DGSM_EINVAL, "null atlas");
    cudaStream_t s = (cudaStream_t)stream;
    const RunShape sh = plan_shape(*plan);
    const PlanLayout p = plan_layout(plan_ws, g->n, n_lights);
    const RunLayout r = run_layout(run_ws, sh);
    cudaMemsetAsync(r.counters, 0, sizeof(uint32_t) * r.zero_words, s);
    const Sorted so = run_binning(g, o, sh, p, r, nullptr, s, plan->light_key_begin);
    run_accumulate(g, lights, o, sh, p, r, so, atlas_out, s);
    return cuda_check("build run");
}

int dgsm_build_bins(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights,
                    const dgsm_build_opts_t* opts, const dgsm_plan_t* plan, void* plan_ws,
                    size_t plan_ws_bytes, void* run_ws, size_t run_ws_bytes, uint32_t* light_out,
                    uint32_t* tile_out, uint32_t* depth_bits_out, uint32_t* index_out,
                    uint32_t* tile_start_out, uint32_t* tile_end_out, void* stream) {
    g_launches = 0;
    dgsm_build_opts_t o;
    if (opts) o = *opts; else dgsm_default_opts(&o);
    int rc = check_run_args(g, lights, n_lights, o, plan, plan_ws, plan_ws_bytes, run_ws, run_ws_bytes);
    if (rc) return rc;
    if (plan->n_keys > 0 && (!light_out || !tile_out || !depth_bits_out || !index_out))
        return fail(DGSM_EINVAL, "null output array");
    cudaStream_t s = (cudaStream_t)stream;
    const PlanLayout p = plan_layout(plan_ws, g->n, n_lights);
    const RunShape sh = plan_shape(*plan);
    const RunLayout r = run_layout(run_ws, sh);
    const int res = plan->atlas_res;
    const int64_t nt = n_lights * (int64_t)(res / kTile) * (res / kTile);
    cudaMemsetAsync(r.counters, 0, sizeof(uint32_t) * r.zero_words, s);
    const Sorted so = run_binning(g, o, sh, p, r, nullptr, s, plan->light_key_begin);
    launch_decode_keys(so.keys, so.vals, p.dup, *plan, light_out, tile_out, depth_bits_out, index_out, s);
    g_launches += 1;
    if (tile_start_out) cudaMemcpyAsync(tile_start_out, r.tile_start, sizeof(uint32_t) * nt, cudaMemcpyDeviceToDevice, s);
    if (tile_end_out) cudaMemcpyAsync(tile_end_out, r.tile_end, sizeof(uint32_t) * nt, cudaMemcpyDeviceToDevice, s);
    return cuda_check("build bins");
}

int dgsm_build(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights, int atlas_res,
               int n_shells, const dgsm_build_opts_t* opts, void* ws, size_t ws_bytes, size_t* ws_required,
               float* atlas_out, void* stream) {
    if (!g) return fail(DGSM_EINVAL, "null gaussians");
    const size_t pb = dgsm_plan_workspace_bytes(g->n, n_lights);
    if (ws_bytes < pb) {
        if (ws_required) *ws_required = pb;
        return fail(DGSM_ENOSPC, "workspace %zu < plan size %zu", ws_bytes, pb);
    }
    dgsm_plan_t plan;
    int rc = dgsm_build_plan(g, lights, n_lights, atlas_res, n_shells, opts, ws, pb, &plan, stream);
    if (rc) return rc;
    const int plan_launches = g_launches;
    const size_t need = pb + plan.run_workspace_bytes;
    if (ws_required) *ws_required = need;
    if (ws_bytes < need) return fail(DGSM_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, need);
    rc = dgsm_build_run(g, lights, n_lights, opts, &plan, ws, pb, (char*)ws + pb, ws_bytes - pb, atlas_out,
                        stream);
    g_launches += plan_launches;
    return rc;
}

size_t dgsm_async_workspace_bytes(int64_t n, int n_lights, int atlas_res, int n_shells, int64_t key_capacity) {
    if (n < 0 || n_lights < 1 || n_lights > DGSM_MAX_LIGHTS || atlas_res < 8 || atlas_res % 8 || atlas_res > 2048 ||
        n_shells < 1 || n_shells > DGSM_MAX_SHELLS || key_capacity < 1 || key_capacity >= ((int64_t)1 << 30))
        return 0;
    return plan_layout(nullptr, n, n_lights).bytes + run_layout(nullptr, make_shape(n, n_lights, atlas_res, n_shells,
                                                                                   key_capacity)).bytes;
}

int dgsm_build_async(const dgsm_gaussians_t* g, const dgsm_light_t* lights, int n_lights, int atlas_res,
                     int n_shells, const dgsm_build_opts_t* opts, int64_t key_capacity, void* ws, size_t ws_bytes,
                     float* atlas_out, dgsm_build_status_t* status, void* stream) {
    g_launches = 0;
    dgsm_build_opts_t o;
    if (opts) o = *opts; else dgsm_default_opts(&o);
    int rc = validate(g, lights, n_lights, atlas_res, n_shells, o);
    if (rc) return rc;
    if (o.flags & DGSM_COLLECT_STATS) return fail(DGSM_EINVAL, "DGSM_COLLECT_STATS needs dgsm_build_plan/run");
    if (!atlas_out || !status || !ws) return fail(DGSM_EINVAL, "null atlas, status or workspace");
    if (key_capacity < 1 || key_capacity >= ((int64_t)1 << 30))
        return fail(DGSM_EINVAL, "key_capacity %lld outside [1, 2^30 - 1]", (long long)key_capacity);
    if ((uintptr_t)ws % kAlign) return fail(DGSM_EINVAL, "workspace not 256-B aligned");
    const size_t need = dgsm_async_workspace_bytes(g->n, n_lights, atlas_res, n_shells, key_capacity);
    if (ws_bytes < need) return fail(DGSM_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    const PlanLayout p = plan_layout(ws, g->n, n_lights);
    const RunShape sh = make_shape(g->n, n_lights, atlas_res, n_shells, key_capacity);
    const RunLayout r = run_layout((char*)ws + p.bytes, sh);
    enqueue_plan(g, nullptr, 1, nullptr, lights, n_lights, atlas_res, n_shells, o, p, s);
    cudaMemsetAsync(r.counters, 0, sizeof(uint32_t) * r.zero_words, s);
    const Sorted so = run_binning(g, o, sh, p, r, status, s);
    run_accumulate(g, lights, o, sh, p, r, so, atlas_out, s);
    return cuda_check("build async");
}

int dgsm_frame_host(const dgsm_gaussians_t* g_host, const dgsm_light_t* lights, int n_lights, int atlas_res,
                    int n_shells, const dgsm_build_opts_t* opts, const float* receivers_host, int64_t m,
                    float* T_host, void* ws, size_t ws_bytes, size_t* ws_required, float* atlas_out,
                    void* stream) {
    if (!g_host) return fail(DGSM_EINVAL, "null gaussians");
    const int64_t n = g_host->n;
    if (n < 0 || m < 0) return fail(DGSM_EINVAL, "n < 0 or m < 0");
    if (n > 0 && (!g_host->means || !g_host->scales || !g_host->rotations || !g_host->opacities))
        return fail(DGSM_EINVAL, "null host Gaussian array");
    if (m > 0 && (!receivers_host || !T_host)) return fail(DGSM_EINVAL, "null receivers or T");
    if (!atlas_out) return fail(DGSM_EINVAL, "null atlas");
    if (n_lights < 1 || n_lights > DGSM_MAX_LIGHTS) return fail(DGSM_EINVAL, "n_lights %d outside [1, %d]", n_lights, DGSM_MAX_LIGHTS);
    if ((uintptr_t)ws % kAlign) return fail(DGSM_EINVAL, "workspace not 256-B aligned");
    Carver c(ws);
    dgsm_gaussians_t gd;
    gd.means = c.take<float>(3 * n);
    gd.scales = c.take<float>(3 * n);
    gd.rotations = c.take<float>(4 * n);
    gd.opacities = c.take<float>(n);
    gd.n = n;
    float* rec = c.take<float>(3 * m);
    float* Td = c.take<float>(m);
    const size_t fixed = c.off;
    const size_t pb = dgsm_plan_workspace_bytes(n, n_lights);
    if (ws_required) *ws_required = fixed + pb;
    if (!ws || ws_bytes < fixed + pb) return fail(DGSM_ENOSPC, "workspace %zu < %zu bytes (plan part)", ws_bytes, fixed + pb);
    void* plan_ws = (char*)ws + fixed;
    // the event marking the end of the previous frame in this workspace
    CopyStream& cs = copy_stream();
    int slot = -1;
    for (int i = 0; i < 4; ++i)
        if (cs.slot_ws[i] == ws) slot = i;
    const bool known = slot >= 0;
    if (!known) {
        slot = cs.slot_next;
        cs.slot_next = (cs.slot_next + 1) % 4;
        cs.slot_ws[slot] = ws;
    }
    cudaEvent_t slot_ev = cs.slot_ev[slot];
    dgsm_plan_t plan;
    // a workspace not seen before (or evicted): wait for everything queued on `stream`
    if (!known) cudaEventRecord(slot_ev, (cudaStream_t)stream);
    int rc = plan_impl(&gd, g_host, kUploadChunks, slot_ev, lights, n_lights, atlas_res, n_shells, opts, plan_ws,
                       pb, &plan, stream);
    if (rc) return rc;
    int launches = g_launches;
    const size_t need = fixed + pb + plan.run_workspace_bytes;
    if (ws_required) *ws_required = need;
    if (ws_bytes < need) return fail(DGSM_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    // receivers ride the copy stream (after the Gaussian chunks) while the atlas is built
    if (m > 0) cudaMemcpyAsync(rec, receivers_host, 12 * (size_t)m, cudaMemcpyHostToDevice, cs.st);
    cudaEventRecord(cs.done, cs.st);
    g_ev_frame_acc = cs.acc;
    rc = dgsm_build_run(&gd, lights, n_lights, opts, &plan, plan_ws, pb, (char*)plan_ws + pb,
                        ws_bytes - fixed - pb, atlas_out, stream);
    g_ev_frame_acc = nullptr;
    if (rc) return rc;
    cs.acc_valid = true;
    launches += g_launches;
    cudaStreamWaitEvent(s, cs.done, 0);
    // page-locked T_host: the query writes it directly over the bus (no separate
    // device-to-host copy on the stream); pageable: device buffer + copy
    float* Tq = Td;
    bool direct = false;
    if (m > 0) {
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, T_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer) {
            Tq = (float*)pa.devicePointer;
            direct = true;
        }
        cudaGetLastError();  // (a pageable pointer is not an error here)
    }
    rc = dgsm_query(atlas_out, lights, n_lights, atlas_res, n_shells, rec, m, Tq, nullptr, stream);
    if (rc) return rc;
    launches += g_launches;
    if (m > 0 && !direct) cudaMemcpyAsync(T_host, Td, 4 * (size_t)m, cudaMemcpyDeviceToHost, s);
    cudaEventRecord(slot_ev, s);  // this workspace is free again after this point
    g_launches = launches;
    return cuda_check("frame");
}

int dgsm_exp_epilogue(const float* tau, float* T, int64_t count, void* stream) {
    g_launches = 0;
    if (count < 0) return fail(DGSM_EINVAL, "count < 0");
    if (count > 0 && (!tau || !T)) return fail(DGSM_EINVAL, "null tau or T");
    launch_exp(tau, T, count, (cudaStream_t)stream);
    g_launches = count > 0 ? 1 : 0;
    return cuda_check("exp epilogue");
}

static int check_query_args(const float* atlas, const dgsm_light_t* lights, int n_lights, int atlas_res,
                            int n_shells, int64_t m) {
    if (!lights) return fail(DGSM_EINVAL, "null lights");
    if (n_lights < 1 || n_lights > DGSM_MAX_LIGHTS) return fail(DGSM_EINVAL, "n_lights %d outside [1, %d]", n_lights, DGSM_MAX_LIGHTS);
    if (atlas_res < 8 || atlas_res % 8 != 0 || atlas_res > 2048) return fail(DGSM_EINVAL, "bad atlas_res %d", atlas_res);
    if (n_shells < 1 || n_shells > DGSM_MAX_SHELLS) return fail(DGSM_EINVAL, "bad n_shells %d", n_shells);
    if (m < 0) return fail(DGSM_EINVAL, "m < 0");
    if (m > 0 && !atlas) return fail(DGSM_EINVAL, "null atlas");
    for (int l = 0; l < n_lights; ++l)
        if (!(lights[l].t_max > 0.0f)) return fail(DGSM_EINVAL, "light %d: t_max <= 0", l);
    return DGSM_OK;
}

int dgsm_query(const float* atlas, const dgsm_light_t* lights, int n_lights, int atlas_res, int n_shells,
               const float* positions, int64_t m, float* T_out, float* colors_inout, void* stream) {
    g_launches = 0;
    if (int rc = check_query_args(atlas, lights, n_lights, atlas_res, n_shells, m)) return rc;
    if (m > 0 && (!positions || !T_out)) return fail(DGSM_EINVAL, "null positions or T_out");
    const LightsParam lp = lights_param(lights, n_lights);
    launch_query(atlas, lp, n_lights, atlas_res, n_shells, positions, m, T_out, colors_inout, (cudaStream_t)stream);
    g_launches = m > 0 ? 1 : 0;
    return cuda_check("query");
}

#ifndef DGSM_ORDER_BITS
#define DGSM_ORDER_BITS 30
#endif
constexpr int kOrderBits = DGSM_ORDER_BITS;  // significant Morton bits sorted (top bits of the 30-bit code)

size_t dgsm_order_workspace_bytes(int64_t m) {
    if (m < 0) return 0;
    Carver c(nullptr);
    c.take<uint32_t>(m);  // Morton keys
    c.take<uint32_t>(m);  // keys (ping-pong)
    c.take<uint32_t>(m);  // values (ping-pong)
    c.take<uint32_t>(8);  // bounding box
    c.take<char>(onesweep_temp_bytes(std::max<int64_t>(m, 1)));
    return c.off;
}

int dgsm_receiver_order(const float* positions, int64_t m, uint32_t* order_out, void* ws, size_t ws_bytes,
                        void* stream) {
    g_launches = 0;
    if (m < 0) return fail(DGSM_EINVAL, "m < 0");
    if (m >= ((int64_t)1 << 30)) return fail(DGSM_ERANGE, "m >= 2^30");
    if (m == 0) return DGSM_OK;
    if (!positions || !order_out || !ws) return fail(DGSM_EINVAL, "null positions, order or workspace");
    if ((uintptr_t)ws % kAlign) return fail(DGSM_EINVAL, "workspace not 256-B aligned");
    if (ws_bytes < dgsm_order_workspace_bytes(m))
        return fail(DGSM_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, dgsm_order_workspace_bytes(m));
    cudaStream_t s = (cudaStream_t)stream;
    Carver c(ws);
    uint32_t* keys = c.take<uint32_t>(m);
    uint32_t* keys_alt = c.take<uint32_t>(m);
    uint32_t* vals_alt = c.take<uint32_t>(m);
    uint32_t* box = c.take<uint32_t>(8);
    void* temp = c.take<char>(onesweep_temp_bytes(m));
    // the Morton kernel fills the sort's digit histograms (no separate histogram pass)
    uint32_t* hist = onesweep_prepare(temp, m, s);
    launch_morton(positions, m, box, keys, order_out, onesweep_digits(kOrderBits), hist, s);
    g_launches += 2;
    const int alt = launch_onesweep_u32(keys, order_out, keys_alt, vals_alt, m, kOrderBits, temp, s, &g_launches,
                                        nullptr, nullptr, /*hist_ready=*/true, /*top_match=*/false);
    if (alt) cudaMemcpyAsync(order_out, vals_alt, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, s);
    return cuda_check("receiver order");
}

int dgsm_query_ordered(const float* atlas, const dgsm_light_t* lights, int n_lights, int atlas_res, int n_shells,
                       const float* positions, const uint32_t* order, int64_t m, float* T_out, float* colors_inout,
                       void* stream) {
    g_launches = 0;
    if (int rc = check_query_args(atlas, lights, n_lights, atlas_res, n_shells, m)) return rc;
    if (m > 0 && (!positions || !T_out || !order)) return fail(DGSM_EINVAL, "null positions, order or T_out");
    const LightsParam lp = lights_param(lights, n_lights);
    launch_query_ordered(atlas, lp, n_lights, atlas_res, n_shells, positions, order, m, T_out, colors_inout,
                         (cudaStream_t)stream);
    g_launches = m > 0 ? 1 : 0;
    return cuda_check("query ordered");
}

int dgsm_query_chunks(const float* const* chunks, const int32_t* k_begin, const int32_t* k_end,
                      const int32_t* split, const dgsm_light_t* lights, int n_lights, int atlas_res, int n_shells,
                      const float* positions, int64_t m, float* T_out, float* partial_out, void* stream) {
    g_launches = 0;
    if (!chunks || !k_begin || !k_end || !split) return fail(DGSM_EINVAL, "null chunk arrays");
    if (int rc = check_query_args(nullptr, lights, n_lights, atlas_res, n_shells, 0)) return rc;
    if (m < 0) return fail(DGSM_EINVAL, "m < 0");
    int n_split = 0, n_full = 0;
    for (int l = 0; l < n_lights; ++l) {
        if (k_begin[l] < 0 || k_begin[l] > k_end[l] || k_end[l] > n_shells)
            return fail(DGSM_EINVAL, "light %d: bad shell chunk [%d, %d)", l, k_begin[l], k_end[l]);
        if (k_end[l] > k_begin[l] && !chunks[l]) return fail(DGSM_EINVAL, "light %d: null chunk", l);
        if (split[l]) ++n_split;
        else if (k_end[l] == k_begin[l]) continue;  // not held here: skipped
        else if (k_begin[l] != 0 || k_end[l] != n_shells)
            return fail(DGSM_EINVAL, "light %d: a complete light needs the chunk [0, %d)", l, n_shells);
        else ++n_full;
    }
    if (m > 0 && !positions) return fail(DGSM_EINVAL, "null positions");
    if (m > 0 && n_split > 0 && !partial_out) return fail(DGSM_EINVAL, "null partial_out");
    if (m > 0 && !T_out && n_full > 0) return fail(DGSM_EINVAL, "null T_out");
    const LightsParam lp = lights_param(lights, n_lights);
    launch_query_chunks(chunks, k_begin, k_end, split, lp, n_lights, atlas_res, n_shells, positions, m, T_out,
                        partial_out, (cudaStream_t)stream);
    g_launches = m > 0 ? 1 : 0;
    return cuda_check("query chunks");
}

int dgsm_query_combine(const float* partial, int n_split, int64_t m, float* T_inout, void* stream) {
    g_launches = 0;
    if (n_split < 0 || m < 0) return fail(DGSM_EINVAL, "n_split < 0 or m < 0");
    if (m > 0 && (!T_inout || (n_split > 0 && !partial))) return fail(DGSM_EINVAL, "null partial or T");
    launch_query_combine(partial, n_split, m, T_inout, (cudaStream_t)stream);
    g_launches = m > 0 ? 1 : 0;
    return cuda_check("query combine");
}

int dgsm_query_footprint(const float* atlas, const dgsm_light_t* lights, int n_lights, int atlas_res,
                         int n_shells, const float* means, const float* scales, const float* rotations, int64_t m,
                         const float* offsets, const float* weights, int n_samples, float* T_out,
                         float* colors_inout, void* stream) {
    g_launches = 0;
    if (int rc = check_query_args(atlas, lights, n_lights, atlas_res, n_shells, m)) return rc;
    if (m > 0 && (!means || !scales || !rotations || !T_out))
        return fail(DGSM_EINVAL, "null means, scales, rotations or T_out");
    if (!offsets || !weights) return fail(DGSM_EINVAL, "null offsets or weights");
    if (n_samples < 1 || n_samples > DGSM_MAX_FOOTPRINT_SAMPLES)
        return fail(DGSM_EINVAL, "n_samples %d outside [1, %d]", n_samples, DGSM_MAX_FOOTPRINT_SAMPLES);
    FootprintParam fp;
    fp.n = n_samples;
    for (int i = 0; i < n_samples; ++i)
        fp.zw[i] = make_float4(offsets[3 * i], offsets[3 * i + 1], offsets[3 * i + 2], weights[i]);
    const LightsParam lp = lights_param(lights, n_lights);
    launch_query_footprint(atlas, lp, fp, n_lights, atlas_res, n_shells, means, scales, rotations, m, T_out,
                           colors_inout, (cudaStream_t)stream);
    g_launches = m > 0 ? 1 : 0;
    return cuda_check("query footprint");
}

int dgsm_footprint_stencil(int kind, float delta, float* offsets_out, float* weights_out, int* n_out) {
    if (!offsets_out || !weights_out || !n_out) return fail(DGSM_EINVAL, "null output");
    if (kind == DGSM_STENCIL_CENTER) {
        offsets_out[0] = offsets_out[1] = offsets_out[2] = 0.0f;
        weights_out[0] = 1.0f;
        *n_out = 1;
        return DGSM_OK;
    }
    if (kind != DGSM_STENCIL_7) return fail(DGSM_EINVAL, "unknown stencil kind %d", kind);
    if (!(delta > 0.0f) || !(delta < 1e30f)) return fail(DGSM_EINVAL, "stencil delta must be finite and > 0");
    // {0, +-delta e_j}; w_i proportional to exp(-|z_i|^2 / 2), normalised (fp64 host arithmetic)
    const double d = delta, wc = 1.0, wa = exp(-0.5 * d * d), sum = wc + 6.0 * wa;
    for (int i = 0; i < 21; ++i) offsets_out[i] = 0.0f;
    weights_out[0] = (float)(wc / sum);
    for (int j = 0; j < 3; ++j) {
        offsets_out[3 * (1 + 2 * j) + j] = delta;
        offsets_out[3 * (2 + 2 * j) + j] = -delta;
        weights_out[1 + 2 * j] = weights_out[2 + 2 * j] = (float)(wa / sum);
    }
    *n_out = 7;
    return DGSM_OK;
}

void dgsm_default_transfer_opts(dgsm_transfer_opts_t* o) {
    if (!o) return;
    o->grid_theta = 64;
    o->grid_phi = 128;
    o->q = 1.0f;
    o->eps = 1e-6f;
    o->s_max = 4.0f;
    o->gamma = 1.0f;
}

static int check_transfer_opts(const dgsm_transfer_opts_t& o) {
    if (o.grid_theta < 1 || o.grid_phi < 1 || (int64_t)o.grid_theta * o.grid_phi > (1 << 24))
        return fail(DGSM_EINVAL, "bad transfer grid %d x %d", o.grid_theta, o.grid_phi);
    if (!(o.q >= 0.0f) || !(o.eps >= 0.0f) || !(o.s_max > 0.0f))
        return fail(DGSM_EINVAL, "transfer: need q >= 0, eps >= 0, s_max > 0");
    return DGSM_OK;
}

size_t dgsm_transfer_workspace_bytes(const dgsm_transfer_opts_t* opts, int64_t n) {
    dgsm_transfer_opts_t o;
    if (opts) o = *opts; else dgsm_default_transfer_opts(&o);
    if (n < 0 || o.grid_theta < 1 || o.grid_phi < 1) return 0;
    return transfer_workspace_bytes(o.grid_theta, o.grid_phi, n);
}

int dgsm_sh_transfer(const float* sh, int sh_degree, const float* normals, const float* colors_in, int64_t n,
                     const dgsm_transfer_opts_t* opts, float* scales_out, float* colors_out, void* ws,
                     size_t ws_bytes, void* stream) {
    g_launches = 0;
    dgsm_transfer_opts_t o;
    if (opts) o = *opts; else dgsm_default_transfer_opts(&o);
    if (int rc = check_transfer_opts(o)) return rc;
    if (!sh) return fail(DGSM_EINVAL, "null sh");
    if (sh_degree < 0 || sh_degree > DGSM_MAX_SH_DEGREE) return fail(DGSM_EINVAL, "sh_degree %d outside [0, %d]", sh_degree, DGSM_MAX_SH_DEGREE);
    if (n < 0) return fail(DGSM_EINVAL, "n < 0");
    if (n > 0 && !normals) return fail(DGSM_EINVAL, "null normals");
    if (colors_out && !colors_in) return fail(DGSM_EINVAL, "colors_out without colors_in");
    if (!ws || (uintptr_t)ws % kAlign) return fail(DGSM_EINVAL, "null or unaligned workspace");
    const size_t need = transfer_workspace_bytes(o.grid_theta, o.grid_phi, n);
    if (ws_bytes < need) return fail(DGSM_ENOSPC, "transfer workspace %zu < %zu bytes", ws_bytes, need);
    ShParam sp;
    memset(&sp, 0, sizeof(sp));
    sp.d = sh_degree;
    const int K = (sh_degree + 1) * (sh_degree + 1);
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < K; ++k) sp.a[c][k] = sh[c * K + k];
    launch_transfer(sp, o.grid_theta, o.grid_phi, o.q, o.eps, o.s_max, o.gamma, normals, colors_in, n, scales_out,
                    colors_out, ws, (cudaStream_t)stream, &g_launches);
    return cuda_check("sh transfer");
}

size_t dgsm_sort_temp_bytes(int64_t n) {
    if (n < 0) return 0;
    return onesweep_temp_bytes(std::max<int64_t>(n, 1));
}

int dgsm_sort_pairs_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int64_t n,
                        int nbits, void* temp, size_t temp_bytes, int* result_in_alt, void* stream) {
    g_launches = 0;
    if (!result_in_alt) return fail(DGSM_EINVAL, "null result_in_alt");
    *result_in_alt = 0;
    if (n < 0 || nbits < 0 || nbits > 32) return fail(DGSM_EINVAL, "need n >= 0 and 0 <= nbits <= 32");
    if (n >= ((int64_t)1 << 30)) return fail(DGSM_ERANGE, "n >= 2^30");
    if (n > 0 && (!keys || !vals || !keys_alt || !vals_alt || !temp)) return fail(DGSM_EINVAL, "null buffer");
    if ((uintptr_t)temp % kAlign) return fail(DGSM_EINVAL, "temp not 256-B aligned");
    if (temp_bytes < dgsm_sort_temp_bytes(n)) return fail(DGSM_ENOSPC, "temp %zu < %zu bytes", temp_bytes, dgsm_sort_temp_bytes(n));
    if (n <= 1 || nbits == 0) return DGSM_OK;
    *result_in_alt = launch_onesweep_u32(keys, vals, keys_alt, vals_alt, n, nbits, temp, (cudaStream_t)stream,
                                         &g_launches);
    return cuda_check("sort");
}

int dgsm_set_frame_event(void* ev) {
    g_ev_frame_ext = (cudaEvent_t)ev;
    return DGSM_OK;
}

int dgsm_set_accumulate_events(void* before, void* after) {
    g_ev_before = (cudaEvent_t)before;
    g_ev_after = (cudaEvent_t)after;
    return DGSM_OK;
}

int dgsm_build_stats(const dgsm_plan_t* plan, void* run_ws, size_t run_ws_bytes, dgsm_build_stats_t* out,
                     void* stream) {
    if (!plan || !run_ws || !out) return fail(DGSM_EINVAL, "null argument");
    if (run_ws_bytes < plan->run_workspace_bytes) return fail(DGSM_ENOSPC, "run workspace too small");
    const RunLayout r = run_layout(run_ws, plan_shape(*plan));
    unsigned long long h[8];
    cudaMemcpyAsync(h, r.stats, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return cuda_check("stats");
    out->pairs = h[0];
    out->pairs_live = h[1];
    out->window_shells = h[2];
    out->steps = h[3];
    out->warp_records = h[4];
    out->warp_live_any = h[5];
    out->warp_live_max = h[6];
    out->band_records = h[7];
    return DGSM_OK;
}

const char* dgsm_strerror(int code) {
    switch (code) {
        case DGSM_OK: return "success";
        case DGSM_EINVAL: return "invalid argument";
        case DGSM_ENOSPC: return "workspace too small";
        case DGSM_ECUDA: return "CUDA error";
        case DGSM_ERANGE: return "problem too large";
        case DGSM_EDATA: return "invalid Gaussian data";
        default: return "unknown error";
    }
}

const char* dgsm_last_error(void) { return g_err; }

int dgsm_last_launch_count(void) { return g_launches; }

}  // extern "C"
