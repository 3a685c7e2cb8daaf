// C ABI of the CLATCH hot paths (include/clatch.h): context, pattern install,
// host-side keypoint preparation, host-buffer wrappers and the match filter pass.
// Reference citations are relative to /root/reference/proj.

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>

#include "clatch_internal.cuh"
#include <atomic>
#include <chrono>

#include "slot_assign.hpp"

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace clatch {
namespace {
#include "default_plan_f8.inc"
#include "default_plan_h16.inc"
#include "default_plan_sw.inc"
}
}

namespace clatch {

namespace {
thread_local std::string g_error = "";
}

void set_error(const std::string& msg) { g_error = msg; }

int cuda_fail(cudaError_t e, const char* what) {
    set_error(std::string("CUDA error '") + cudaGetErrorString(e) + "' in " + what);
    return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? CLATCH_ERR_NO_DEVICE
                                                                       : CLATCH_ERR_CUDA;
}

int DeviceBuffer::reserve(size_t bytes) {
    if (bytes <= cap) return CLATCH_OK;
    if (ptr) CLATCH_CUDA(cudaFree(ptr));
    ptr = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    CLATCH_CUDA(cudaMalloc(&ptr, want));
    cap = want;
    return CLATCH_OK;
}

int PinnedBuffer::reserve(size_t bytes) {
    if (bytes <= cap) return CLATCH_OK;
    if (ptr) CLATCH_CUDA(cudaFreeHost(ptr));
    ptr = nullptr;
    cap = 0;
    const size_t want = bytes + bytes / 4;
    CLATCH_CUDA(cudaHostAlloc(&ptr, want, cudaHostAllocDefault));
    cap = want;
    return CLATCH_OK;
}

void PinnedBuffer::release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    cap = 0;
}

void DeviceBuffer::release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
}

namespace {

// Persistent host workers for the trig pass: spawning std::threads per call (what the
// reference's parallel_for does, src/parallel.hpp:26-37) costs more than the work itself at
// 10 k keypoints.
class WorkerPool {
public:
    static WorkerPool& instance() {
        static WorkerPool pool;
        return pool;
    }
    // Runs fn(i) for i in [0, parts) on up to `parts` threads (the caller takes part 0).
    void run(int parts, const std::function<void(int)>& fn) {
        if (parts <= 1) {
            fn(0);
            return;
        }
        std::unique_lock<std::mutex> call_lock(call_mutex_);   // one parallel region at a time
        ensure(parts - 1);
        {
            std::lock_guard<std::mutex> lock(mutex_);
            fn_ = &fn;
            next_ = 1;
            parts_ = parts;
            pending_ = parts - 1;
        }
        wake_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> lock(mutex_);
        done_.wait(lock, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    WorkerPool() = default;
    ~WorkerPool() {
        {
            std::lock_guard<std::mutex> lock(mutex_);
            stop_ = true;
        }
        wake_.notify_all();
        for (std::thread& t : threads_) t.join();
    }
    void ensure(int n) {
        while (static_cast<int>(threads_.size()) < n) threads_.emplace_back([this] { loop(); });
    }
    void loop() {
        for (;;) {
            int part = -1;
            const std::function<void(int)>* fn = nullptr;
            {
                std::unique_lock<std::mutex> lock(mutex_);
                wake_.wait(lock, [&] { return stop_ || next_ < parts_; });
                if (stop_) return;
                part = next_++;
                fn = fn_;
            }
            (*fn)(part);
            {
                std::lock_guard<std::mutex> lock(mutex_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::mutex call_mutex_, mutex_;
    std::condition_variable wake_, done_;
    std::vector<std::thread> threads_;
    const std::function<void(int)>* fn_ = nullptr;
    int next_ = 0, parts_ = 0, pending_ = 0;
    bool stop_ = false;
};

// CLATCH_TRACE=1: host-clock stamps of the host-API stages on stderr (diagnostics).
struct Trace {
    bool on = std::getenv("CLATCH_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void stamp(const char* what) {
        if (!on) return;
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[clatch] %-28s %9.1f us\n", what, us);
    }
};

int invalid(const std::string& msg) {
    set_error(msg);
    return CLATCH_ERR_INVALID;
}

int resolve_workers(int workers) {   // src/parallel.hpp:9-13
    if (workers > 0) return workers;
    // workers <= 0 means "all hardware threads" in the reference; here the pool only runs the trig pass
    // next to the CUDA driver's own threads and the caller's, and taking every core made the batch
    // pipeline stall for milliseconds at random (describe_batch, 8 x 50 k keypoints on a 16-thread host:
    // 7.5-33 ms with 16 workers, 6.9 ms flat with 12 or 4): leave four threads free, use at most 12.
    const unsigned hw = std::thread::hardware_concurrency();
    return hw > 4 ? static_cast<int>(std::min(hw - 4, 12u)) : std::max(1, static_cast<int>(hw / 2));
}

// Host-side promotion of a float64 image whose pixels are all integers in [0, 255] (every
// PGM-sourced image, src/image.cpp:75-76) to u8: rows [r0, r1) -> dst, false at the first pixel
// that is not such a value (NaN and out-of-range values fail the round trip). Same rule as the
// device's classify_convert_kernel; it exists because 1 byte per pixel crosses the bus 8x faster
// than 8, and the host can read its own memory faster than PCIe can carry it. SSE2 only (baseline
// x86-64): 8 pixels per step.
bool promote_rows_u8(const double* src, size_t src_pitch, uint8_t* dst, size_t dst_pitch, int width, int r0,
                     int r1) {
    for (int r = r0; r < r1; ++r) {
        const double* s = src + static_cast<size_t>(r) * src_pitch;
        uint8_t* d = dst + static_cast<size_t>(r) * dst_pitch;
        int x = 0;
        bool bad = false;
#if defined(__SSE2__)
        __m128d ne = _mm_setzero_pd();
        __m128i high = _mm_setzero_si128();
        for (; x + 8 <= width; x += 8) {
            const __m128d a0 = _mm_loadu_pd(s + x), a1 = _mm_loadu_pd(s + x + 2), a2 = _mm_loadu_pd(s + x + 4),
                          a3 = _mm_loadu_pd(s + x + 6);
            const __m128i i0 = _mm_cvttpd_epi32(a0), i1 = _mm_cvttpd_epi32(a1), i2 = _mm_cvttpd_epi32(a2),
                          i3 = _mm_cvttpd_epi32(a3);
            ne = _mm_or_pd(_mm_or_pd(_mm_cmpneq_pd(_mm_cvtepi32_pd(i0), a0), _mm_cmpneq_pd(_mm_cvtepi32_pd(i1), a1)),
                           _mm_or_pd(_mm_or_pd(_mm_cmpneq_pd(_mm_cvtepi32_pd(i2), a2),
                                               _mm_cmpneq_pd(_mm_cvtepi32_pd(i3), a3)),
                                     ne));
            const __m128i lo = _mm_unpacklo_epi64(i0, i1), hi = _mm_unpacklo_epi64(i2, i3);
            high = _mm_or_si128(high, _mm_or_si128(lo, hi));
            const __m128i p16 = _mm_packs_epi32(lo, hi);
            _mm_storel_epi64(reinterpret_cast<__m128i*>(d + x), _mm_packus_epi16(p16, p16));
        }
        high = _mm_andnot_si128(_mm_set1_epi32(0xFF), high);   // any bit above the low byte (or the sign)
        bad = _mm_movemask_pd(ne) != 0 || _mm_movemask_epi8(_mm_cmpeq_epi32(high, _mm_setzero_si128())) != 0xFFFF;
#endif
        for (; x < width; ++x) {
            const double v = s[x];
            const bool ok = v >= 0.0 && v <= 255.0 && v == std::floor(v);
            bad = bad || !ok;
            d[x] = ok ? static_cast<uint8_t>(v) : 0;
        }
        if (bad) return false;
    }
    return true;
}

// Should this float64 host image be promoted to u8 by the host workers (clatch_ctx::host_promote)?
bool is_pageable(const void* p);
bool want_host_promote(const clatch_ctx* ctx, const void* img) {
    if (ctx->host_promote == 1) return true;
    if (ctx->host_promote == 2) return false;
    return is_pageable(img);   // ordinary malloc'd / numpy memory
}

// Ordinary (pageable) host memory? The driver copies such memory through its own bounce buffers — row by row for a
// 2-D copy: a 1920x1080 u8 image took 2.3 ms instead of 40 us — so big pageable images are first gathered into
// page-locked staging by the host workers and sent as one flat DMA.
bool is_pageable(const void* p) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return attr.type == cudaMemoryTypeUnregistered;
}

// WeightMask::seven_by_seven (src/pattern.cpp:28-35): ones on the top-left 7x7, zero last row/col.
bool is_seven_by_seven(const std::vector<double>& w, int K) {
    if (K != 8) return false;
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c)
            if (w[r * 8 + c] != ((r < 7 && c < 7) ? 1.0 : 0.0)) return false;
    return true;
}

} // namespace

} // namespace clatch

using namespace clatch;

extern "C" {

const char* clatch_last_error(void) { return g_error.c_str(); }

int clatch_ctx_create(int device, clatch_ctx** out) {
    if (!out) return invalid("clatch_ctx_create: out is null");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        set_error(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                  "); the CLATCH paths have no CPU fallback");
        return CLATCH_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= count) return invalid("clatch_ctx_create: device index out of range");
    CLATCH_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    CLATCH_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error(std::string("device '") + prop.name + "' is sm_" + std::to_string(prop.major) +
                  std::to_string(prop.minor) + "; this library is built for sm_100a only");
        return CLATCH_ERR_NO_DEVICE;
    }
    auto* ctx = new clatch_ctx;
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
    ctx->sm_clock_khz = khz;
    std::snprintf(ctx->name, sizeof(ctx->name), "%s", prop.name);
    cudaError_t se = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (se != cudaSuccess) {
        delete ctx;
        return cuda_fail(se, "cudaStreamCreateWithFlags");
    }
    if (const char* v = std::getenv("CLATCH_MATCH_VARIANT")) ctx->match_variant = std::atoi(v);
    if (const char* v = std::getenv("CLATCH_MATCH_2CTA")) ctx->match_2cta = std::atoi(v) != 0;
    if (const char* v = std::getenv("CLATCH_MATCH_STREAMK_PAIRS")) ctx->match_streamk_pairs = std::atoi(v) != 0;
    if (const char* v = std::getenv("CLATCH_EXTRACT_VARIANT")) {
        const int ev = std::atoi(v);
        if (ev >= 0 && ev <= 6) ctx->extract_variant = ev;
    }
    // per-CTA slots of the extraction router, written by the device into page-locked host memory (no copy, no sync)
    if (cudaHostAlloc(reinterpret_cast<void**>(&ctx->route_host), sizeof(uint2) * ctx->sm_count, cudaHostAllocMapped) == cudaSuccess) {
        std::memset(ctx->route_host, 0, sizeof(uint2) * ctx->sm_count);
        if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->route_dev), ctx->route_host, 0) != cudaSuccess) {
            cudaFreeHost(ctx->route_host);
            ctx->route_host = nullptr;
        }
    } else {
        ctx->route_host = nullptr;
    }
    cudaGetLastError();
    *out = ctx;
    return CLATCH_OK;
}

void clatch_ctx_destroy(clatch_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
    }
    for (DeviceBuffer* b : {&ctx->img, &ctx->kps, &ctx->desc, &ctx->q, &ctx->t, &ctx->res,
                            &ctx->partial, &ctx->flags, &ctx->img_u8, &ctx->exp_q, &ctx->exp_t, &ctx->items, &ctx->scores, &ctx->counts, &ctx->det, &ctx->pattern.slots, &ctx->pattern.slots_quad,
                            &ctx->pattern.slots_f8, &ctx->pattern.slots_h16, &ctx->extract_stats, &ctx->filt_pairs, &ctx->filt_rows, &ctx->filt_out,
                            &ctx->filt_counts, &ctx->pattern.triplets, &ctx->pattern.d_weights})
        b->release();
    for (auto& t : ctx->tex_images) {
        if (t.tex) cudaDestroyTextureObject(t.tex);
        if (t.texn) cudaDestroyTextureObject(t.texn);
        if (t.texf) cudaDestroyTextureObject(t.texf);
        if (t.surff) cudaDestroySurfaceObject(t.surff);
        if (t.arrayf) cudaFreeArray(t.arrayf);
        if (t.tickets) cudaFree(t.tickets);
        if (t.surf) cudaDestroySurfaceObject(t.surf);
        if (t.array) cudaFreeArray(t.array);
    }
    if (ctx->scratch_event) cudaEventDestroy(ctx->scratch_event);
    if (ctx->route_host) cudaFreeHost(ctx->route_host);
    ctx->pinned.release();
    ctx->pin_img.release();
    ctx->pin_xycs.release();
    ctx->pin_desc.release();
    if (ctx->copy_stream) {
        cudaStreamDestroy(ctx->copy_stream);
        for (cudaEvent_t e : ctx->band_events)
            if (e) cudaEventDestroy(e);
    }
    for (int s = 0; s < 2; ++s) {
        for (DeviceBuffer* b : {&ctx->pipe[s].img, &ctx->pipe[s].kps, &ctx->pipe[s].desc, &ctx->pipe[s].img_u8,
                                &ctx->pipe[s].flags})
            b->release();
        ctx->pipe[s].h_xycs.release();
        ctx->pipe[s].h_desc.release();
        ctx->pipe[s].h_img.release();
        if (ctx->pipe[s].stream) cudaStreamDestroy(ctx->pipe[s].stream);
    }
    delete ctx;
}

int clatch_device_info(clatch_ctx* ctx, int* sm_count, int* sm_clock_khz, char* name, size_t cap) {
    if (!ctx) return invalid("clatch_device_info: ctx is null");
    if (sm_count) *sm_count = ctx->sm_count;
    if (sm_clock_khz) *sm_clock_khz = ctx->sm_clock_khz;
    if (name && cap) {
        std::strncpy(name, ctx->name, cap - 1);
        name[cap - 1] = 0;
    }
    return CLATCH_OK;
}

int clatch_set_option(clatch_ctx* ctx, const char* key, int value) {
    if (!ctx || !key) return invalid("clatch_set_option: null argument");
    if (std::strcmp(key, "match_variant") == 0) {
        if (value < 0 || value > 4) return invalid("match_variant must be 0..4");
        ctx->match_variant = value;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "extract_variant") == 0) {
        if (value < 0 || value > 6) return invalid("extract_variant must be 0..6");
        ctx->extract_variant = value;
        ctx->route_quad = ctx->route_pending = false;
        ctx->route_age = 0;
        ctx->route_period = 16;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "pdl") == 0) {   // programmatic dependent launch inside the library's kernel chains
        ctx->pdl = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "extract_route") == 0) {   // route degenerate image streams to the all-fp64 quad kernel (1, default) or never (0)
        ctx->extract_route = value != 0;
        ctx->route_quad = ctx->route_pending = false;
        ctx->route_age = 0;
        ctx->route_period = 16;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "upload_bands") == 0) {   // describe_all, float64 images: row bands of the upload (1 = one piece)
        if (value < 0 || value > 6) return invalid("upload_bands must be 0 (auto) or 1..6");
        ctx->upload_bands = value;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "pairs_filter_on_device") == 0) {   // batched set pairs: filter pass on the device (1) or host (0)
        ctx->pairs_filter_on_device = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "match_form_auto") == 0) {   // variant 4: let mid-sized single matches use the int8 form
        ctx->match_form_auto = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "match_pairs") == 0) {   // tensor matcher: CTA pairs sharing the train stream by TMA multicast
        ctx->match_pairs = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "match_2cta") == 0) {   // tensor matcher, paired e2m1 launches: one M = 256 MMA stream per CTA pair
        ctx->match_2cta = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "match_streamk") == 0) {   // tensor matcher: stream-K partition for small problems
        ctx->match_streamk = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "extract_f64_h16") == 0) {   // tame non-u8 float64 images: packed-plane kernel (1) or the all-fp64 quad kernel (0)
        ctx->extract_f64_h16 = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "match_streamk_pairs") == 0) {   // ... cut over query tile pairs, runs on CTA pairs (multicast)
        ctx->match_streamk_pairs = value != 0;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "host_promote") == 0) {   // float64 -> u8 on the host workers when lossless: 0 auto, 1 always, 2 never
        if (value < 0 || value > 2) return invalid("host_promote must be 0 (pageable sources), 1 (always) or 2 (never)");
        ctx->host_promote = value;
        return CLATCH_OK;
    }
    if (std::strcmp(key, "extract_stats") == 0) {   // count exact recomputes of the filtered kernel
        CLATCH_CUDA(cudaSetDevice(ctx->device));
        if (int rc = ctx->extract_stats.reserve(2 * sizeof(unsigned long long))) return rc;
        CLATCH_CUDA(cudaMemsetAsync(ctx->extract_stats.ptr, 0, 2 * sizeof(unsigned long long), ctx->stream));
        ctx->extract_stats_on = value != 0;
        return CLATCH_OK;
    }
    return invalid(std::string("clatch_set_option: unknown key '") + key + "'");
}

int clatch_synchronize(clatch_ctx* ctx) {
    if (!ctx) return invalid("clatch_synchronize: ctx is null");
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    CLATCH_CUDA(cudaStreamSynchronize(ctx->stream));
    return CLATCH_OK;
}

uint64_t clatch_launch_count(clatch_ctx* ctx) { return ctx ? ctx->launches : 0; }

int clatch_host_alloc(size_t bytes, void** out) {
    if (!out) return invalid("clatch_host_alloc: out is null");
    *out = nullptr;
    CLATCH_CUDA(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable));
    return CLATCH_OK;
}

int clatch_host_free(void* ptr) {
    if (ptr) CLATCH_CUDA(cudaFreeHost(ptr));
    return CLATCH_OK;
}

int clatch_extract_stats(clatch_ctx* ctx, uint64_t* exact_triplets, uint64_t* exact_warps) {
    if (!ctx) return invalid("clatch_extract_stats: ctx is null");
    unsigned long long h[2] = {0, 0};
    if (ctx->extract_stats.ptr) {
        CLATCH_CUDA(cudaSetDevice(ctx->device));
        CLATCH_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int s = 0; s < 2; ++s)
            if (ctx->pipe[s].stream) CLATCH_CUDA(cudaStreamSynchronize(ctx->pipe[s].stream));
        CLATCH_CUDA(cudaMemcpy(h, ctx->extract_stats.ptr, sizeof(h), cudaMemcpyDeviceToHost));
    }
    if (exact_triplets) *exact_triplets = h[0];
    if (exact_warps) *exact_warps = h[1];
    return CLATCH_OK;
}

int clatch_descriptor_bytes(clatch_ctx* ctx) { return ctx ? ctx->pattern.T / 8 : 0; }

int clatch_set_pattern(clatch_ctx* ctx, const int16_t* triplets, int T, int K, const double* mask) {
    if (!ctx || !triplets) return invalid("clatch_set_pattern: null argument");
    // Same acceptance rules as parse_pattern (src/pattern.cpp:78-82, 54-66, 118-131).
    if (T <= 0 || T % 8 != 0) {
        set_error("BadHeader: T must be a positive multiple of 8, got " + std::to_string(T));
        return CLATCH_ERR_BAD_HEADER;
    }
    if (T > 32768) return invalid("clatch_set_pattern: T > 32768 is not supported");
    if (K < 1 || K > kWindow) {
        set_error("BadHeader: K out of range: " + std::to_string(K));
        return CLATCH_ERR_BAD_HEADER;
    }
    const int max_coord = kWindow - K;
    for (int t = 0; t < T; ++t) {
        const int16_t* v = triplets + 6 * t;
        for (int i = 0; i < 6; ++i)
            if (v[i] < 0 || v[i] > max_coord) {
                set_error("CoordinateOutOfRange: coordinate " + std::to_string(v[i]) +
                          " outside [0, " + std::to_string(max_coord) + "]");
                return CLATCH_ERR_COORD_RANGE;
            }
        if (v[2] == v[4] && v[3] == v[5]) {
            set_error("DegenerateTriplet: companion patches coincide at (" + std::to_string(v[2]) +
                      ", " + std::to_string(v[3]) + ")");
            return CLATCH_ERR_DEGENERATE;
        }
    }
    std::vector<double> w(static_cast<size_t>(K) * K, 1.0);
    if (mask) {
        bool any = false;
        for (size_t i = 0; i < w.size(); ++i) {
            if (!std::isfinite(mask[i]) || mask[i] < 0.0) {
                set_error("BadHeader: bad weight in row " + std::to_string(i / K));
                return CLATCH_ERR_BAD_HEADER;
            }
            w[i] = mask[i];
            any = any || mask[i] > 0.0;
        }
        if (!any) {
            set_error("BadHeader: weight mask is all zeros");
            return CLATCH_ERR_BAD_HEADER;
        }
    }

    CLATCH_CUDA(cudaSetDevice(ctx->device));
    CLATCH_CUDA(cudaDeviceSynchronize());   // kernels queued on any stream may still read the tables replaced below
    Pattern& pat = ctx->pattern;
    pat.T = T;
    pat.K = K;
    pat.weights = w;
    pat.fast = (T == kFastT) && is_seven_by_seven(w, K);
    if (int rc = pat.triplets.reserve(sizeof(int16_t) * 6 * T)) return rc;
    CLATCH_CUDA(cudaMemcpy(pat.triplets.ptr, triplets, sizeof(int16_t) * 6 * T, cudaMemcpyHostToDevice));
    if (int rc = pat.d_weights.reserve(sizeof(double) * w.size())) return rc;
    CLATCH_CUDA(cudaMemcpy(pat.d_weights.ptr, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
    pat.host_triplets.assign(triplets, triplets + 6 * static_cast<size_t>(T));
    pat.slots_planned = false;
    if (pat.fast) {
        // Lane placements that keep the window loads (nearly) bank-conflict free (slot_assign.hpp).
        static_assert(sizeof(SlotEntry) == sizeof(ushort4), "slot layout");
        const SlotPlan quad = plan_slots_quad(triplets, T, kWinStride, 300000);
        pat.slot_degree_quad = quad.avg_degree;
        if (int rc = pat.slots_quad.reserve(sizeof(SlotEntry) * T)) return rc;
        CLATCH_CUDA(cudaMemcpy(pat.slots_quad.ptr, quad.slots.data(), sizeof(SlotEntry) * T, cudaMemcpyHostToDevice));
        if (int rc = pat.slots_f8.reserve(sizeof(SlotEntry) * T)) return rc;
        if (triplet_hash(triplets, T) == kDefaultPlanHash && kDefaultPlanStride == kWinStride) {
            // the built-in table: placement precomputed by a long anneal (tools/gen_default_plan.py)
            static_assert(sizeof(kDefaultPlanF8) == sizeof(SlotEntry) * kFastT, "embedded plan size");
            pat.slot_degree_f8 = kDefaultPlanDegree;
            CLATCH_CUDA(cudaMemcpy(pat.slots_f8.ptr, kDefaultPlanF8, sizeof(kDefaultPlanF8), cudaMemcpyHostToDevice));
            pat.slots_f8_planned = true;
        } else {
            pat.slots_f8_planned = false;   // planned on first use (variants 2-4 are A/B selections now): 0.3 s of annealing
        }
        if (triplet_hash(triplets, T) == kDefaultPlanHash && kDefaultPlanSWStride == kWinStride) {
            // ... and the one-window placement (variant 0; the packed-plane kernel's window-wide exact pass)
            static_assert(sizeof(kDefaultPlanSW) == sizeof(SlotEntry) * kFastT, "embedded plan size");
            if (int rc = pat.slots.reserve(sizeof(SlotEntry) * T)) return rc;
            pat.slot_degree = kDefaultPlanSWDegree;
            pat.slot_degree_identity = kDefaultPlanSWDegreeIdentity;
            CLATCH_CUDA(cudaMemcpy(pat.slots.ptr, kDefaultPlanSW, sizeof(kDefaultPlanSW), cudaMemcpyHostToDevice));
            pat.slots_planned = true;
        } else if (ctx->extract_variant == 5) {
            // another table: plan it here (0.2 s of annealing) rather than inside the first describe() that meets a flat window
            const SlotPlan sw = plan_slots(triplets, T, kWinStride, 1000000);
            pat.slot_degree = sw.avg_degree;
            pat.slot_degree_identity = sw.avg_degree_identity;
            if (int rc = pat.slots.reserve(sizeof(SlotEntry) * T)) return rc;
            CLATCH_CUDA(cudaMemcpy(pat.slots.ptr, sw.slots.data(), sizeof(SlotEntry) * T, cudaMemcpyHostToDevice));
            pat.slots_planned = true;
        }
        if (int rc = pat.slots_h16.reserve(sizeof(SlotEntry) * T)) return rc;
        if (triplet_hash(triplets, T) == kDefaultPlanHash && kDefaultPlanH16RowWords == kH16RowWords) {
            static_assert(sizeof(kDefaultPlanH16) == sizeof(SlotEntry) * kFastT, "embedded plan size");
            pat.slot_degree_h16 = kDefaultPlanH16Degree;
            CLATCH_CUDA(cudaMemcpy(pat.slots_h16.ptr, kDefaultPlanH16, sizeof(kDefaultPlanH16), cudaMemcpyHostToDevice));
        } else {
            const SlotPlan h16 = plan_slots_h16(triplets, T, 1500000);
            pat.slot_degree_h16 = h16.avg_degree;
            CLATCH_CUDA(cudaMemcpy(pat.slots_h16.ptr, h16.slots.data(), sizeof(SlotEntry) * T, cudaMemcpyHostToDevice));
        }
    }
    return CLATCH_OK;
}

} // extern "C"

namespace {

// keypoint_in_margin over the whole list (src/descriptor.cpp:23-27, 94-97; NaN fails every comparison):
// kept[0..count) = input indices that keep the 46 px margin, in input order.
size_t margin_filter(const double* kps, size_t n, int cols, int width, int height, int64_t* kept) {
    const double xmax = static_cast<double>(width - 1), ymax = static_cast<double>(height - 1);
    size_t count = 0;
    for (size_t i = 0; i < n; ++i) {
        const double x = kps[i * cols], y = kps[i * cols + 1];
        if (x - kMargin >= 0.0 && y - kMargin >= 0.0 && x + kMargin <= xmax && y + kMargin <= ymax)
            kept[count++] = static_cast<int64_t>(i);
    }
    return count;
}

// cos/sin of extract_window (src/descriptor.cpp:35-36) through the host libm: record j of xycs comes
// from input keypoint src[j]. Chunks of 256 records are claimed from a shared counter, so the calling
// thread starts at once and the workers join in as they wake up.
int trig_pass(const double* kps, int cols, const int64_t* src, size_t count, int workers, double* xycs) {
    if (count == 0) return CLATCH_OK;
    int nthreads = std::min<size_t>(resolve_workers(workers), (count + 1023) / 1024);
    nthreads = std::max(nthreads, 1);
    std::vector<int> bad(nthreads, 0);
    // Records written by many cores and read next by the copy engine: with ordinary stores the DMA has
    // to snoop them out of the cores' caches (measured 6 GB/s for the 1.6 MB of 50 k records instead of
    // 50 GB/s); non-temporal stores put them in memory.
    const bool streaming = reinterpret_cast<uintptr_t>(xycs) % 16 == 0 && std::getenv("CLATCH_NO_STREAM_STORES") == nullptr;
    std::atomic<size_t> next_chunk{0};
    constexpr size_t kChunk = 256;
    auto work = [&](int w) {
        for (;;) {
            const size_t begin = next_chunk.fetch_add(kChunk, std::memory_order_relaxed);
            if (begin >= count) break;
            const size_t end = std::min(count, begin + kChunk);
            for (size_t j = begin; j < end; ++j) {
                const double* k = kps + static_cast<size_t>(src[j]) * cols;
                const double theta = cols > 2 ? k[2] : 0.0;
                const double c = std::cos(theta), s = std::sin(theta);
                if (!std::isfinite(c) || !std::isfinite(s)) bad[w] = 1;
#if defined(__SSE2__)
                if (streaming) {   // straight to memory: the DMA engine reads these lines next, not a CPU
                    _mm_stream_pd(xycs + 4 * j, _mm_set_pd(k[1], k[0]));
                    _mm_stream_pd(xycs + 4 * j + 2, _mm_set_pd(s, c));
                    continue;
                }
#endif
                xycs[4 * j + 0] = k[0];
                xycs[4 * j + 1] = k[1];
                xycs[4 * j + 2] = c;
                xycs[4 * j + 3] = s;
            }
        }
#if defined(__SSE2__)
        if (streaming) _mm_sfence();
#endif
    };
    WorkerPool::instance().run(nthreads, work);
    for (int b : bad)
        if (b) {
            set_error("a keypoint inside the margin has a non-finite orientation");
            return CLATCH_ERR_NONFINITE;
        }
    return CLATCH_OK;
}

} // namespace

extern "C" {

int clatch_take_keypoints(const double* kps, int cols, const int64_t* kept, size_t m, int workers, double* out) {
    if (cols < 2 || cols > 4) return invalid("keypoints must be (N, 2..4): x, y[, theta[, score]]");
    if (m == 0) return CLATCH_OK;
    if (!kps || !kept || !out) return invalid("clatch_take_keypoints: null buffer");
    // (below ~16 k rows the gather costs less than waking a worker)
    const int parts = static_cast<int>(std::max<size_t>(1, std::min<size_t>(resolve_workers(workers), m / 16384)));
    std::atomic<size_t> next{0};
    WorkerPool::instance().run(parts, [&](int) {
        for (;;) {
            const size_t begin = next.fetch_add(2048, std::memory_order_relaxed);
            if (begin >= m) break;
            const size_t end = std::min(m, begin + 2048);
            for (size_t j = begin; j < end; ++j) {
                const double* k = kps + static_cast<size_t>(kept[j]) * cols;
                double* o = out + 4 * j;
                o[0] = k[0];
                o[1] = k[1];
                o[2] = cols > 2 ? k[2] : 0.0;   // missing theta / score read as 0 (bindings/module.cpp:49-62)
                o[3] = cols > 3 ? k[3] : 0.0;
            }
        }
    });
    return CLATCH_OK;
}

int clatch_prepare_keypoints(const double* kps, size_t n, int cols, int width, int height,
                             int workers, double* xycs, int64_t* kept, size_t* m) {
    if (!m) return invalid("clatch_prepare_keypoints: m is null");
    *m = 0;
    if (cols < 2 || cols > 4) return invalid("keypoints must be (N, 2..4): x, y[, theta[, score]]");
    if (n == 0) return CLATCH_OK;
    if (!kps || !xycs || !kept) return invalid("clatch_prepare_keypoints: null buffer");
    const size_t count = margin_filter(kps, n, cols, width, height, kept);
    *m = count;
    return trig_pass(kps, cols, kept, count, workers, xycs);
}

// ---- extraction ---------------------------------------------------------------

static int check_extract(clatch_ctx* ctx, const void* img, int width, int height, size_t pitch,
                         const void* xycs, size_t M, const void* out) {
    if (!ctx) return invalid("extract: ctx is null");
    if (ctx->pattern.T == 0) return invalid("extract: no pattern installed (clatch_set_pattern)");
    if (!img || width <= 0 || height <= 0 || pitch < static_cast<size_t>(width))
        return invalid("extract: bad image (null, empty or pitch < width)");
    if (M > 0 && (!xycs || !out)) return invalid("extract: null keypoint/output buffer");
    return CLATCH_OK;
}

int clatch_extract_u8_dev(clatch_ctx* ctx, const uint8_t* d_img, int width, int height,
                          size_t pitch, const double* d_xycs, size_t M, uint8_t* d_out,
                          void* stream) {
    if (int rc = check_extract(ctx, d_img, width, height, pitch, d_xycs, M, d_out)) return rc;
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    return launch_extract_u8(ctx, d_img, width, height, pitch, d_xycs, M, d_out,
                             static_cast<cudaStream_t>(stream));
}

int clatch_estimate_planes_u8_dev(clatch_ctx* ctx, const uint8_t* d_img, int width, int height, size_t pitch,
                                  const double* d_xycs, size_t M, uint16_t* d_out, void* stream) {
    if (int rc = check_extract(ctx, d_img, width, height, pitch, d_xycs, M, d_out)) return rc;
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    return launch_estimate_planes_u8(ctx, d_img, width, height, pitch, d_xycs, M, d_out, static_cast<cudaStream_t>(stream));
}

int clatch_extract_f64_dev(clatch_ctx* ctx, const double* d_img, int width, int height,
                           size_t pitch, const double* d_xycs, size_t M, uint8_t* d_out,
                           void* stream) {
    if (int rc = check_extract(ctx, d_img, width, height, pitch, d_xycs, M, d_out)) return rc;
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    return launch_extract_f64(ctx, d_img, width, height, pitch, d_xycs, M, d_out,
                              static_cast<cudaStream_t>(stream));
}

int clatch_extract_u8(clatch_ctx* ctx, const uint8_t* img, int width, int height, size_t pitch,
                      const double* xycs, size_t M, uint8_t* out) {
    if (int rc = check_extract(ctx, img, width, height, pitch, xycs, M, out)) return rc;
    if (M == 0) return CLATCH_OK;
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    const size_t dpitch = (static_cast<size_t>(width) + 15) / 16 * 16;   // 16-byte rows for vector staging
    const size_t bytes = static_cast<size_t>(ctx->pattern.T) / 8;
    if (int rc = ctx->img.reserve(dpitch * height)) return rc;
    if (int rc = ctx->kps.reserve(sizeof(double) * 4 * M)) return rc;
    if (int rc = ctx->desc.reserve(bytes * M)) return rc;
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpy2DAsync(ctx->img.ptr, dpitch, img, pitch, width, height,
                                  cudaMemcpyHostToDevice, st));
    CLATCH_CUDA(cudaMemcpyAsync(ctx->kps.ptr, xycs, sizeof(double) * 4 * M, cudaMemcpyHostToDevice, st));
    if (int rc = launch_extract_u8(ctx, ctx->img.as<uint8_t>(), width, height, dpitch,
                                   ctx->kps.as<double>(), M, ctx->desc.as<uint8_t>(), st))
        return rc;
    CLATCH_CUDA(cudaMemcpyAsync(out, ctx->desc.ptr, bytes * M, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    return CLATCH_OK;
}

int clatch_extract_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch,
                       const double* xycs, size_t M, uint8_t* out) {
    if (int rc = check_extract(ctx, img, width, height, pitch, xycs, M, out)) return rc;
    if (M == 0) return CLATCH_OK;
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    const size_t bytes = static_cast<size_t>(ctx->pattern.T) / 8;
    if (int rc = ctx->img.reserve(sizeof(double) * width * height)) return rc;
    if (int rc = ctx->kps.reserve(sizeof(double) * 4 * M)) return rc;
    if (int rc = ctx->desc.reserve(bytes * M)) return rc;
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpy2DAsync(ctx->img.ptr, sizeof(double) * width, img, sizeof(double) * pitch,
                                  sizeof(double) * width, height, cudaMemcpyHostToDevice, st));
    CLATCH_CUDA(cudaMemcpyAsync(ctx->kps.ptr, xycs, sizeof(double) * 4 * M, cudaMemcpyHostToDevice, st));
    if (int rc = launch_extract_f64(ctx, ctx->img.as<double>(), width, height, width,
                                    ctx->kps.as<double>(), M, ctx->desc.as<uint8_t>(), st))
        return rc;
    CLATCH_CUDA(cudaMemcpyAsync(out, ctx->desc.ptr, bytes * M, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    return CLATCH_OK;
}

} // extern "C"

// describe_all. The image DMA is queued first so that it overlaps the host-side margin filter
// and trig pass. Optionally (see `bands` below) the image goes up in row bands on a copy stream,
// keypoints are bucketed by the band in which their 92-row footprint ends, and each bucket's
// extraction is queued behind that band's arrival event.
static int describe_all_bands_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch,
                                  const double* kps, size_t n, int cols, int workers, int64_t* kept, uint8_t* out,
                                  size_t* m, int bands);

// promote_rows_u8 over the whole image on the host workers; false if some pixel is not a u8 value.
static bool promote_image_u8(const double* img, size_t pitch, uint8_t* staged, size_t upitch, int width, int height,
                             int workers) {
    const int parts = std::max(1, std::min(resolve_workers(workers), height / 8));
    std::vector<int> ok(parts, 0);
    const int rows = (height + parts - 1) / parts;
    WorkerPool::instance().run(parts, [&](int w) {
        const int r0 = std::min(height, w * rows), r1 = std::min(height, r0 + rows);
        ok[w] = promote_rows_u8(img, pitch, staged, upitch, width, r0, r1);
    });
    for (int v : ok)
        if (!v) return false;
    return true;
}

// Rows [0, height) of a u8 image into page-locked staging with pitch `dpitch`, on the host workers.
static void stage_rows_u8(const uint8_t* src, size_t pitch, uint8_t* dst, size_t dpitch, int width, int height, int workers) {
    const int parts = std::max(1, std::min(resolve_workers(workers), height / 64));
    const int rows = (height + parts - 1) / parts;
    WorkerPool::instance().run(parts, [&](int w) {
        const int r0 = std::min(height, w * rows), r1 = std::min(height, r0 + rows);
        if (pitch == dpitch && pitch == static_cast<size_t>(width)) {
            if (r1 > r0) std::memcpy(dst + static_cast<size_t>(r0) * dpitch, src + static_cast<size_t>(r0) * pitch, static_cast<size_t>(r1 - r0) * pitch);
        } else {
            for (int r = r0; r < r1; ++r) std::memcpy(dst + static_cast<size_t>(r) * dpitch, src + static_cast<size_t>(r) * pitch, width);
        }
    });
}

template <typename Pixel>
static int describe_all_impl(clatch_ctx* ctx, const Pixel* img, int width, int height, size_t pitch,
                             const double* kps, size_t n, int cols, int workers, int64_t* kept,
                             uint8_t* out, size_t* m) {
    if (!m) return invalid("describe_all: m is null");
    *m = 0;
    if (int rc = check_extract(ctx, img, width, height, pitch, kps, 0, out)) return rc;
    if (cols < 2 || cols > 4) return invalid("keypoints must be (N, 2..4): x, y[, theta[, score]]");
    if (n == 0) return CLATCH_OK;
    if (!kps || !kept || !out) return invalid("describe_all: null keypoint/output buffer");
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    constexpr bool kU8 = sizeof(Pixel) == 1;
    if (!kU8 && n >= 256 && want_host_promote(ctx, img)) {
        // float64 image: try the lossless u8 promotion on the host workers first (page-locked
        // staging); a non-u8-valued image stops at its first such pixel and takes the f64 route.
        const size_t upitch = (static_cast<size_t>(width) + 15) / 16 * 16;
        if (int rc = ctx->pin_img.reserve(upitch * height)) return rc;
        uint8_t* const staged = static_cast<uint8_t*>(ctx->pin_img.ptr);
        if (promote_image_u8(reinterpret_cast<const double*>(img), pitch, staged, upitch, width, height, workers))
            return describe_all_impl<uint8_t>(ctx, staged, width, height, upitch, kps, n, cols, workers, kept, out, m);
    }
    if (!kU8) {
        // float64: upload in row bands when the frame is big enough for the overlap to pay
        const size_t image_bytes = sizeof(double) * static_cast<size_t>(width) * height;
        int bands = ctx->upload_bands;
        if (const char* env = std::getenv("CLATCH_UPLOAD_BANDS")) bands = std::atoi(env);
        // auto: two bands. More bands shorten the tail that cannot overlap (the last band's extraction) but
        // each costs ~50 us of host-side launches, which delays everything behind it: 1920x1080 with 10 k
        // keypoints takes 535 us in one piece, 454 / 523 / 549 us in 2 / 3 / 4 bands; 3840x2160 with 50 k
        // keypoints 2.23 ms in one piece, 1.81 / 2.10 / 2.28 ms in 2 / 4 / 6.
        if (bands <= 0) {
            bands = 2;
            // A frame that is visibly not u8-valued goes up in one piece: its keypoints then take the packed-plane kernel
            // over a float texture of the whole frame (51 M desc/s), which needs the frame's value range before the first
            // keypoint is extracted; in bands they would run the all-fp64 kernel (19 M desc/s). 256 probes on the host.
            const double* const px = reinterpret_cast<const double*>(img);
            uint64_t lcg = 0x9E3779B97F4A7C15ull;
            for (int i = 0; i < 256; ++i) {
                lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
                const size_t y = static_cast<size_t>((lcg >> 33) % static_cast<uint64_t>(height));
                const size_t x = static_cast<size_t>((lcg >> 13) % static_cast<uint64_t>(width));
                const double v = px[y * pitch + x];
                if (!(v >= 0.0 && v <= 255.0 && v == std::floor(v))) {
                    bands = 1;
                    break;
                }
            }
        }
        bands = std::max(1, std::min(6, bands));
        if (bands > 1 && n >= 4096 && image_bytes >= (4u << 20) && height >= 64 * bands && n < 0xffffffffull &&
            extract_supports_out_index(ctx))
            return describe_all_bands_f64(ctx, reinterpret_cast<const double*>(img), width, height, pitch, kps, n, cols,
                                          workers, kept, out, m, bands);
    }
    const size_t dpitch = kU8 ? (static_cast<size_t>(width) + 15) / 16 * 16 : static_cast<size_t>(width);
    const size_t bytes = static_cast<size_t>(ctx->pattern.T) / 8;
    if (int rc = ctx->img.reserve(sizeof(Pixel) * dpitch * height)) return rc;
    if (int rc = ctx->kps.reserve(sizeof(double) * 4 * n)) return rc;
    if (int rc = ctx->desc.reserve(bytes * n)) return rc;
    if (int rc = ctx->pin_xycs.reserve(sizeof(double) * 4 * n)) return rc;
    cudaStream_t st = ctx->stream;

    Trace trace;
    // 1. image DMA first ...
    if (kU8 && static_cast<size_t>(width) * height >= (256u << 10) && static_cast<const void*>(img) != ctx->pin_img.ptr &&
        is_pageable(img)) {
        // ... a big pageable u8 image: gathered into page-locked staging by the workers, then one flat DMA
        if (int rc = ctx->pin_img.reserve(dpitch * height)) return rc;
        stage_rows_u8(reinterpret_cast<const uint8_t*>(img), pitch, static_cast<uint8_t*>(ctx->pin_img.ptr), dpitch, width,
                      height, workers);
        CLATCH_CUDA(cudaMemcpyAsync(ctx->img.ptr, ctx->pin_img.ptr, dpitch * height, cudaMemcpyHostToDevice, st));
    } else if (!kU8 && sizeof(Pixel) * static_cast<size_t>(width) * height >= (4u << 20) && height >= 64 &&
               static_cast<const void*>(img) != ctx->pin_img.ptr && is_pageable(img) &&
               (ctx->pin_img.cap >= sizeof(Pixel) * static_cast<size_t>(width) * height || ++ctx->pageable_f64_frames >= 2)) {
        // (from the second such frame on, or when the staging is already there: page-locking 16.6 MB takes ~50 ms once)
        // ... a big float64 frame in ordinary memory (one that is not u8-valued, or host_promote = never): the driver
        // would bounce it through its own staging at ~13 GB/s; instead the workers copy it into page-locked staging in
        // eight row chunks and each chunk's DMA runs while the next one is being copied.
        const size_t row_bytes = sizeof(Pixel) * static_cast<size_t>(width);
        if (int rc = ctx->pin_img.reserve(row_bytes * height)) return rc;
        uint8_t* const staging = static_cast<uint8_t*>(ctx->pin_img.ptr);
        const uint8_t* const src = reinterpret_cast<const uint8_t*>(img);
        const size_t src_pitch = sizeof(Pixel) * pitch;
        const int chunks = 8, rows_per = (height + chunks - 1) / chunks;
        for (int c = 0; c < chunks; ++c) {
            const int c0 = std::min(height, c * rows_per), c1 = std::min(height, c0 + rows_per);
            if (c1 <= c0) break;
            const int parts = std::max(1, std::min(resolve_workers(workers), (c1 - c0) / 8));
            const int rows = (c1 - c0 + parts - 1) / parts;
            WorkerPool::instance().run(parts, [&](int w) {
                const int r0 = std::min(c1, c0 + w * rows), r1 = std::min(c1, r0 + rows);
                for (int r = r0; r < r1; ++r) std::memcpy(staging + static_cast<size_t>(r) * row_bytes, src + static_cast<size_t>(r) * src_pitch, row_bytes);
            });
            CLATCH_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(ctx->img.ptr) + static_cast<size_t>(c0) * row_bytes,
                                        staging + static_cast<size_t>(c0) * row_bytes, row_bytes * (c1 - c0), cudaMemcpyHostToDevice, st));
        }
    } else
    CLATCH_CUDA(cudaMemcpy2DAsync(ctx->img.ptr, sizeof(Pixel) * dpitch, img, sizeof(Pixel) * pitch,
                                  sizeof(Pixel) * width, height, cudaMemcpyHostToDevice, st));
    // 2. ... while the host filters by margin and evaluates cos/sin with its own libm
    double* const xycs = static_cast<double*>(ctx->pin_xycs.ptr);
    size_t count = 0;
    trace.stamp("image copy queued");
    if (int rc = clatch_prepare_keypoints(kps, n, cols, width, height, workers, xycs, kept, &count)) {
        cudaStreamSynchronize(st);
        return rc;
    }
    trace.stamp("keypoints prepared");
    *m = count;
    if (count == 0) {
        cudaStreamSynchronize(st);
        return CLATCH_OK;
    }
    cudaEvent_t tev[4] = {};
    if (trace.on) {
        for (cudaEvent_t& e : tev) cudaEventCreate(&e);
        cudaEventRecord(tev[0], st);   // image copy done (stream order)
    }
    CLATCH_CUDA(cudaMemcpyAsync(ctx->kps.ptr, xycs, sizeof(double) * 4 * count, cudaMemcpyHostToDevice, st));
    if (trace.on) cudaEventRecord(tev[1], st);
    // 3. extraction (a float64 image is classified first: u8-valued -> the u8 kernels)
    int rc;
    if (kU8)
        rc = launch_extract_u8(ctx, ctx->img.as<uint8_t>(), width, height, dpitch, ctx->kps.as<double>(), count,
                               ctx->desc.as<uint8_t>(), st);
    else
        rc = launch_extract_f64(ctx, ctx->img.as<double>(), width, height, dpitch, ctx->kps.as<double>(), count,
                                ctx->desc.as<uint8_t>(), st);
    if (rc) {
        cudaStreamSynchronize(st);
        return rc;
    }
    trace.stamp("kernels queued");
    if (trace.on) cudaEventRecord(tev[2], st);
    // 4. descriptors straight into the caller's array
    CLATCH_CUDA(cudaMemcpyAsync(out, ctx->desc.ptr, bytes * count, cudaMemcpyDeviceToHost, st));
    trace.stamp("download queued");
    if (trace.on) cudaEventRecord(tev[3], st);
    CLATCH_CUDA(cudaStreamSynchronize(st));
    trace.stamp("stream drained");
    if (trace.on) {
        float a = 0, b = 0, c = 0;
        cudaEventElapsedTime(&a, tev[0], tev[1]);
        cudaEventElapsedTime(&b, tev[1], tev[2]);
        cudaEventElapsedTime(&c, tev[2], tev[3]);
        std::fprintf(stderr, "[clatch] device: keypoint upload %.1f us, kernels %.1f us, download %.1f us\n", a * 1e3,
                     b * 1e3, c * 1e3);
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    return CLATCH_OK;
}

// float64 images are eight bytes a pixel: the upload of a 1920x1080 frame (16.6 MB, 0.33 ms over PCIe 5)
// takes twice as long as extracting 10 k descriptors from it. So the frame goes up in row bands and the
// keypoints whose footprints (rows floor(y)-45 .. floor(y)+46) end inside band b are extracted while
// band b+1 is still in flight. Order of the H2D queue matters — one copy engine serves it in issue
// order — so: band 0, then the keypoint records (ready by then: the host prepared them meanwhile),
// then the other bands. Records are prepared in band order; the kernels write each descriptor to its
// input-order row (ExtractParams::out_index), so the download is one contiguous copy again.
// Classification is per band and cumulative (launch_classify_rows): a band whose rows are all
// u8-valued so far takes the u8 kernel, and a keypoint only ever reads rows of its own and earlier bands.
static int describe_all_bands_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch,
                                  const double* kps, size_t n, int cols, int workers, int64_t* kept, uint8_t* out,
                                  size_t* m, int bands) {
    const size_t dpitch = static_cast<size_t>(width), bytes = static_cast<size_t>(ctx->pattern.T) / 8;
    const size_t rec_bytes = sizeof(double) * 4 * n, idx_bytes = sizeof(unsigned) * n;
    if (int rc = ctx->img.reserve(sizeof(double) * dpitch * height)) return rc;
    if (int rc = ctx->kps.reserve(rec_bytes + idx_bytes)) return rc;
    if (int rc = ctx->desc.reserve(bytes * n)) return rc;
    if (int rc = ctx->pin_xycs.reserve(rec_bytes + idx_bytes)) return rc;
    cudaStream_t st = ctx->stream;
    if (!ctx->copy_stream) {
        CLATCH_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (cudaEvent_t& e : ctx->band_events) CLATCH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaStream_t cs = ctx->copy_stream;
    Trace trace;
    // Band heights: band b+1 should land just as band b's keypoints are done, so that neither the copy
    // engine nor the SMs wait — heights in geometric progression with ratio (extraction time) / (upload
    // time), which for a 1920x1080 frame with 10 k keypoints is about 0.5: a tall first band, a short
    // last one, and only the last band's extraction is left when the upload ends.
    int row_end[8];
    {
        const double upload_s = sizeof(double) * static_cast<double>(width) * height / 50e9;
        const double extract_s = 20e-6 + 17.5e-9 * static_cast<double>(n);
        const double ratio = std::min(3.0, std::max(0.3, extract_s / upload_s));
        double weight[8], total = 0.0, w = 1.0;
        for (int b = 0; b < bands; ++b, w *= ratio) total += weight[b] = w;
        double cum = 0.0;
        int prev = 0;
        for (int b = 0; b < bands; ++b) {
            cum += weight[b] / total;
            int end = b == bands - 1 ? height : static_cast<int>(std::lround(cum * height));
            end = std::min(height - 48 * (bands - 1 - b), std::max(prev + 48, end));   // every band at least 48 rows
            row_end[b] = prev = end;
        }
        row_end[bands - 1] = height;
    }
    auto copy_band = [&](int b) -> int {
        const int r0 = b == 0 ? 0 : row_end[b - 1], r1 = row_end[b];
        double* dst = ctx->img.as<double>() + static_cast<size_t>(r0) * dpitch;
        const double* src = img + static_cast<size_t>(r0) * pitch;
        if (pitch == dpitch)   // contiguous rows: one flat DMA
            CLATCH_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * dpitch * (r1 - r0), cudaMemcpyHostToDevice, cs));
        else
            CLATCH_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * dpitch, src, sizeof(double) * pitch, sizeof(double) * width,
                                          r1 - r0, cudaMemcpyHostToDevice, cs));
        CLATCH_CUDA(cudaEventRecord(ctx->band_events[b], cs));
        return CLATCH_OK;
    };
    auto drain = [&] {
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(st);
    };
    // the copy stream must not overwrite the image while earlier work on `st` still reads it
    CLATCH_CUDA(cudaEventRecord(ctx->band_events[7], st));
    CLATCH_CUDA(cudaStreamWaitEvent(cs, ctx->band_events[7], 0));
    if (int rc = copy_band(0)) return rc;
    trace.stamp("band 0 copy queued");

    // host, meanwhile: margin filter, band of every kept keypoint, records in band order
    const size_t count = margin_filter(kps, n, cols, width, height, kept);
    *m = count;
    if (count == 0) {
        drain();
        return CLATCH_OK;
    }
    std::vector<int64_t>& src = ctx->band_src;      // record j <- input keypoint src[j]
    src.resize(count);
    unsigned* const h_index = reinterpret_cast<unsigned*>(static_cast<uint8_t*>(ctx->pin_xycs.ptr) + rec_bytes);
    size_t begin[9] = {0};
    {
        std::vector<uint8_t>& band_of = ctx->band_of;
        band_of.resize(count);
        size_t hist[9] = {0};
        for (size_t j = 0; j < count; ++j) {
            const int bottom = static_cast<int>(std::floor(kps[static_cast<size_t>(kept[j]) * cols + 1])) + 46;
            int b = 0;
            while (b < bands - 1 && bottom >= row_end[b]) ++b;   // first band that holds the footprint's last row
            band_of[j] = static_cast<uint8_t>(b);
            ++hist[b + 1];
        }
        for (int b = 0; b < bands; ++b) begin[b + 1] = begin[b] + hist[b + 1];
        size_t cursor[8];
        for (int b = 0; b < bands; ++b) cursor[b] = begin[b];
        for (size_t j = 0; j < count; ++j) {       // stable: input order inside a band
            const size_t slot = cursor[band_of[j]]++;
            src[slot] = kept[j];
            h_index[slot] = static_cast<unsigned>(j);
        }
    }
    double* const xycs = static_cast<double*>(ctx->pin_xycs.ptr);
    if (int rc = trig_pass(kps, cols, src.data(), count, workers, xycs)) {
        drain();
        return rc;
    }
    trace.stamp("keypoints prepared");
    // records + output rows ride the H2D queue right behind band 0, ahead of the other bands
    uint8_t* const d_rec = ctx->kps.as<uint8_t>();
    CLATCH_CUDA(cudaMemcpyAsync(d_rec, xycs, sizeof(double) * 4 * count, cudaMemcpyHostToDevice, cs));
    CLATCH_CUDA(cudaMemcpyAsync(d_rec + rec_bytes, h_index, sizeof(unsigned) * count, cudaMemcpyHostToDevice, cs));
    CLATCH_CUDA(cudaEventRecord(ctx->band_events[7], cs));
    for (int b = 1; b < bands; ++b)
        if (int rc = copy_band(b)) {
            drain();
            return rc;
        }
    CLATCH_CUDA(cudaStreamWaitEvent(st, ctx->band_events[7], 0));
    trace.stamp("copies queued");
    int rc = CLATCH_OK;
    ctx->extract_out_index = reinterpret_cast<const unsigned*>(d_rec + rec_bytes);
    for (int b = 0; b < bands && !rc; ++b) {
        const int r0 = b == 0 ? 0 : row_end[b - 1], r1 = row_end[b];
        if (cudaError_t e = cudaStreamWaitEvent(st, ctx->band_events[b], 0); e != cudaSuccess) {
            rc = cuda_fail(e, "cudaStreamWaitEvent(band)");
            break;
        }
        rc = launch_classify_rows(ctx, ctx->img.as<double>(), width, height, dpitch, r0, r1, b == 0, st);
        const size_t cnt = begin[b + 1] - begin[b];
        if (!rc && cnt > 0) {
            ctx->extract_out_index = reinterpret_cast<const unsigned*>(d_rec + rec_bytes) + begin[b];
            rc = launch_extract_f64_classified(ctx, ctx->img.as<double>(), width, height, dpitch,
                                               reinterpret_cast<const double*>(d_rec) + 4 * begin[b], cnt,
                                               ctx->desc.as<uint8_t>(), st);
        }
    }
    ctx->extract_out_index = nullptr;
    if (rc) {
        drain();
        return rc;
    }
    trace.stamp("kernels queued");
    CLATCH_CUDA(cudaMemcpyAsync(out, ctx->desc.ptr, bytes * count, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    trace.stamp("stream drained");
    return CLATCH_OK;
}

template <typename Pixel>
static int detect_impl(clatch_ctx* ctx, const Pixel* img, int width, int height, size_t pitch, double threshold,
                       int nms, int orient, int radius, double* out, size_t cap, size_t* count) {
    if (!count) return invalid("detect: count is null");
    *count = 0;
    if (!ctx) return invalid("detect: ctx is null");
    if (!img || width <= 0 || height <= 0 || pitch < static_cast<size_t>(width))
        return invalid("detect: bad image (null, empty or pitch < width)");
    if (width < 7 || height < 7) {   // src/detect.cpp:77-78
        set_error("ImageTooSmall: FAST needs at least a 7x7 image");
        return CLATCH_ERR_IMAGE_TOO_SMALL;
    }
    if (radius < 0 || !std::isfinite(threshold)) return invalid("detect: bad radius or threshold");
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    if (int rc = ctx->img.reserve(sizeof(Pixel) * static_cast<size_t>(width) * height)) return rc;
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpy2DAsync(ctx->img.ptr, sizeof(Pixel) * width, img, sizeof(Pixel) * pitch,
                                  sizeof(Pixel) * width, height, cudaMemcpyHostToDevice, st));
    unsigned total = 0;
    int rc;
    if (sizeof(Pixel) == 1)
        rc = launch_detect_u8(ctx, ctx->img.as<uint8_t>(), width, height, width, threshold, nms, orient, radius, st,
                              &total);
    else
        rc = launch_detect_f64(ctx, ctx->img.as<double>(), width, height, width, threshold, nms, orient, radius, st,
                               &total);
    if (rc) return rc;
    if (total == 0) return CLATCH_OK;
    std::vector<Detection> det(total);
    CLATCH_CUDA(cudaMemcpyAsync(det.data(), ctx->det.ptr, sizeof(Detection) * total, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    size_t m = 0;
    for (const Detection& d : det) {
        if (orient && !d.valid) continue;   // disc leaves the image, src/detect.cpp:152-154
        if (m < cap && out) {
            out[4 * m + 0] = static_cast<double>(d.x);
            out[4 * m + 1] = static_cast<double>(d.y);
            // src/detect.cpp:144 — host libm, like the reference
            out[4 * m + 2] = orient ? ((d.m10 == 0.0 && d.m01 == 0.0) ? 0.0 : std::atan2(d.m01, d.m10)) : 0.0;
            out[4 * m + 3] = d.score;
        }
        ++m;
    }
    *count = m;
    if (m > cap) return invalid("detect: output buffer too small (see *count)");
    return CLATCH_OK;
}

// Two-slot software pipeline over images: slot = i % 2 owns a stream and its own device
// scratch, so image i+1 uploads / prepares while image i computes and downloads.
// Inside describe_batch's image loop a CUDA failure must not return: the other pipeline stream may still
// be writing into caller arrays and a slot may hold a pending copy. Record it and leave through the
// common epilogue, which drains both streams and clears the pending state.
#define BATCH_CUDA(expr)                                    \
    if (cudaError_t e_ = (expr); e_ != cudaSuccess) {       \
        rc = ::clatch::cuda_fail(e_, #expr);                \
        break;                                              \
    } else                                                  \
        (void)0

template <typename Pixel>
static int describe_batch_impl(clatch_ctx* ctx, const Pixel* const* imgs, const int* widths, const int* heights,
                               const size_t* pitches, const double* const* kps, const size_t* counts, int cols,
                               size_t num_images, int workers, int64_t* const* kept, uint8_t* const* out, size_t* m) {
    if (!ctx) return invalid("describe_batch: ctx is null");
    if (num_images == 0) return CLATCH_OK;
    if (!imgs || !widths || !heights || !pitches || !kps || !counts || !kept || !out || !m)
        return invalid("describe_batch: null array");
    if (ctx->pattern.T == 0) return invalid("extract: no pattern installed (clatch_set_pattern)");
    if (cols < 2 || cols > 4) return invalid("keypoints must be (N, 2..4): x, y[, theta[, score]]");
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    constexpr bool kU8 = sizeof(Pixel) == 1;
    const size_t bytes = static_cast<size_t>(ctx->pattern.T) / 8;
    for (int s = 0; s < 2; ++s)
        if (!ctx->pipe[s].stream) CLATCH_CUDA(cudaStreamCreateWithFlags(&ctx->pipe[s].stream, cudaStreamNonBlocking));
    int rc = CLATCH_OK;
    Trace trace;
    std::vector<cudaEvent_t> bev;   // trace mode: per image {upload done, kernels done, download done}, + origin
    if (trace.on) {
        bev.resize(3 * num_images + 1);
        for (cudaEvent_t& e : bev) cudaEventCreate(&e);
        cudaEventRecord(bev[3 * num_images], ctx->pipe[0].stream);
    }
    for (size_t i = 0; i < num_images && !rc; ++i) {
        clatch_ctx::PipeSlot& slot = ctx->pipe[i & 1];
        cudaStream_t st = slot.stream;
        m[i] = 0;
        const int w = widths[i], h = heights[i];
        const size_t n = counts[i];
        if (!imgs[i] || w <= 0 || h <= 0 || pitches[i] < static_cast<size_t>(w)) {
            rc = invalid("describe_batch: bad image (null, empty or pitch < width)");
            break;
        }
        if (n == 0) continue;
        if (!kps[i] || !kept[i] || !out[i]) {
            rc = invalid("describe_batch: null keypoint/output buffer");
            break;
        }
        // the slot's previous image (i-2) must have left its buffers before they are reused;
        // its descriptors wait in page-locked staging and move to the caller's array now
        trace.stamp("batch: image begins");
        BATCH_CUDA(cudaStreamSynchronize(st));
        trace.stamp("batch: slot free");
        if (slot.pending_out) {
            std::memcpy(slot.pending_out, slot.h_desc.ptr, slot.pending_bytes);
            slot.pending_out = nullptr;
        }
        const size_t dpitch = kU8 ? (static_cast<size_t>(w) + 15) / 16 * 16 : static_cast<size_t>(w);
        const size_t u8_pitch = (static_cast<size_t>(w) + 15) / 16 * 16;
        if ((rc = slot.kps.reserve(sizeof(double) * 4 * n))) break;
        if ((rc = slot.desc.reserve(bytes * n))) break;
        bool promoted = false;   // float64 image sent up as its lossless u8 copy (host workers, page-locked staging)
        if (!kU8) {
            if ((rc = slot.img_u8.reserve(u8_pitch * h))) break;
            if ((rc = slot.flags.reserve(64))) break;   // the flag block (clatch_extract.cu: kFlagBlockBytes)
            if (n >= 256 && want_host_promote(ctx, imgs[i])) {
                if ((rc = slot.h_img.reserve(u8_pitch * h))) break;
                promoted = promote_image_u8(reinterpret_cast<const double*>(imgs[i]), pitches[i],
                                            static_cast<uint8_t*>(slot.h_img.ptr), u8_pitch, w, h, workers);
                trace.stamp(promoted ? "batch: image promoted to u8 on the host" : "batch: image is not u8-valued");
            }
        }
        if (promoted) {
            BATCH_CUDA(cudaMemcpyAsync(slot.img_u8.ptr, slot.h_img.ptr, u8_pitch * h, cudaMemcpyHostToDevice, st));
        } else if (kU8 && static_cast<size_t>(w) * h >= (256u << 10) && is_pageable(imgs[i])) {
            // big pageable u8 image: workers gather it into page-locked staging, one flat DMA (see is_pageable)
            if ((rc = slot.img.reserve(dpitch * h))) break;
            if ((rc = slot.h_img.reserve(dpitch * h))) break;
            stage_rows_u8(reinterpret_cast<const uint8_t*>(imgs[i]), pitches[i], static_cast<uint8_t*>(slot.h_img.ptr), dpitch, w, h,
                          workers);
            BATCH_CUDA(cudaMemcpyAsync(slot.img.ptr, slot.h_img.ptr, dpitch * h, cudaMemcpyHostToDevice, st));
        } else {
            if ((rc = slot.img.reserve(sizeof(Pixel) * dpitch * h))) break;
            BATCH_CUDA(cudaMemcpy2DAsync(slot.img.ptr, sizeof(Pixel) * dpitch, imgs[i], sizeof(Pixel) * pitches[i],
                                         sizeof(Pixel) * w, h, cudaMemcpyHostToDevice, st));
        }
        if ((rc = slot.h_xycs.reserve(sizeof(double) * 4 * n))) break;
        if ((rc = slot.h_desc.reserve(bytes * n))) break;
        double* const xycs = static_cast<double*>(slot.h_xycs.ptr);
        size_t count = 0;
        if ((rc = clatch_prepare_keypoints(kps[i], n, cols, w, h, workers, xycs, kept[i], &count))) break;
        trace.stamp("batch: keypoints prepared");
        m[i] = count;
        if (count == 0) continue;
        BATCH_CUDA(cudaMemcpyAsync(slot.kps.ptr, xycs, sizeof(double) * 4 * count, cudaMemcpyHostToDevice, st));
        if (trace.on) cudaEventRecord(bev[3 * i], st);
        if (kU8) {
            rc = launch_extract_u8(ctx, slot.img.template as<uint8_t>(), w, h, dpitch, slot.kps.template as<double>(),
                                   count, slot.desc.template as<uint8_t>(), st);
        } else if (promoted) {
            rc = launch_extract_u8(ctx, slot.img_u8.template as<uint8_t>(), w, h, u8_pitch, slot.kps.template as<double>(),
                                   count, slot.desc.template as<uint8_t>(), st);
        } else {
            // the f64 launcher uses ctx-level promotion scratch: point it at this slot's buffers
            std::swap(ctx->img_u8, slot.img_u8);
            std::swap(ctx->flags, slot.flags);
            ctx->scratch_private = true;
            rc = launch_extract_f64(ctx, slot.img.template as<double>(), w, h, dpitch, slot.kps.template as<double>(),
                                    count, slot.desc.template as<uint8_t>(), st);
            ctx->scratch_private = false;
            std::swap(ctx->img_u8, slot.img_u8);
            std::swap(ctx->flags, slot.flags);
        }
        if (rc) break;
        // A page-locked out[i] (clatch_host_alloc — what the Python layer passes) takes the DMA directly;
        // pageable memory goes through page-locked staging so that the download stays asynchronous, and
        // is copied out when the slot comes round again.
        trace.stamp("batch: kernels queued");
        if (trace.on) cudaEventRecord(bev[3 * i + 1], st);
        cudaPointerAttributes attr{};
        const bool direct = cudaPointerGetAttributes(&attr, out[i]) == cudaSuccess && attr.type == cudaMemoryTypeHost;
        if (!direct) cudaGetLastError();   // an unregistered pointer is not an error here
        if (direct) {
            BATCH_CUDA(cudaMemcpyAsync(out[i], slot.desc.ptr, bytes * count, cudaMemcpyDeviceToHost, st));
        } else {
            BATCH_CUDA(cudaMemcpyAsync(slot.h_desc.ptr, slot.desc.ptr, bytes * count, cudaMemcpyDeviceToHost, st));
            slot.pending_out = out[i];
            slot.pending_bytes = bytes * count;
        }
        if (trace.on) cudaEventRecord(bev[3 * i + 2], st);
    }
    if (trace.on && !rc) {
        for (int s = 0; s < 2; ++s) cudaStreamSynchronize(ctx->pipe[s].stream);
        for (size_t i = 0; i < num_images; ++i) {
            float a = 0, b = 0, c = 0;
            if (cudaEventElapsedTime(&a, bev[3 * num_images], bev[3 * i]) == cudaSuccess &&
                cudaEventElapsedTime(&b, bev[3 * num_images], bev[3 * i + 1]) == cudaSuccess &&
                cudaEventElapsedTime(&c, bev[3 * num_images], bev[3 * i + 2]) == cudaSuccess)
                std::fprintf(stderr, "[clatch] device: image %zu uploaded at %.0f us, extracted at %.0f us, downloaded at %.0f us\n",
                             i, a * 1e3, b * 1e3, c * 1e3);
        }
        cudaGetLastError();
    }
    for (cudaEvent_t e : bev) cudaEventDestroy(e);
    for (int s = 0; s < 2; ++s) {
        clatch_ctx::PipeSlot& slot = ctx->pipe[s];
        cudaError_t e = cudaStreamSynchronize(slot.stream);
        if (e != cudaSuccess && !rc) rc = cuda_fail(e, "cudaStreamSynchronize(batch)");
        if (slot.pending_out && !rc) std::memcpy(slot.pending_out, slot.h_desc.ptr, slot.pending_bytes);
        slot.pending_out = nullptr;
    }
    return rc;
}

extern "C" {

int clatch_detect_u8(clatch_ctx* ctx, const uint8_t* img, int width, int height, size_t pitch, double threshold,
                     int nms, int orient, int radius, double* out, size_t cap, size_t* count) {
    return detect_impl<uint8_t>(ctx, img, width, height, pitch, threshold, nms, orient, radius, out, cap, count);
}

int clatch_detect_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch, double threshold,
                      int nms, int orient, int radius, double* out, size_t cap, size_t* count) {
    return detect_impl<double>(ctx, img, width, height, pitch, threshold, nms, orient, radius, out, cap, count);
}

int clatch_describe_batch_u8(clatch_ctx* ctx, const uint8_t* const* imgs, const int* widths, const int* heights,
                             const size_t* pitches, const double* const* kps, const size_t* counts, int cols,
                             size_t num_images, int workers, int64_t* const* kept, uint8_t* const* out, size_t* m) {
    return describe_batch_impl<uint8_t>(ctx, imgs, widths, heights, pitches, kps, counts, cols, num_images, workers,
                                        kept, out, m);
}

int clatch_describe_batch_f64(clatch_ctx* ctx, const double* const* imgs, const int* widths, const int* heights,
                              const size_t* pitches, const double* const* kps, const size_t* counts, int cols,
                              size_t num_images, int workers, int64_t* const* kept, uint8_t* const* out, size_t* m) {
    return describe_batch_impl<double>(ctx, imgs, widths, heights, pitches, kps, counts, cols, num_images, workers,
                                       kept, out, m);
}

int clatch_describe_all_u8(clatch_ctx* ctx, const uint8_t* img, int width, int height, size_t pitch,
                           const double* kps, size_t n, int cols, int workers, int64_t* kept,
                           uint8_t* out, size_t* m) {
    return describe_all_impl<uint8_t>(ctx, img, width, height, pitch, kps, n, cols, workers, kept, out, m);
}

int clatch_describe_all_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch,
                            const double* kps, size_t n, int cols, int workers, int64_t* kept,
                            uint8_t* out, size_t* m) {
    return describe_all_impl<double>(ctx, img, width, height, pitch, kps, n, cols, workers, kept, out, m);
}

// ---- matching -----------------------------------------------------------------

static int check_match(clatch_ctx* ctx, const void* q, size_t Q, const void* t, size_t N, int bytes) {
    if (!ctx) return invalid("match: ctx is null");
    if (bytes <= 0) return invalid("match: descriptor length must be positive");
    if (N == 0) {   // before the empty-probes early-out, src/match.cpp:55-56
        set_error("EmptyGallery: matching needs a nonempty gallery");
        return CLATCH_ERR_EMPTY_GALLERY;
    }
    if (N > 0x7fffffffull) return invalid("match: more than 2^31-1 train descriptors");
    if (!t || (Q > 0 && !q)) return invalid("match: null descriptor buffer");
    return CLATCH_OK;
}

int clatch_match_top2_dev(clatch_ctx* ctx, const uint8_t* d_queries, size_t Q,
                          const uint8_t* d_train, size_t N, int bytes, int32_t* d_best_idx,
                          int32_t* d_best_dist, int32_t* d_second_dist, void* stream) {
    if (int rc = check_match(ctx, d_queries, Q, d_train, N, bytes)) return rc;
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    return launch_match_top2(ctx, d_queries, Q, d_train, N, bytes, d_best_idx, d_best_dist,
                             d_second_dist, static_cast<cudaStream_t>(stream));
}

int clatch_match_top2(clatch_ctx* ctx, const uint8_t* queries, size_t Q, const uint8_t* train,
                      size_t N, int bytes, int32_t* best_idx, int32_t* best_dist,
                      int32_t* second_dist) {
    if (int rc = check_match(ctx, queries, Q, train, N, bytes)) return rc;
    if (Q == 0) return CLATCH_OK;
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    if (int rc = ctx->q.reserve(Q * bytes)) return rc;
    if (int rc = ctx->res.reserve(sizeof(int32_t) * 3 * Q)) return rc;
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpyAsync(ctx->q.ptr, queries, Q * bytes, cudaMemcpyHostToDevice, st));
    const uint8_t* d_train = ctx->q.as<uint8_t>();
    if (train != queries || N != Q) {   // self-match uploads the set once
        if (int rc = ctx->t.reserve(N * bytes)) return rc;
        CLATCH_CUDA(cudaMemcpyAsync(ctx->t.ptr, train, N * bytes, cudaMemcpyHostToDevice, st));
        d_train = ctx->t.as<uint8_t>();
    }
    int32_t* r = ctx->res.as<int32_t>();
    if (int rc = launch_match_top2(ctx, ctx->q.as<uint8_t>(), Q, d_train, N, bytes, r, r + Q, r + 2 * Q, st))
        return rc;
    if (best_idx) CLATCH_CUDA(cudaMemcpyAsync(best_idx, r, sizeof(int32_t) * Q, cudaMemcpyDeviceToHost, st));
    if (best_dist) CLATCH_CUDA(cudaMemcpyAsync(best_dist, r + Q, sizeof(int32_t) * Q, cudaMemcpyDeviceToHost, st));
    if (second_dist)
        CLATCH_CUDA(cudaMemcpyAsync(second_dist, r + 2 * Q, sizeof(int32_t) * Q, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    return CLATCH_OK;
}

} // extern "C"

struct clatch_set {
    clatch_ctx* ctx = nullptr;
    size_t n = 0;
    uint8_t* block = nullptr;   // one stream-ordered allocation: packed | int8 operand form
    uint8_t* packed = nullptr;
    uint8_t* exp = nullptr;
    size_t exp_cap = 0;         // bytes behind `exp` (sized for the larger operand form)
    int fmt = 0;                // operand form `exp` holds (tc_format at expansion time); re-expanded when it changes
};

namespace {

// Forward (+ reverse) top-2 of a batch of set pairs in one launch, results to `host`:
// per pair [best_idx n_i][best_dist n_i][second n_i][reverse_best n_j if cross_check].
int run_pair_batch(clatch_ctx* ctx, const clatch_set* const* sets, const int32_t* pairs, size_t first, size_t count,
                   bool cross_check, int32_t** host, std::vector<size_t>& pair_offset) {
    pair_offset.assign(count + 1, 0);
    size_t items = 0;
    for (size_t p = 0; p < count; ++p)     // the matcher's operand form changed since a set was expanded: redo it
        for (int side = 0; side < 2; ++side) {
            clatch_set* s = const_cast<clatch_set*>(sets[pairs[2 * (first + p) + side]]);
            if (s->fmt != tc_format(ctx) && s->n > 0) {
                if (int rc = launch_tc_expand(ctx, s->packed, s->n, s->exp, ctx->stream)) return rc;
                s->fmt = tc_format(ctx);
            }
        }
    for (size_t p = 0; p < count; ++p) {
        const clatch_set* a = sets[pairs[2 * (first + p)]];
        const clatch_set* b = sets[pairs[2 * (first + p) + 1]];
        pair_offset[p + 1] = pair_offset[p] + 3 * a->n + (cross_check ? b->n : 0);
        items += tc_query_tiles(a->n) + 1 + (cross_check ? tc_query_tiles(b->n) + 1 : 0);   // (+1: a filler per odd pass)
    }
    const size_t total = pair_offset[count];
    if (int rc = ctx->res.reserve(sizeof(int32_t) * std::max<size_t>(total, 1))) return rc;
    if (int rc = ctx->items.reserve(sizeof(TcItem) * std::max<size_t>(items, 1))) return rc;
    int32_t* r = ctx->res.as<int32_t>();
    std::vector<TcItem> table;
    table.reserve(items);
    for (size_t p = 0; p < count; ++p) {
        const clatch_set* a = sets[pairs[2 * (first + p)]];
        const clatch_set* b = sets[pairs[2 * (first + p) + 1]];
        int32_t* base = r + pair_offset[p];
        const bool paired = tc_items_paired(ctx);   // CTA pairs: entries (2k, 2k + 1) must scan the same train set
        const unsigned a_atoms = static_cast<unsigned>(tc_padded_rows(ctx, a->n) / 8);
        const unsigned b_atoms = static_cast<unsigned>(tc_padded_rows(ctx, b->n) / 8);
        for (int q = 0; q < tc_query_tiles(a->n); ++q)
            table.push_back({a->exp, b->exp, static_cast<unsigned>(a->n),
                             static_cast<unsigned>(b->n), static_cast<unsigned>(q), 0, a_atoms, b_atoms, base, base + a->n,
                             base + 2 * a->n});
        if (paired && (table.size() & 1)) {         // odd tile count: a filler keeps the last tile's partner in step
            table.push_back(table.back());
            table.back().ghost = 1;
        }
        if (cross_check) {   // reverse_best[g] = knn2(gallery[g], probes).best_index, src/match.cpp:62-67
            for (int q = 0; q < tc_query_tiles(b->n); ++q)
                table.push_back({b->exp, a->exp, static_cast<unsigned>(b->n),
                                 static_cast<unsigned>(a->n), static_cast<unsigned>(q), 0, b_atoms, a_atoms, base + 3 * a->n,
                                 nullptr, nullptr});
            if (paired && (table.size() & 1)) {
                table.push_back(table.back());
                table.back().ghost = 1;
            }
        }
    }
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpyAsync(ctx->items.ptr, table.data(), sizeof(TcItem) * table.size(), cudaMemcpyHostToDevice, st));
    if (int rc = launch_match_tc_items(ctx, ctx->items.as<TcItem>(), table.size(), st)) return rc;
    if (host == nullptr) {   // results stay on the device (filtered there)
        CLATCH_CUDA(cudaStreamSynchronize(st));   // keeps `table` alive until the H2D copy is done
        return CLATCH_OK;
    }
    if (int rc = ctx->pinned.reserve(sizeof(int32_t) * std::max<size_t>(total, 1))) return rc;
    *host = static_cast<int32_t*>(ctx->pinned.ptr);
    CLATCH_CUDA(cudaMemcpyAsync(*host, r, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));   // also keeps `table` alive until the H2D copy is done
    return CLATCH_OK;
}

int filter_table_on_device(clatch_ctx* ctx, const std::vector<FilterPair>& table, unsigned long long probes, int has_ratio,
                           double ratio, int has_max, int max_distance, const int32_t** rows,
                           std::vector<unsigned long long>& offsets);

// The filter pass of a batch on the device: kept rows of all pairs back to back in page-locked memory
// (*rows), row offsets per pair in offsets[0..count]. Only the surviving rows cross the bus.
int filter_pair_batch(clatch_ctx* ctx, const clatch_set* const* sets, const int32_t* pairs, size_t first, size_t count,
                      bool cross_check, const std::vector<size_t>& pair_offset, int has_ratio, double ratio,
                      int has_max, int max_distance, const int32_t** rows, std::vector<unsigned long long>& offsets) {
    std::vector<FilterPair> table(count);
    const int32_t* r = ctx->res.as<int32_t>();
    unsigned long long probes = 0;
    for (size_t p = 0; p < count; ++p) {
        const size_t n = sets[pairs[2 * (first + p)]]->n;
        const int32_t* base = r + pair_offset[p];
        table[p] = {base, base + n, base + 2 * n, cross_check ? base + 3 * n : nullptr, static_cast<unsigned>(n), 0, probes};
        probes += n;
    }
    return filter_table_on_device(ctx, table, probes, has_ratio, ratio, has_max, max_distance, rows, offsets);
}

// The filter pass (src/match.cpp:69-79) of `table.size()` result blocks that already sit on the device.
int filter_table_on_device(clatch_ctx* ctx, const std::vector<FilterPair>& table, unsigned long long probes, int has_ratio,
                           double ratio, int has_max, int max_distance, const int32_t** rows,
                           std::vector<unsigned long long>& offsets) {
    const size_t count = table.size();
    if (int rc = ctx->filt_pairs.reserve(sizeof(FilterPair) * count)) return rc;
    if (int rc = ctx->filt_rows.reserve(sizeof(int32_t) * 4 * std::max<unsigned long long>(probes, 1))) return rc;
    if (int rc = ctx->filt_out.reserve(sizeof(int32_t) * 4 * std::max<unsigned long long>(probes, 1))) return rc;
    if (int rc = ctx->filt_counts.reserve(sizeof(unsigned) * count + sizeof(unsigned long long) * (count + 2))) return rc;
    unsigned long long* d_offsets = ctx->filt_counts.as<unsigned long long>();
    unsigned* d_kept = reinterpret_cast<unsigned*>(d_offsets + count + 2);
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpyAsync(ctx->filt_pairs.ptr, table.data(), sizeof(FilterPair) * count, cudaMemcpyHostToDevice, st));
    if (int rc = launch_filter_pairs(ctx, ctx->filt_pairs.as<FilterPair>(), count, has_ratio, ratio, has_max, max_distance,
                                     ctx->filt_rows.as<int32_t>(), d_kept, d_offsets, ctx->filt_out.as<int32_t>(), st))
        return rc;
    offsets.resize(count + 1);
    CLATCH_CUDA(cudaMemcpyAsync(offsets.data(), d_offsets, sizeof(unsigned long long) * (count + 1), cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));   // (also keeps `table` alive until its upload is done)
    const unsigned long long total = offsets[count];
    if (int rc = ctx->pinned.reserve(sizeof(int32_t) * 4 * std::max<unsigned long long>(total, 1))) return rc;
    CLATCH_CUDA(cudaMemcpyAsync(ctx->pinned.ptr, ctx->filt_out.ptr, sizeof(int32_t) * 4 * total, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    *rows = static_cast<const int32_t*>(ctx->pinned.ptr);
    return CLATCH_OK;
}

} // namespace

extern "C" {

int clatch_triplet_bits(clatch_ctx* ctx, const double* windows, size_t n, const int16_t* candidates, size_t C, int K,
                        const double* mask, uint8_t* out, size_t row_bytes) {
    if (!ctx) return invalid("clatch_triplet_bits: ctx is null");
    if (K < 1 || K > kWindow) return invalid("clatch_triplet_bits: K out of range");
    if (n == 0 || C == 0) return CLATCH_OK;
    if (!windows || !candidates || !out) return invalid("clatch_triplet_bits: null buffer");
    if (row_bytes < (n + 7) / 8) return invalid("clatch_triplet_bits: row_bytes < ceil(n / 8)");
    if (n > 0x7fffffffu || C > 0x7fffffffu) return invalid("clatch_triplet_bits: too many patches or candidates");
    for (size_t c = 0; c < C; ++c)
        for (int i = 0; i < 6; ++i)
            if (candidates[6 * c + i] < 0 || candidates[6 * c + i] > kWindow - K) {
                set_error("CoordinateOutOfRange: candidate coordinate outside [0, " + std::to_string(kWindow - K) + "]");
                return CLATCH_ERR_COORD_RANGE;
            }
    std::vector<double> w(static_cast<size_t>(K) * K, 1.0);
    if (mask) w.assign(mask, mask + w.size());
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    const size_t words_per_patch = (C + 31) / 32, out_words = (n + 31) / 32;
    if (int rc = ctx->img.reserve(sizeof(double) * 4096 * n)) return rc;
    if (int rc = ctx->kps.reserve(sizeof(int16_t) * 6 * C)) return rc;
    if (int rc = ctx->partial.reserve(sizeof(unsigned) * words_per_patch * n)) return rc;
    if (int rc = ctx->res.reserve(sizeof(unsigned) * out_words * C)) return rc;
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpyAsync(ctx->img.ptr, windows, sizeof(double) * 4096 * n, cudaMemcpyHostToDevice, st));
    CLATCH_CUDA(cudaMemcpyAsync(ctx->kps.ptr, candidates, sizeof(int16_t) * 6 * C, cudaMemcpyHostToDevice, st));
    if (int rc = launch_triplet_bits(ctx, ctx->img.as<double>(), n, ctx->kps.as<short>(), C, K, w.data(),
                                     ctx->partial.as<unsigned>(), ctx->res.as<unsigned>(), st))
        return rc;
    std::vector<unsigned> host(out_words * C);
    CLATCH_CUDA(cudaMemcpyAsync(host.data(), ctx->res.ptr, sizeof(unsigned) * host.size(), cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));   // also covers the constant-memory upload of `w`
    const size_t live = (n + 7) / 8;
    for (size_t c = 0; c < C; ++c) {
        std::memcpy(out + c * row_bytes, host.data() + c * out_words, live);   // little-endian words == byte order
        if (row_bytes > live) std::memset(out + c * row_bytes + live, 0, row_bytes - live);
    }
    return CLATCH_OK;
}

int clatch_set_create(clatch_ctx* ctx, const uint8_t* descriptors, size_t n, int on_device, clatch_set** out) {
    if (!ctx || !out) return invalid("clatch_set_create: null argument");
    *out = nullptr;
    if (n > 0 && !descriptors) return invalid("clatch_set_create: null descriptors");
    if (n > 0x7fffffffull) return invalid("clatch_set_create: too many descriptors");
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    auto* set = new clatch_set;
    set->ctx = ctx;
    set->n = n;
    int rc = CLATCH_OK;
    if (n > 0) {
        cudaStream_t st = ctx->stream;
        const size_t packed_bytes = (n * 64 + 1023) / 1024 * 1024;
        const size_t exp_bytes = (n + 255) / 256 * 256 * 512 + 128 * 512;   // room for either operand form
        // cudaMallocAsync: pooled, stream-ordered — set churn does not pay cudaMalloc/cudaFree latency.
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&set->block), packed_bytes + exp_bytes, st);
        if (e != cudaSuccess) rc = cuda_fail(e, "cudaMallocAsync(set)");
        if (!rc) {
            set->packed = set->block;
            set->exp = set->block + packed_bytes;
            e = cudaMemcpyAsync(set->packed, descriptors, n * 64,
                                on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync(set)");
        }
        set->exp_cap = exp_bytes;
        set->fmt = tc_format(ctx);
        if (!rc) rc = launch_tc_expand(ctx, set->packed, n, set->exp, st);
        if (!rc && !on_device) {   // the caller may reuse its host buffer as soon as we return
            e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) rc = cuda_fail(e, "cudaStreamSynchronize(set)");
        }
    }
    if (rc) {
        clatch_set_destroy(set);
        return rc;
    }
    *out = set;
    return CLATCH_OK;
}

void clatch_set_destroy(clatch_set* set) {
    if (!set) return;
    cudaSetDevice(set->ctx->device);
    if (set->block) cudaFreeAsync(set->block, set->ctx->stream);
    delete set;
}

size_t clatch_set_count(const clatch_set* set) { return set ? set->n : 0; }

int clatch_match_set_pairs(clatch_ctx* ctx, const clatch_set* const* sets, size_t num_sets, const int32_t* pairs,
                           size_t num_pairs, int has_ratio, double ratio, int cross_check, int has_max,
                           int max_distance, int32_t* out, size_t cap_rows, size_t* offsets) {
    if (!ctx || !offsets) return invalid("clatch_match_set_pairs: null argument");
    offsets[0] = 0;
    if (num_pairs == 0) return CLATCH_OK;
    if (!sets || !pairs || !out) return invalid("clatch_match_set_pairs: null buffer");
    for (size_t p = 0; p < num_pairs; ++p) {
        const int32_t i = pairs[2 * p], j = pairs[2 * p + 1];
        if (i < 0 || j < 0 || static_cast<size_t>(i) >= num_sets || static_cast<size_t>(j) >= num_sets || !sets[i] ||
            !sets[j])
            return invalid("clatch_match_set_pairs: pair index out of range");
        if (sets[i]->ctx != ctx || sets[j]->ctx != ctx) return invalid("clatch_match_set_pairs: set from another context");
        if (sets[j]->n == 0) {   // src/match.cpp:55
            set_error("EmptyGallery: matching needs a nonempty gallery");
            return CLATCH_ERR_EMPTY_GALLERY;
        }
    }
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    // Chunks bounded by result bytes (<= 256 MiB of top-2 triples per launch).
    const size_t kChunkInts = (256u << 20) / sizeof(int32_t);
    int32_t* host = nullptr;   // pinned staging owned by the context
    std::vector<size_t> pair_offset;
    std::unique_ptr<int32_t[]> scratch;
    size_t scratch_cap = 0;
    size_t rows_out = 0;
    for (size_t first = 0; first < num_pairs;) {
        size_t count = 0, ints = 0;
        while (first + count < num_pairs) {
            const size_t need = 3 * sets[pairs[2 * (first + count)]]->n +
                                (cross_check ? sets[pairs[2 * (first + count) + 1]]->n : 0);
            if (count > 0 && ints + need > kChunkInts) break;
            ints += need;
            ++count;
        }
        if (ctx->pairs_filter_on_device) {
            // top-2 results stay on the device; the filter pass (src/match.cpp:69-79) runs there too
            if (int rc = run_pair_batch(ctx, sets, pairs, first, count, cross_check != 0, nullptr, pair_offset)) return rc;
            const int32_t* rows = nullptr;
            std::vector<unsigned long long> off;
            if (int rc = filter_pair_batch(ctx, sets, pairs, first, count, cross_check != 0, pair_offset, has_ratio, ratio,
                                           has_max, max_distance, &rows, off))
                return rc;
            if (rows_out + off[count] > cap_rows) return invalid("clatch_match_set_pairs: cap_rows too small");
            std::memcpy(out + 4 * rows_out, rows, sizeof(int32_t) * 4 * off[count]);
            for (size_t p = 0; p < count; ++p) offsets[first + p + 1] = rows_out + off[p + 1];
            rows_out += off[count];
            first += count;
            continue;
        }
        if (int rc = run_pair_batch(ctx, sets, pairs, first, count, cross_check != 0, &host, pair_offset)) return rc;
        // filter pass per pair (src/match.cpp:69-79): parallel into per-pair scratch, then compact in order
        std::vector<size_t> scratch_off(count + 1, 0), kept(count, 0);
        for (size_t p = 0; p < count; ++p) scratch_off[p + 1] = scratch_off[p] + 4 * sets[pairs[2 * (first + p)]]->n;
        if (scratch_off[count] > scratch_cap) {   // uninitialised on purpose: every kept row is written
            scratch_cap = scratch_off[count];
            scratch.reset(new int32_t[scratch_cap]);
        }
        const int parts = static_cast<int>(std::min<size_t>(count, resolve_workers(0)));
        WorkerPool::instance().run(parts, [&](int part) {
            for (size_t p = part; p < count; p += parts) {
                const size_t n = sets[pairs[2 * (first + p)]]->n;
                const int32_t* base = host + pair_offset[p];
                clatch_filter_matches(base, base + n, base + 2 * n, n, has_ratio, ratio, has_max, max_distance,
                                      cross_check ? base + 3 * n : nullptr, scratch.get() + scratch_off[p], &kept[p]);
            }
        });
        for (size_t p = 0; p < count; ++p) {
            if (rows_out + kept[p] > cap_rows) return invalid("clatch_match_set_pairs: cap_rows too small");
            std::memcpy(out + 4 * rows_out, scratch.get() + scratch_off[p], sizeof(int32_t) * 4 * kept[p]);
            rows_out += kept[p];
            offsets[first + p + 1] = rows_out;
        }
        first += count;
    }
    return CLATCH_OK;
}

int clatch_match_sets(clatch_ctx* ctx, const clatch_set* probes, const clatch_set* gallery, int has_ratio,
                      double ratio, int cross_check, int has_max, int max_distance, int32_t* out,
                      size_t* count) {
    if (!count) return invalid("clatch_match_sets: count is null");
    *count = 0;
    if (!ctx || !probes || !gallery) return invalid("clatch_match_sets: null argument");
    const clatch_set* sets[2] = {probes, gallery};
    const int32_t pair[2] = {0, 1};
    size_t offsets[2] = {0, 0};
    if (int rc = clatch_match_set_pairs(ctx, sets, 2, pair, 1, has_ratio, ratio, cross_check, has_max, max_distance,
                                        out, probes->n, offsets))
        return rc;
    *count = offsets[1];
    return CLATCH_OK;
}

int clatch_debug_tc_tile(clatch_ctx* ctx, const uint8_t* queries, size_t Q, const uint8_t* train, size_t N,
                         int32_t* tile_out, int32_t* best_idx, int32_t* best_dist, int32_t* second_dist) {
    if (int rc = check_match(ctx, queries, Q, train, N, 64)) return rc;
    if (Q == 0 || !tile_out) return invalid("clatch_debug_tc_tile: empty query set or null output");
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    if (int rc = ctx->q.reserve(Q * 64)) return rc;
    if (int rc = ctx->t.reserve(N * 64)) return rc;
    if (int rc = ctx->res.reserve(sizeof(int32_t) * (3 * Q + 128 * 256))) return rc;
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpyAsync(ctx->q.ptr, queries, Q * 64, cudaMemcpyHostToDevice, st));
    CLATCH_CUDA(cudaMemcpyAsync(ctx->t.ptr, train, N * 64, cudaMemcpyHostToDevice, st));
    int32_t* r = ctx->res.as<int32_t>();
    CLATCH_CUDA(cudaMemsetAsync(r + 3 * Q, 0, sizeof(int32_t) * 128 * 256, st));
    if (int rc = launch_match_top2_tc(ctx, ctx->q.as<uint8_t>(), Q, ctx->t.as<uint8_t>(), N, r, r + Q, r + 2 * Q, st,
                                      r + 3 * Q))
        return rc;
    CLATCH_CUDA(cudaMemcpyAsync(tile_out, r + 3 * Q, sizeof(int32_t) * 128 * 256, cudaMemcpyDeviceToHost, st));
    if (best_idx) CLATCH_CUDA(cudaMemcpyAsync(best_idx, r, sizeof(int32_t) * Q, cudaMemcpyDeviceToHost, st));
    if (best_dist) CLATCH_CUDA(cudaMemcpyAsync(best_dist, r + Q, sizeof(int32_t) * Q, cudaMemcpyDeviceToHost, st));
    if (second_dist)
        CLATCH_CUDA(cudaMemcpyAsync(second_dist, r + 2 * Q, sizeof(int32_t) * Q, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    return CLATCH_OK;
}

int clatch_filter_matches(const int32_t* best_idx, const int32_t* best_dist,
                          const int32_t* second_dist, size_t Q, int has_ratio, double ratio,
                          int has_max, int max_distance, const int32_t* reverse_best,
                          int32_t* out, size_t* count) {
    if (!count) return invalid("clatch_filter_matches: count is null");
    *count = 0;
    if (Q == 0) return CLATCH_OK;
    if (!best_idx || !best_dist || !second_dist || !out)
        return invalid("clatch_filter_matches: null buffer");
    size_t m = 0;
    for (size_t p = 0; p < Q; ++p) {   // src/match.cpp:69-79, same order of tests
        const int best = best_dist[p], second = second_dist[p], idx = best_idx[p];
        if (has_ratio && !(best < ratio * second)) continue;   // int -> double, as in the reference
        if (has_max && best > max_distance) continue;
        if (reverse_best && reverse_best[idx] != static_cast<int32_t>(p)) continue;
        out[4 * m + 0] = static_cast<int32_t>(p);
        out[4 * m + 1] = idx;
        out[4 * m + 2] = best;
        out[4 * m + 3] = second;
        ++m;
    }
    *count = m;
    return CLATCH_OK;
}

int clatch_match_brute_force(clatch_ctx* ctx, const uint8_t* probes, size_t Q,
                             const uint8_t* gallery, size_t N, int bytes, int has_ratio,
                             double ratio, int cross_check, int has_max, int max_distance,
                             int32_t* out, size_t* count) {
    if (!count) return invalid("clatch_match_brute_force: count is null");
    *count = 0;
    if (int rc = check_match(ctx, probes, Q, gallery, N, bytes)) return rc;
    if (Q == 0) return CLATCH_OK;   // src/match.cpp:56
    if (!out) return invalid("clatch_match_brute_force: out is null");
    CLATCH_CUDA(cudaSetDevice(ctx->device));
    const bool on_device = ctx->pairs_filter_on_device && bytes == 64 && ctx->match_variant >= 3;
    {
        // Cross-check between two sets of similar size (an image pair): both passes go out as ONE launch over two
        // temporary resident sets — forward and reverse query tiles in one item table — and the filter pass runs on
        // the device, so only the surviving rows come back (src/match.cpp:58-79).
        const size_t tq = (Q + 127) / 128, tn = (N + 127) / 128;
        if (on_device && cross_check && Q >= 1024 && N >= 1024 && std::max(tq, tn) <= 2 * std::min(tq, tn)) {
            clatch_set *a = nullptr, *b = nullptr;
            const bool self = gallery == probes && N == Q;
            int rc = clatch_set_create(ctx, probes, Q, 0, &a);
            if (!rc && !self) rc = clatch_set_create(ctx, gallery, N, 0, &b);
            if (!rc) {
                const clatch_set* sets[2] = {a, self ? a : b};
                const int32_t pair[2] = {0, 1};
                size_t offsets[2] = {0, 0};
                rc = clatch_match_set_pairs(ctx, sets, 2, pair, 1, has_ratio, ratio, 1, has_max, max_distance, out, Q, offsets);
                *count = rc ? 0 : offsets[1];
            }
            clatch_set_destroy(a);
            clatch_set_destroy(b);
            return rc;
        }
    }
    // Both sets go up once; forward and (optionally) reverse passes reuse them on the device.
    if (int rc = ctx->q.reserve(Q * bytes)) return rc;
    if (int rc = ctx->res.reserve(sizeof(int32_t) * (3 * Q + N))) return rc;
    cudaStream_t st = ctx->stream;
    CLATCH_CUDA(cudaMemcpyAsync(ctx->q.ptr, probes, Q * bytes, cudaMemcpyHostToDevice, st));
    const uint8_t* d_gallery = ctx->q.as<uint8_t>();
    if (gallery != probes || N != Q) {   // self-match uploads the set once
        if (int rc = ctx->t.reserve(N * bytes)) return rc;
        CLATCH_CUDA(cudaMemcpyAsync(ctx->t.ptr, gallery, N * bytes, cudaMemcpyHostToDevice, st));
        d_gallery = ctx->t.as<uint8_t>();
    }
    int32_t* r = ctx->res.as<int32_t>();
    if (int rc = launch_match_top2(ctx, ctx->q.as<uint8_t>(), Q, d_gallery, N, bytes, r, r + Q, r + 2 * Q, st))
        return rc;
    const size_t host_count = 3 * Q + (cross_check ? N : 0);
    if (int rc = ctx->pinned.reserve(sizeof(int32_t) * host_count)) return rc;   // page-locked: a plain DMA
    int32_t* const host = static_cast<int32_t*>(ctx->pinned.ptr);
    if (cross_check) {   // reverse_best[g] = knn2(gallery[g], probes).best_index, src/match.cpp:62-67
        if (int rc = launch_match_top2(ctx, d_gallery, N, ctx->q.as<uint8_t>(), Q, bytes, r + 3 * Q, nullptr,
                                       nullptr, st))
            return rc;
    }
    if (on_device && (has_ratio || has_max || cross_check) && Q >= 4096) {
        // some rows will be dropped: decide on the device and bring back the survivors only
        std::vector<FilterPair> table(1);
        table[0] = {r, r + Q, r + 2 * Q, cross_check ? r + 3 * Q : nullptr, static_cast<unsigned>(Q), 0, 0ull};
        const int32_t* rows = nullptr;
        std::vector<unsigned long long> off;
        if (int rc = filter_table_on_device(ctx, table, Q, has_ratio, ratio, has_max, max_distance, &rows, off)) return rc;
        std::memcpy(out, rows, sizeof(int32_t) * 4 * off[1]);
        *count = off[1];
        return CLATCH_OK;
    }
    CLATCH_CUDA(cudaMemcpyAsync(host, r, sizeof(int32_t) * host_count, cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    return clatch_filter_matches(host, host + Q, host + 2 * Q, Q, has_ratio, ratio, has_max, max_distance,
                                 cross_check ? host + 3 * Q : nullptr, out, count);
}

} // extern "C"
