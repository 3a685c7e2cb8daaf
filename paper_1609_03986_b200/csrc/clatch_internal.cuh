// Internal declarations shared by the C-ABI translation units. Not installed.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "clatch.h"

namespace clatch {

constexpr int kWindow = 64;        // oriented window side (proj/include/latch/pattern.hpp:12)
constexpr int kMargin = 46;        // proj/include/latch/descriptor.hpp:17
constexpr int kWinStride = 65;     // padded row stride of the fp64 window in shared memory
constexpr int kTileW = 112;        // staged u8 footprint: 92 px + 16-byte alignment slack
constexpr int kTileH = 92;         // rows floor(y)-45 .. floor(y)+46
constexpr int kFastT = 512;        // specialised kernel: T = 512, K = 8, 7x7-of-8x8 mask
constexpr int kMaxConstWeights = 64 * 64;

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define CLATCH_CUDA(expr)                                            \
    do {                                                             \
        cudaError_t _e = (expr);                                     \
        if (_e != cudaSuccess) return ::clatch::cuda_fail(_e, #expr); \
    } while (0)

// Grow-only device scratch buffer.
struct DeviceBuffer {
    void* ptr = nullptr;
    size_t cap = 0;
    int reserve(size_t bytes);
    void release();
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
};

// Grow-only page-locked host staging buffer.
struct PinnedBuffer {
    void* ptr = nullptr;
    size_t cap = 0;
    int reserve(size_t bytes);
    void release();
};

struct Pattern {
    int T = 0;
    int K = 0;
    bool fast = false;             // T=512, K=8, 7x7-of-8x8 binary mask
    // Slot tables (device): slot j of the specialised kernel computes bit `bit[j]`
    // from window offsets (row*kWinStride+col) a/b/c; packed as ushort4 {a, b, c, bit}.
    DeviceBuffer slots;            // T * ushort4 (single-window kernel: half-warps of 16 triplets)
    DeviceBuffer slots_quad;       // T * ushort4 (quad kernel: half-warps of 4 triplets x 4 keypoints)
    DeviceBuffer slots_f8;         // T * ushort4 (filtered kernel: warps of 8 triplets x 4 keypoints)
    DeviceBuffer slots_h16;        // T * ushort4 (packed-plane kernel: the same lanes, word offsets into the 16-bit copies)
    std::vector<int16_t> host_triplets;   // T * 6, for plans made on first use
    bool slots_planned = false;    // `slots` holds a plan for the current table
    bool slots_f8_planned = false; // `slots_f8` does (the built-in table's ships precomputed; others are planned on first use)
    DeviceBuffer triplets;         // generic kernel: T * 6 int16
    DeviceBuffer d_weights;        // generic kernel: K*K mask weights (per context, not a module-level __constant__)
    std::vector<double> weights;   // K*K
    double slot_degree = 0.0;           // planned / table-order shared-load conflict degree
    double slot_degree_identity = 0.0;
    double slot_degree_quad = 0.0;
    double slot_degree_f8 = 0.0;
    double slot_degree_h16 = 0.0;
};

} // namespace clatch

struct clatch_ctx {
    int device = 0;
    int sm_count = 0;
    int sm_clock_khz = 0;
    char name[256] = {0};
    cudaStream_t stream = nullptr;
    clatch::Pattern pattern;
    uint64_t launches = 0;
    bool tc_configured = false, quad_configured = false, filt_configured = false, pipe_configured = false;   // opt-in smem sizes set on this device
    // 0: one window per CTA (4 CTAs/SM); 1: quad kernel (4 fp64 windows per CTA); 2: filtered kernel
    // (4 split windows per CTA, fp32 estimate + exact recompute); 3: pipelined kernel (resampling
    // overlapped with the estimate, footprints from the texture unit); 4: variant 3 with dedicated
    // producer / consumer warps; 5: packed 16-bit planes resampled in fp32 (dedicated roles, the default); 6: variant 5
    // with every warp doing both halves. 2-6 take u8 images — others run variant 1.
    int extract_variant = 5;
    struct TexImage {                // pipelined kernel: the image as a gather-enabled CUDA array
        cudaStream_t stream = nullptr;
        cudaArray_t array = nullptr;
        cudaTextureObject_t tex = 0;
        cudaTextureObject_t texn = 0;    // the same array, texels read as value / 255 (packed-plane kernel)
        cudaArray_t arrayf = nullptr;    // float64 images that are not u8-valued: the image scaled to [0, 1] as floats
        cudaTextureObject_t texf = 0;
        cudaSurfaceObject_t surff = 0;
        int widthf = 0, heightf = 0;
        cudaSurfaceObject_t surf = 0;    // the same array, for the fill kernel
        int width = 0, height = 0;
        unsigned* tickets = nullptr;     // {next quad ticket, CTAs finished}: the packed-plane kernel hands out its quads dynamically
    };
    std::vector<TexImage> tex_images;
    // extraction routing for degenerate images (launch_extract): host-mapped per-CTA slots written by the default kernel
    bool extract_route = true;       // set_option "extract_route"
    bool extract_f64_h16 = true;     // set_option "extract_f64_h16": tame float64 images that are not u8-valued take the packed-plane kernel
    uint2* route_host = nullptr;     // page-locked, mapped
    uint2* route_dev = nullptr;      // the device's view of route_host
    bool route_pending = false, route_quad = false;
    unsigned route_age = 0;
    unsigned route_period = 16, route_probe_at = 0;   // while routed: the default kernel probes again at launch route_probe_at
    const unsigned* extract_out_index = nullptr;   // set around a launch: record j -> output row (banded upload)
    bool extract_stats_on = false;           // count exact recomputes (clatch_extract_stats)
    clatch::DeviceBuffer extract_stats;      // 2 x u64
    bool pairs_filter_on_device = true;   // clatch_match_set_pairs: ratio / max / cross-check decisions on the device
    // tensor matcher: clusters of two CTAs share the train-set stream through TMA multicast (one L2 read feeds two
    // SMs) wherever two query tiles scan the same train tiles; set_option "match_pairs" 0 = every CTA on its own.
    bool pdl = true;               // programmatic dependent launch inside the library's own kernel chains (set_option "pdl")
    bool match_pairs = true;
    bool match_2cta = false;       // paired launches of the e2m1 form run one M = 256 MMA stream per pair (tcgen05 cta_group::2; set_option
                                   // "match_2cta"). Correct, and the bare instruction runs at full rate (tools/tc_pair_probe.cu), but next to
                                   // the TMA stream a tile takes 2 240 clk instead of 1 400: off
    bool match_form_auto = false;  // match_variant 4: 1 = mid-sized single matches run the int8 form (it was ahead there before the parked-chunk epilogue; kept for A/B)
    bool match_streamk = true;     // tensor matcher: equal-share partition for small problems (set_option "match_streamk")
    bool match_streamk_pairs = false;  // ... over (query tile pair, train tile) units on CTA pairs (set_option "match_streamk_pairs";
                                       // measured equal at 10 k x 10 k — 31.2 vs 31.1 us under ncu, 44.0 vs 42.9 us in bench — so off)
    int match_variant = 4;         // 0: 16 POPC, 1: 7 CSA + 9 POPC, 2: 9 CSA + 7 POPC, 3: tcgen05 int8 GEMM, 4: tcgen05 mxf4 (e2m1) GEMM (CLATCH_MATCH_VARIANT)
    // The scratch below is shared by every call on this context, whatever stream the call queues on
    // (the *_dev entry points take the caller's stream). scratch_event marks the last use; a call on a
    // different stream waits for it first (clatch::scratch_acquire / scratch_release), so two device-form
    // calls on different streams — or a device-form call followed by a host-form one — are ordered.
    cudaEvent_t scratch_event = nullptr;
    cudaStream_t scratch_stream = nullptr;
    bool scratch_used = false;
    bool scratch_private = false;   // describe_batch has swapped in a pipeline slot's own buffers: no guard
    // scratch for the host-buffer entry points
    clatch::DeviceBuffer img, kps, desc, q, t, res, partial, flags, img_u8, exp_q, exp_t, items, scores, counts, det;
    clatch::DeviceBuffer filt_pairs, filt_rows, filt_out, filt_counts;   // on-device filter pass of batched set pairs
    std::vector<double> host_xycs;   // describe_all staging
    std::vector<int64_t> band_src;   // banded float64 upload: record j <- input keypoint
    std::vector<uint8_t> band_of;
    int upload_bands = 0;            // describe_all, float64 images: 0 = auto (set_option "upload_bands")
    clatch::PinnedBuffer pinned;     // D2H staging for batched pair results
    clatch::PinnedBuffer pin_xycs, pin_desc;   // describe_all staging (banded upload path)
    clatch::PinnedBuffer pin_img;              // describe_all: host-promoted u8 copy of a float64 image
    // float64 -> u8 on the host workers before the upload: 0 = when the image lies in ordinary (pageable)
    // memory (the driver would stage such a copy through its own bounce buffers at ~12 GB/s; reading it
    // once with the workers and sending 1 byte per pixel is faster), 1 = always, 2 = never. For page-locked
    // sources the plain DMA of the doubles won (profiles/r1y_e2e_breakdown.log).
    int host_promote = 0;
    int pageable_f64_frames = 0;   // big float64 frames in ordinary memory seen without page-locked staging (describe_all)
    cudaStream_t copy_stream = nullptr;        // image bands stream in here while kernels run on `stream`
    cudaEvent_t band_events[8] = {};
    struct PipeSlot {                // describe_batch: one of two pipeline slots
        cudaStream_t stream = nullptr;
        clatch::DeviceBuffer img, kps, desc, img_u8, flags;
        clatch::PinnedBuffer h_xycs, h_desc, h_img;   // page-locked staging (h_img: host-promoted u8 copy of a float64 image)
        uint8_t* pending_out = nullptr;         // caller array awaiting h_desc
        size_t pending_bytes = 0;
    } pipe[2];
};

namespace clatch {

// Programmatic dependent launch (PDL): a kernel launched with launch_kernel(..., pdl = true) may start while its
// predecessor in the stream is still running — its CTAs get scheduled and run their set-up — and must execute
// pdl_wait() before it touches anything the predecessor writes (or writes anything the predecessor reads); the
// predecessor calls pdl_launch_dependents() as early as it likes (here: at its start). Without the attribute both
// instructions are no-ops. Only kernels whose predecessor was launched the ordinary way (fully ordered behind
// ITS predecessors) or is itself a PDL kernel that waits at its start are launched like this, so that
// pdl_wait() transitively covers everything earlier in the stream.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, bool pdl,
                                 unsigned cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attrs[2]{};
    unsigned n = 0;
    if (cluster_x > 1) {
        attrs[n].id = cudaLaunchAttributeClusterDimension;
        attrs[n].val.clusterDim.x = cluster_x;
        attrs[n].val.clusterDim.y = 1;
        attrs[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl) {
        attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#endif

inline int scratch_acquire(clatch_ctx* ctx, cudaStream_t st) {
    if (ctx->scratch_private) return CLATCH_OK;
    if (ctx->scratch_used && ctx->scratch_stream != st) CLATCH_CUDA(cudaStreamWaitEvent(st, ctx->scratch_event, 0));
    return CLATCH_OK;
}
inline int scratch_release(clatch_ctx* ctx, cudaStream_t st) {
    if (ctx->scratch_private) return CLATCH_OK;
    if (!ctx->scratch_event) CLATCH_CUDA(cudaEventCreateWithFlags(&ctx->scratch_event, cudaEventDisableTiming));
    CLATCH_CUDA(cudaEventRecord(ctx->scratch_event, st));
    ctx->scratch_stream = st;
    ctx->scratch_used = true;
    return CLATCH_OK;
}

// extraction (clatch_extract.cu)
bool extract_supports_out_index(const clatch_ctx* ctx);
int launch_extract_u8(clatch_ctx* ctx, const uint8_t* d_img, int width, int height, size_t pitch,
                      const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream);
int launch_estimate_planes_u8(clatch_ctx* ctx, const uint8_t* d_img, int width, int height, size_t pitch,
                              const double* d_xycs, size_t M, uint16_t* d_out, cudaStream_t stream);
int launch_extract_f64(clatch_ctx* ctx, const double* d_img, int width, int height, size_t pitch,
                       const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream);
int launch_classify_rows(clatch_ctx* ctx, const double* d_img, int width, int height, size_t pitch, int row0,
                         int row1, bool reset, cudaStream_t stream);
int launch_extract_f64_classified(clatch_ctx* ctx, const double* d_img, int width, int height, size_t pitch,
                                  const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream, bool whole_image = false);

// detection (clatch_detect.cu)
struct Detection {   // one FAST detection as the device leaves it (row-major order)
    int x, y;
    double score, m10, m01;
    int valid, pad;  // valid = 0: orientation disc leaves the image
};
int launch_detect_u8(clatch_ctx* ctx, const uint8_t* d_img, int w, int h, size_t pitch, double threshold, int nms,
                     int orient, int radius, cudaStream_t st, unsigned* count);
int launch_detect_f64(clatch_ctx* ctx, const double* d_img, int w, int h, size_t pitch, double threshold, int nms,
                      int orient, int radius, cudaStream_t st, unsigned* count);

// trainer scoring (clatch_score.cu)
int launch_triplet_bits(clatch_ctx* ctx, const double* d_windows, size_t n, const short* d_candidates, size_t C, int K,
                        const double* weights, unsigned* d_by_patch, unsigned* d_out, cudaStream_t st);

// matching (clatch_match.cu, clatch_match_tc.cu)
struct Partial {   // per (train split, query) partial top-2
    int best_idx;
    int best_dist;
    int second_dist;
    int pad;
};
struct TcItem {    // one CTA of the tensor-core matcher in batched mode: 128 queries x a whole train set
    const uint8_t* a_exp;    // query set, expanded
    const uint8_t* b_exp;    // train set, expanded (same layout)
    unsigned Q, N;           // real row counts
    unsigned qtile;          // which 128-row query tile
    unsigned ghost;          // CTA-pair tables: 1 = filler that only keeps its partner's operand stream company
    unsigned a_atoms, b_atoms;   // 8-row atoms per K-block of the two expanded sets (tc_padded_rows / 8)
    int32_t* best_idx;       // outputs for the whole query set (any may be null)
    int32_t* best_dist;
    int32_t* second_dist;
};
struct FilterPair {   // one set pair of the on-device filter pass
    const int32_t* best_idx;       // forward top-2 of the pair's probes
    const int32_t* best_dist;
    const int32_t* second_dist;
    const int32_t* reverse_best;   // reverse pass (cross-check) or null
    unsigned n;                    // probes
    unsigned pad;
    unsigned long long out_base;   // first row of this pair's worst-case slice
};
int launch_filter_pairs(clatch_ctx* ctx, const FilterPair* d_pairs, size_t count, int has_ratio, double ratio, int has_max,
                        int max_distance, int32_t* d_rows, unsigned* d_kept, unsigned long long* d_offsets,
                        int32_t* d_out, cudaStream_t stream);
size_t tc_padded_rows(const clatch_ctx* ctx, size_t rows);    // rows of an expanded set in the context's operand form
size_t tc_expanded_bytes(const clatch_ctx* ctx, size_t rows);
int tc_format(const clatch_ctx* ctx);                          // 8 = int8 operands, 4 = e2m1 operands (match_variant 4)
int tc_query_tiles(size_t rows);
bool tc_items_paired(const clatch_ctx* ctx);   // item tables must hold entries (2k, 2k + 1) over one train set; TcItem::ghost = 1 marks a filler
int launch_tc_expand(clatch_ctx* ctx, const uint8_t* d_packed, size_t n, uint8_t* d_out, cudaStream_t stream);
int launch_match_tc_items(clatch_ctx* ctx, const TcItem* d_items, size_t count, cudaStream_t stream);
void launch_merge_partials(const Partial* partial, unsigned long long Q, int splits, int sentinel,
                           int32_t* best_idx, int32_t* best_dist, int32_t* second_dist, cudaStream_t stream, bool pdl = false);
int launch_match_top2_tc(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                         int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second, cudaStream_t stream,
                         int32_t* d_dump = nullptr);
int launch_match_top2(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                      int bytes, int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second,
                      cudaStream_t stream);

} // namespace clatch
