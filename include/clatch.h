/* clatch.h — C ABI of the B200-native CLATCH hot paths (sm_100a).
 *
 * Drop-in boundary for the two data-parallel paths of the reference
 * ("latchkit", arXiv 1609.03986): LATCH descriptor extraction and brute-force
 * Hamming top-2 matching. Plain C: pointers, sizes, int status codes — no C++
 * types, no torch types, no exceptions. The reference's C++ functions
 * (namespace latch) and Python bindings call these through the shims shown in
 * INTEGRATION.md; paths below are relative to /root/reference/proj.
 *
 * Division of labour:
 *   host shim   margin filter, glibc cos/sin (bit parity needs the host libm),
 *               ratio / max-distance / cross-check filter pass, error re-raise
 *   this ABI    everything per-sample and per-pair: window resampling, triplet
 *               SSD compares, bit packing, XOR+popcount, top-2 selection
 *
 * There is NO CPU fallback: every compute entry point fails with
 * CLATCH_ERR_NO_DEVICE / CLATCH_ERR_CUDA when the GPU path cannot run.
 *
 * Threading: a clatch_ctx owns one CUDA device, one stream and its scratch
 * buffers; calls on one ctx must be serialised by the caller, distinct ctxs are
 * independent (one process or thread per GPU).
 */
#ifndef CLATCH_H
#define CLATCH_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CLATCH_API __attribute__((visibility("default")))
#else
#define CLATCH_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct clatch_ctx clatch_ctx;

/* Status codes. Codes >= 100 are 100 + latch::ErrorCode (include/latch/errors.hpp:10-40)
 * so a shim can re-raise latch::Error(static_cast<ErrorCode>(rc - 100), clatch_last_error()). */
enum {
    CLATCH_OK = 0,
    CLATCH_ERR_IMAGE_TOO_SMALL = 106,     /* ErrorCode::ImageTooSmall     (src/detect.cpp:77-78) */
    CLATCH_ERR_INVALID = 1,      /* null pointer, bad size, bad pitch ... */
    CLATCH_ERR_CUDA = 2,         /* a CUDA runtime call failed; see clatch_last_error() */
    CLATCH_ERR_NO_DEVICE = 3,    /* no CUDA device / not an sm_100 part */
    CLATCH_ERR_NONFINITE = 5,    /* non-finite keypoint coordinate or angle reached the device path
                                    (the reference would std::terminate in a worker thread,
                                    src/parallel.hpp:33-35 + src/image.cpp:110-112) */
    CLATCH_ERR_TOO_CLOSE_TO_BORDER = 107, /* ErrorCode::TooCloseToBorder  (src/descriptor.cpp:30-33) */
    CLATCH_ERR_BAD_HEADER = 108,          /* ErrorCode::BadHeader         (src/pattern.cpp:73-82) */
    CLATCH_ERR_BAD_TRIPLET_COUNT = 109,   /* ErrorCode::BadTripletCount */
    CLATCH_ERR_COORD_RANGE = 110,         /* ErrorCode::CoordinateOutOfRange (src/pattern.cpp:54-61) */
    CLATCH_ERR_DEGENERATE = 111,          /* ErrorCode::DegenerateTriplet (src/pattern.cpp:62-65) */
    CLATCH_ERR_LENGTH_MISMATCH = 119,     /* ErrorCode::LengthMismatch    (src/match.cpp:15-18) */
    CLATCH_ERR_EMPTY_GALLERY = 120        /* ErrorCode::EmptyGallery      (src/match.cpp:34,55) */
};

/* Message for the last failing call on this thread (never NULL). */
CLATCH_API const char* clatch_last_error(void);

/* ---- context ---------------------------------------------------------------- */

/* Binds a context to CUDA device `device` (one per GPU; replaces the reference's
 * std::thread fan-out, src/parallel.hpp:17-38). No pattern is installed yet: call
 * clatch_set_pattern before extracting. */
CLATCH_API int clatch_ctx_create(int device, clatch_ctx** out);
CLATCH_API void clatch_ctx_destroy(clatch_ctx* ctx);

/* Device facts for reporting: SM count, SM clock (kHz), name (<= 255 chars). */
CLATCH_API int clatch_device_info(clatch_ctx* ctx, int* sm_count, int* sm_clock_khz, char* name, size_t cap);

/* Tuning knobs (never change results). key "match_variant": 0 = XOR + 16 POPC, 1 = carry-save
 * compression + 9 POPC, 2 = 9 CSA + 7 POPC, 3 = tcgen05 int8 GEMM on the tensor cores, 4 = tcgen05 block-scaled
 * FP4 GEMM (e2m1 +-1.0 operands, every scale 2^0, f32 accumulators: exact, twice the MACs per clock; default).
 * key "extract_variant": 0 = one window per CTA, 1 = four fp64 windows per CTA with conflict-free
 * shared loads, 2 = four split (fp32 + low word) windows per CTA: a proven fp32 estimate decides
 * each bit and the rare undecided ones are recomputed exactly, 3 = the same estimate with
 * double-buffered planes, texture-unit footprints and resampling overlapped with the estimate,
 * 4 = variant 3 with dedicated producer / consumer warps, 5 = the estimate from packed 16-bit planes (two shifted
 * copies: a 7-pixel patch row is four aligned 32-bit words) resampled in fp32 with fixed-point coordinates, dedicated
 * producer / consumer warps, its groups of four keypoints drawn from a per-stream device counter that rewinds itself
 * (default; the launches of one stream must not overlap, which stream order guarantees), 6 = variant 5 with every warp
 * doing both halves and a static round-robin. 2-6 take u8-valued images;
 * any other image runs variant 1. Every variant returns the same bytes (an estimate only ever decides a bit under a
 * proven error bound; undecided bits are recomputed with the reference's exact arithmetic). The environment variable
 * CLATCH_EXTRACT_VARIANT sets the initial value of a new context.
 * key "pdl": 1 (default) launches the dependent kernels of the library's own chains (array fill -> extraction; operand
 * expansion -> tensor-core matcher -> merge) with programmatic stream serialization: their CTAs are scheduled and run
 * their set-up while the predecessor finishes, and wait (griddepcontrol.wait) before touching its output; 0 = plain launches.
 * key "extract_route": 1 (default) lets a context whose last u8 launch needed the window-wide exact pass for more than 25 %
 * of its windows (18 % with extract_variant 6, 35 % with extract_variant 4; flat / saturated images: exact ties) run the next launches on the all-fp64 quad kernel, probing the default
 * kernel again after 16 launches (then 32, 64, 128 while the probes keep finding the stream degenerate); 0 = always the selected variant.
 * key "extract_f64_h16": 1 (default) sends a float64 image that is not u8-valued but tame (finite, a value range between
 * 2^-400 and 2^400, no pixel further than 2^20 ranges from zero) through the packed-plane kernel, its estimate planes resampled from a
 * float texture of the image scaled to [0, 1] and every undecided bit recomputed from the doubles; 0 = the all-fp64
 * kernel (variant 1), which also takes whatever is not tame and frames that arrive in row bands.
 * key "upload_bands": clatch_describe_all_f64 uploads a big float64 frame in this many row bands and
 * extracts each band's keypoints while the next band is in flight (0 = choose by frame size, the
 * default; 1 = one piece; up to 6). Results never depend on it.
 * key "host_promote": clatch_describe_all_f64 / clatch_describe_batch_f64 can convert a float64 image
 * whose pixels are all integers in [0, 255] to u8 on the host workers before the upload (8x fewer
 * bytes over the bus; lossless, same descriptors). 0 (default) does so when the image lies in ordinary
 * pageable memory — which the driver could only copy through its own bounce buffers — and uploads the
 * doubles of a page-locked image as they are (classified on the device); 1 = always, 2 = never.
 * key "match_form_auto": 1 lets match_variant 4 run mid-sized single matches (3e7 .. 6e8 compares) in the int8
 * form (an A/B switch from before the e2m1 form's parked-chunk epilogue); 0 (default) = always e2m1.
 * key "match_pairs": 1 (default) runs the tensor-core matcher as clusters of two CTAs that share one stream of
 * train tiles through TMA multicast (half the L2 traffic per compare); 0 = every CTA streams for itself.
 * key "match_2cta": 1 runs paired launches of the e2m1 form as ONE M = 256 MMA stream per CTA pair (tcgen05 cta_group::2,
 * each CTA holding half of every train tile); 0 (default) = two M = 128 streams over multicast train tiles (measured faster).
 * key "match_streamk": 1 (default) lets the tensor-core matcher split small problems (expanded train set
 * within 32 MB) into equal shares of (query tile, train tile) units per CTA; 0 keeps whole rounds.
 * key "match_streamk_pairs": 1 cuts those shares over (query tile pair, train tile) units and runs them on CTA pairs
 * that share the train stream by multicast (needs match_pairs); 0 (default) = one CTA per share (measured equal).
 * key "pairs_filter_on_device": 1 (default) runs the ratio / max-distance / cross-check decisions of
 * clatch_match_set_pairs on the device so only surviving rows cross the bus; 0 filters on the host.
 * key "extract_stats": non-zero starts counting variant 2's exact recomputes (and zeroes the
 * counters), 0 stops. Unknown keys fail with CLATCH_ERR_INVALID. */
CLATCH_API int clatch_set_option(clatch_ctx* ctx, const char* key, int value);

/* Counters of the filtered extraction kernel since "extract_stats" was switched on: triplets
 * whose bit was recomputed in exact fp64, and warp passes that entered the exact path. Waits for
 * the context's streams. Diagnostics only. */
CLATCH_API int clatch_extract_stats(clatch_ctx* ctx, uint64_t* exact_triplets, uint64_t* exact_warps);

/* Block until everything queued on the context's own stream has finished. */
CLATCH_API int clatch_synchronize(clatch_ctx* ctx);

/* ---- pattern (replaces TripletPattern / WeightMask, include/latch/pattern.hpp:19-52) ----
 * triplets: T rows {ax, ay, bx, by, cx, cy}, top-left patch corners in window
 * coordinates; mask: K*K row-major non-negative finite weights, or NULL for all
 * ones. Validation mirrors parse_pattern (src/pattern.cpp:54-66,78-82,118-131):
 * T > 0 and T % 8 == 0, 1 <= K <= 64, coords in [0, 64-K], companions distinct,
 * weights finite, >= 0 and not all zero. T=512, K=8 with the 7x7-emulating 0/1
 * mask selects the specialised kernel; anything else runs the generic kernel. */
CLATCH_API int clatch_set_pattern(clatch_ctx* ctx, const int16_t* triplets, int T, int K, const double* mask);

/* Bytes per descriptor (T/8) of the installed pattern, 0 if none. */
CLATCH_API int clatch_descriptor_bytes(clatch_ctx* ctx);

/* ---- host-side keypoint preparation (no GPU work) ----------------------------
 * Replaces the serial margin pre-pass of describe_all (src/descriptor.cpp:94-97,
 * keypoint_in_margin :23-27) and hoists the per-keypoint trig of extract_window
 * (:35-36) onto the host's glibc so results stay bit-identical to the reference.
 * kps: n rows of `cols` (2..4) doubles {x, y[, theta[, score]]}; missing theta = 0
 * (bindings/module.cpp:49-62). Writes, for the m keypoints inside the 46 px
 * margin of a width x height image, in input order: xycs[4*j] = {x, y, cos(theta),
 * sin(theta)} and kept[j] = input index. `workers` <= 0 uses all cores. Fails with
 * CLATCH_ERR_NONFINITE if a kept keypoint has a non-finite theta. */
CLATCH_API int clatch_prepare_keypoints(const double* kps, size_t n, int cols, int width, int height,
                             int workers, double* xycs, int64_t* kept, size_t* m);

/* The kept keypoints of describe_all as (m, 4) rows [x, y, theta, score] (missing columns read as 0):
 * out[j] = kps[kept[j]], gathered on the host workers. What the reference returns as the first half
 * of its (Keypoint, Descriptor) pairs (src/descriptor.cpp:99-104). */
CLATCH_API int clatch_take_keypoints(const double* kps, int cols, const int64_t* kept, size_t m, int workers,
                                     double* out);

/* ---- detection (the step before the path: fast_detect / detect_and_orient,
 * src/detect.cpp:76-157) -------------------------------------------------------------------
 * FAST-9 segment test with `threshold`, optional 3x3 non-maximum suppression (ties keep the
 * smallest (y, x)), and — when `orient` — the intensity-centroid angle over a disc of `radius`
 * (15 in the reference); detections whose disc leaves the image are dropped. The moments are
 * accumulated on the device in the reference's order; atan2 runs on the host libm. Output
 * rows {x, y, theta, score} in (y, x) order, bit-identical to the reference. If more than
 * `cap` rows are found, *count still reports the number and the call fails with
 * CLATCH_ERR_INVALID (call again with a larger buffer). Images smaller than 7x7 fail with
 * CLATCH_ERR_IMAGE_TOO_SMALL. */
CLATCH_API int clatch_detect_u8(clatch_ctx* ctx, const uint8_t* img, int width, int height, size_t pitch,
                     double threshold, int nms, int orient, int radius, double* out, size_t cap,
                     size_t* count);
CLATCH_API int clatch_detect_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch,
                      double threshold, int nms, int orient, int radius, double* out, size_t cap,
                      size_t* count);

/* ---- extraction (replaces describe / describe_all, src/descriptor.cpp:79-105; the
 * arithmetic of extract_window :29-49, sample_bilinear src/image.cpp:109-126 and
 * triplet_bit src/descriptor.cpp:51-77 runs on the device, fp64, unfused) --------
 * Host-buffer forms copy in, run, copy out and return when `out` is ready.
 * img: row-major, `pitch` in ELEMENTS between rows (>= width). xycs: M rows from
 * clatch_prepare_keypoints (all inside the margin — not re-checked on device).
 * out: M * T/8 bytes, bit t of a descriptor at byte t>>3, bit t&7 (LSB first). */
CLATCH_API int clatch_extract_u8(clatch_ctx* ctx, const uint8_t* img, int width, int height, size_t pitch,
                      const double* xycs, size_t M, uint8_t* out);
CLATCH_API int clatch_extract_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch,
                       const double* xycs, size_t M, uint8_t* out);

/* describe_all in one call (src/descriptor.cpp:90-105): margin filter + host trig +
 * upload + extraction + download. The image upload is queued first so the DMA overlaps
 * the host-side trig pass. kps: n rows of `cols` (2..4) doubles; kept: room for n input
 * indices; out: room for n descriptors; *m receives the number kept (input order).
 * A big float64 frame goes up in row bands and each band's keypoints are extracted while the
 * next band is in flight ("upload_bands"). Page-locked img / out buffers (cudaHostAlloc,
 * clatch_host_alloc) make the transfers plain DMAs; ordinary memory works, only slower. */
CLATCH_API int clatch_describe_all_u8(clatch_ctx* ctx, const uint8_t* img, int width, int height, size_t pitch,
                           const double* kps, size_t n, int cols, int workers, int64_t* kept,
                           uint8_t* out, size_t* m);
CLATCH_API int clatch_describe_all_f64(clatch_ctx* ctx, const double* img, int width, int height, size_t pitch,
                            const double* kps, size_t n, int cols, int workers, int64_t* kept,
                            uint8_t* out, size_t* m);

/* describe_all over a batch of images (BASELINE config 3: many images x many keypoints per GPU).
 * Image i is imgs[i] (widths[i] x heights[i], pitches[i] elements per row) with counts[i]
 * keypoint rows of `cols` doubles at kps[i]; results go to kept[i] (room for counts[i]
 * indices), out[i] (room for counts[i] descriptors) and m[i]. Uploads, host trig, kernels and
 * downloads of consecutive images are pipelined over two streams; with page-locked host
 * buffers the copies are fully asynchronous. Results are identical to num_images calls of
 * clatch_describe_all_*. */
CLATCH_API int clatch_describe_batch_u8(clatch_ctx* ctx, const uint8_t* const* imgs, const int* widths, const int* heights,
                             const size_t* pitches, const double* const* kps, const size_t* counts, int cols,
                             size_t num_images, int workers, int64_t* const* kept, uint8_t* const* out,
                             size_t* m);
CLATCH_API int clatch_describe_batch_f64(clatch_ctx* ctx, const double* const* imgs, const int* widths, const int* heights,
                              const size_t* pitches, const double* const* kps, const size_t* counts, int cols,
                              size_t num_images, int workers, int64_t* const* kept, uint8_t* const* out,
                              size_t* m);

/* Device-resident forms: all pointers are device memory on the context's device,
 * work is queued on `stream` (a cudaStream_t; NULL = the legacy default stream)
 * and NOT synchronised. */
CLATCH_API int clatch_extract_u8_dev(clatch_ctx* ctx, const uint8_t* d_img, int width, int height,
                          size_t pitch, const double* d_xycs, size_t M, uint8_t* d_out,
                          void* stream);
CLATCH_API int clatch_extract_f64_dev(clatch_ctx* ctx, const double* d_img, int width, int height,
                           size_t pitch, const double* d_xycs, size_t M, uint8_t* d_out,
                           void* stream);

/* Diagnostics, device-resident form: the samples the default extraction kernel's ESTIMATE works from — for each
 * prepared keypoint record its 64 x 64 window as round(256 * v) uint16, resampled in fp32 with fixed-point
 * coordinates (M x 4096 values, row-major). Nothing in the reference corresponds to it: the reference's window
 * (src/descriptor.cpp:29-49) is what these values must stay within 0.66 units of for the estimate's error bound to
 * hold, and a test checks exactly that; descriptors never depend on it beyond that bound. */
CLATCH_API int clatch_estimate_planes_u8_dev(clatch_ctx* ctx, const uint8_t* d_img, int width, int height,
                                  size_t pitch, const double* d_xycs, size_t M, uint16_t* d_out,
                                  void* stream);

/* ---- matching (replaces knn2 / the two parallel_for passes of match_brute_force,
 * src/match.cpp:33-67; hamming :14-31 is the per-pair arithmetic) -----------------
 * For every query q: best_idx = lowest train index at the minimum Hamming
 * distance, best_dist = that distance, second_dist = the runner-up distance (may
 * equal best_dist; 8*bytes+1 when N == 1). Any of the three outputs may be NULL.
 * N == 0 fails with CLATCH_ERR_EMPTY_GALLERY (checked before Q == 0, as the
 * reference does); Q == 0 succeeds and writes nothing. `bytes` is the descriptor
 * length (any > 0; 64 takes the tiled kernel). */
CLATCH_API int clatch_match_top2(clatch_ctx* ctx, const uint8_t* queries, size_t Q, const uint8_t* train,
                      size_t N, int bytes, int32_t* best_idx, int32_t* best_dist,
                      int32_t* second_dist);
CLATCH_API int clatch_match_top2_dev(clatch_ctx* ctx, const uint8_t* d_queries, size_t Q,
                          const uint8_t* d_train, size_t N, int bytes, int32_t* d_best_idx,
                          int32_t* d_best_dist, int32_t* d_second_dist, void* stream);

/* Filter pass of match_brute_force (src/match.cpp:69-79), host side, over forward
 * top-2 triples: ratio (accept iff best < ratio * second, evaluated in double),
 * max_distance (accept iff best <= max), cross-check (accept iff
 * reverse_best[best_idx] == q; pass NULL to skip). out: up to Q rows {probe,
 * gallery, distance, second_distance} in ascending probe order; *count rows. */
CLATCH_API int clatch_filter_matches(const int32_t* best_idx, const int32_t* best_dist,
                          const int32_t* second_dist, size_t Q, int has_ratio, double ratio,
                          int has_max, int max_distance, const int32_t* reverse_best,
                          int32_t* out, size_t* count);

/* Whole match_brute_force (src/match.cpp:52-81) on host buffers: forward top-2 on
 * the device, reverse pass on the device when cross_check, filter pass on the host. */
CLATCH_API int clatch_match_brute_force(clatch_ctx* ctx, const uint8_t* probes, size_t Q,
                             const uint8_t* gallery, size_t N, int bytes, int has_ratio,
                             double ratio, int cross_check, int has_max, int max_distance,
                             int32_t* out, size_t* count);

/* ---- trainer scoring (the parallel body of select_triplets, src/pattern.cpp:340-346,397-400) ---
 * bit (c, i) = triplet_bit(window i, candidate c, mask) for n upright 64x64 training patches
 * (`windows`: n x 4096 doubles, row-major, as Window64::from_image lays them out) and C candidate
 * triplets (`candidates`: C rows {ax, ay, bx, by, cx, cy}, coordinates in [0, 64-K]). `mask` is
 * K*K weights or NULL for all ones. out: C rows of row_bytes >= ceil(n/8) bytes in BitVector
 * order (bit i of row c at byte i>>3, bit i&7; include/latch/pattern.hpp:70-90). Greedy
 * selection (src/pattern.cpp:431-450) stays on the host. */
CLATCH_API int clatch_triplet_bits(clatch_ctx* ctx, const double* windows, size_t n, const int16_t* candidates,
                        size_t C, int K, const double* mask, uint8_t* out, size_t row_bytes);

/* ---- device-resident descriptor sets (64-byte descriptors) -----------------------------
 * A set owns a device copy of n descriptors plus the int8 operand forms the tensor-core
 * matcher consumes, so that extraction output can feed any number of matches without
 * going back to the host and without being re-expanded (the SfM-style "every image against
 * every other image" workload; the reference has no counterpart — it re-reads
 * std::vector<Descriptor> per call, src/match.cpp:52-67).
 * `descriptors` is host memory (on_device = 0) or device memory on the context's device
 * (on_device = 1, and any work producing it must already be complete or ordered before the
 * context's stream); it is copied, the caller keeps ownership. */
typedef struct clatch_set clatch_set;
CLATCH_API int clatch_set_create(clatch_ctx* ctx, const uint8_t* descriptors, size_t n, int on_device, clatch_set** out);
CLATCH_API void clatch_set_destroy(clatch_set* set);
CLATCH_API size_t clatch_set_count(const clatch_set* set);

/* match_brute_force (src/match.cpp:52-81) between two resident sets; same outputs as
 * clatch_match_brute_force. */
CLATCH_API int clatch_match_sets(clatch_ctx* ctx, const clatch_set* probes, const clatch_set* gallery, int has_ratio,
                      double ratio, int cross_check, int has_max, int max_distance, int32_t* out,
                      size_t* count);

/* Batched form: pairs[2*p], pairs[2*p+1] index `sets`; pair p matches sets[pairs[2p]] (probes)
 * against sets[pairs[2p+1]] (gallery) with the given filters. All pairs (and, with
 * cross_check, their reverse passes) run in as few kernel launches as memory allows. The
 * accepted rows {probe, gallery, distance, second_distance} of all pairs are concatenated in
 * `out` (room for cap_rows rows); pair p owns rows [offsets[p], offsets[p+1]). Fails with
 * CLATCH_ERR_INVALID if cap_rows is too small, CLATCH_ERR_EMPTY_GALLERY on an empty gallery. */
CLATCH_API int clatch_match_set_pairs(clatch_ctx* ctx, const clatch_set* const* sets, size_t num_sets,
                           const int32_t* pairs, size_t num_pairs, int has_ratio, double ratio,
                           int cross_check, int has_max, int max_distance, int32_t* out, size_t cap_rows,
                           size_t* offsets);

/* Diagnostic for the tensor-core matcher: runs it on host buffers and also returns the raw
 * int32 accumulators of the first 128-query x 256-train tile (row-major 128 x 256; entry
 * (i, j) must equal 512 - 2 * hamming(query i, train j) for i < Q, j < N). */
CLATCH_API int clatch_debug_tc_tile(clatch_ctx* ctx, const uint8_t* queries, size_t Q, const uint8_t* train,
                         size_t N, int32_t* tile_out, int32_t* best_idx, int32_t* best_dist,
                         int32_t* second_dist);

/* Kernel launches issued through this context since creation (bench.py's
 * gpu_launches claim is read from here, not estimated). */
CLATCH_API uint64_t clatch_launch_count(clatch_ctx* ctx);

/* Page-locked host memory for buffers that cross the bus (descriptor arrays a caller passes from
 * describe to match): with it the transfers above are plain DMAs instead of copies staged through
 * the driver's bounce buffer. Optional — every entry point accepts ordinary memory. */
CLATCH_API int clatch_host_alloc(size_t bytes, void** out);
CLATCH_API int clatch_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* CLATCH_H */
