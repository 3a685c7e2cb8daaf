// FAST-9 detection, 3x3 non-maximum suppression and intensity-centroid moments for sm_100a —
// the step that feeds the extraction path ("next" row of SURVEY.md §8f), bit-identical to the
// reference (paths relative to /root/reference/proj):
//   evaluate_arc        src/detect.cpp:26-66    segment test + score of the maximal arc
//   fast_detect         src/detect.cpp:76-117   score field, NMS with (y, x) tie rule, row-major order
//   orient              src/detect.cpp:119-146  m10 / m01 over the radius-15 disc
//   detect_and_orient   src/detect.cpp:148-157  drop detections whose disc leaves the image
// Exactness: scores and moments are accumulated in the reference's order with individually
// rounded fp64 operations; atan2 stays on the host libm (the C ABI wrapper applies it), for the
// same reason cos/sin do.
//
// Kernels: (1) score field, one thread per pixel; (2) keep-flags + per-block counts over
// row-major blocks of 256 pixels; (3) single-block exclusive scan of the block counts;
// (4) ordered compaction (ballot ranks inside the block) -> detections in (y, x) order;
// (5) one thread per detection walks the disc sequentially for the moments.

#include "clatch_internal.cuh"

namespace clatch {

namespace {

constexpr int kBlock = 256;

__constant__ int c_circle_x[16] = {0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3, -3, -3, -2, -1};
__constant__ int c_circle_y[16] = {-3, -3, -2, -1, 0, 1, 2, 3, 3, 3, 2, 1, 0, -1, -2, -3};

template <typename Pixel>
__device__ __forceinline__ double pixel(const Pixel* img, size_t pitch, int x, int y) {
    return static_cast<double>(img[static_cast<size_t>(y) * pitch + x]);
}

// Longest circular run of set bits in a 16-bit mask, scanned the way the reference does
// (two laps, first maximal run wins): returns its length (capped at 16) and start.
__device__ __forceinline__ int longest_run(unsigned mask, int& start) {
    int best_len = 0, best_start = 0, run = 0;
    for (int i = 0; i < 32; ++i) {
        if ((mask >> (i & 15)) & 1u) {
            ++run;
            if (run > best_len) {
                best_len = run;
                best_start = i - run + 1;
            }
        } else {
            run = 0;
        }
    }
    start = best_start;
    return best_len > 16 ? 16 : best_len;
}

template <typename Pixel>
__global__ void fast_score_kernel(const Pixel* __restrict__ img, int w, int h, size_t pitch, double threshold,
                                  double* __restrict__ scores) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= w || y >= h) return;
    double score = 0.0;
    if (x >= 3 && y >= 3 && x < w - 3 && y < h - 3) {
        const double center = pixel(img, pitch, x, y);
        const double hi = __dadd_rn(center, threshold);
        const double lo = __dsub_rn(center, threshold);
        double v[16];
        unsigned bright = 0, dark = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            v[i] = pixel(img, pitch, x + c_circle_x[i], y + c_circle_y[i]);
            bright |= (v[i] > hi ? 1u : 0u) << i;
            dark |= (v[i] < lo ? 1u : 0u) << i;
        }
        if (__popc(bright) >= 9 || __popc(dark) >= 9) {
            for (int pol = 0; pol < 2; ++pol) {   // bright first, src/detect.cpp:41
                int start;
                const int len = longest_run(pol == 0 ? bright : dark, start);
                if (len < 9) continue;
                double s = 0.0;
                for (int i = start; i < start + len; ++i)
                    s = __dadd_rn(s, __dsub_rn(fabs(__dsub_rn(v[i & 15], center)), threshold));
                score = s;
                break;
            }
        }
    }
    scores[static_cast<size_t>(y) * w + x] = score;
}

// keep(x, y): fired and (without NMS) anything, (with NMS) a 3x3 maximum under the reference's
// tie rule — an equal neighbour earlier in (y, x) order suppresses (src/detect.cpp:97-108).
__device__ __forceinline__ bool keep_pixel(const double* scores, int w, int h, int x, int y, bool nms) {
    if (x < 3 || y < 3 || x >= w - 3 || y >= h - 3) return false;
    const double s = scores[static_cast<size_t>(y) * w + x];
    if (!(s > 0.0)) return false;
    if (!nms) return true;
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            if (dx == 0 && dy == 0) continue;
            const int nx = x + dx, ny = y + dy;
            if (nx < 3 || ny < 3 || nx >= w - 3 || ny >= h - 3) continue;
            const double ns = scores[static_cast<size_t>(ny) * w + nx];
            if (ns > s || (ns == s && (ny < y || (ny == y && nx < x)))) return false;
        }
    return true;
}

__global__ void count_kernel(const double* __restrict__ scores, int w, int h, int nms, unsigned* __restrict__ counts) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * kBlock + threadIdx.x;
    const bool keep = idx < static_cast<size_t>(w) * h &&
                      keep_pixel(scores, w, h, static_cast<int>(idx % w), static_cast<int>(idx / w), nms != 0);
    const int total = __syncthreads_count(keep);
    if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

// Exclusive scan of n block counts by one 1024-thread block; counts[n] receives the total.
__global__ void scan_kernel(unsigned* counts, unsigned n) {
    __shared__ unsigned s_part[1024];
    const unsigned per = (n + 1023) / 1024;
    const unsigned begin = threadIdx.x * per, end = min(n, begin + per);
    unsigned sum = 0;
    for (unsigned i = begin; i < end; ++i) sum += counts[i];
    s_part[threadIdx.x] = sum;
    __syncthreads();
    for (unsigned off = 1; off < 1024; off <<= 1) {   // Hillis-Steele inclusive scan
        const unsigned v = threadIdx.x >= off ? s_part[threadIdx.x - off] : 0;
        __syncthreads();
        s_part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned run = threadIdx.x == 0 ? 0 : s_part[threadIdx.x - 1];
    for (unsigned i = begin; i < end; ++i) {
        const unsigned c = counts[i];
        counts[i] = run;
        run += c;
    }
    if (threadIdx.x == 1023) counts[n] = s_part[1023];
}

__global__ void compact_kernel(const double* __restrict__ scores, int w, int h, int nms,
                               const unsigned* __restrict__ offsets, Detection* __restrict__ out) {
    __shared__ unsigned s_warp[kBlock / 32];
    const size_t idx = static_cast<size_t>(blockIdx.x) * kBlock + threadIdx.x;
    const int x = static_cast<int>(idx % w), y = static_cast<int>(idx / w);
    const bool keep = idx < static_cast<size_t>(w) * h && keep_pixel(scores, w, h, x, y, nms != 0);
    const unsigned ballot = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_warp[warp] = __popc(ballot);
    __syncthreads();
    unsigned base = offsets[blockIdx.x];
    for (int i = 0; i < warp; ++i) base += s_warp[i];
    if (keep) {
        Detection d;
        d.x = x;
        d.y = y;
        d.score = scores[idx];
        d.m10 = d.m01 = 0.0;
        d.valid = 1;
        d.pad = 0;
        out[base + __popc(ballot & ((1u << lane) - 1))] = d;
    }
}

// orient for an integer-centred keypoint: sequential row-major walk of the disc, each
// product and sum individually rounded (no FMA), src/detect.cpp:128-141.
template <typename Pixel>
__global__ void moments_kernel(const Pixel* __restrict__ img, int w, int h, size_t pitch, int radius,
                               Detection* __restrict__ det, unsigned n) {
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Detection d = det[i];
    if (d.x - radius < 0 || d.y - radius < 0 || d.x + radius > w - 1 || d.y + radius > h - 1) {
        det[i].valid = 0;   // detect_and_orient drops it, src/detect.cpp:152-154
        return;
    }
    double m10 = 0.0, m01 = 0.0;
    const int r2 = radius * radius;
    for (int v = -radius; v <= radius; ++v)
        for (int u = -radius; u <= radius; ++u) {
            if (u * u + v * v > r2) continue;
            const double intensity = pixel(img, pitch, d.x + u, d.y + v);
            m10 = __dadd_rn(m10, __dmul_rn(static_cast<double>(u), intensity));
            m01 = __dadd_rn(m01, __dmul_rn(static_cast<double>(v), intensity));
        }
    det[i].m10 = m10;
    det[i].m01 = m01;
}

} // namespace

// Runs detection on a device image. Leaves `*count` detections (row-major order) in
// ctx->det as DetectionRecord rows; the caller downloads them and finishes on the host.
template <typename Pixel>
static int detect_device(clatch_ctx* ctx, const Pixel* d_img, int w, int h, size_t pitch, double threshold, int nms,
                         int orient, int radius, cudaStream_t st, unsigned* count) {
    const size_t pixels = static_cast<size_t>(w) * h;
    const unsigned blocks = static_cast<unsigned>((pixels + kBlock - 1) / kBlock);
    if (int rc = ctx->scores.reserve(sizeof(double) * pixels)) return rc;
    if (int rc = ctx->counts.reserve(sizeof(unsigned) * (blocks + 1))) return rc;
    double* scores = ctx->scores.as<double>();
    unsigned* counts = ctx->counts.as<unsigned>();
    dim3 b2(32, 8), g2((w + 31) / 32, (h + 7) / 8);
    fast_score_kernel<Pixel><<<g2, b2, 0, st>>>(d_img, w, h, pitch, threshold, scores);
    count_kernel<<<blocks, kBlock, 0, st>>>(scores, w, h, nms, counts);
    scan_kernel<<<1, 1024, 0, st>>>(counts, blocks);
    ctx->launches += 3;
    CLATCH_CUDA(cudaGetLastError());
    unsigned total = 0;
    CLATCH_CUDA(cudaMemcpyAsync(&total, counts + blocks, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CLATCH_CUDA(cudaStreamSynchronize(st));
    *count = total;
    if (total == 0) return CLATCH_OK;
    if (int rc = ctx->det.reserve(sizeof(Detection) * total)) return rc;
    Detection* det = ctx->det.as<Detection>();
    compact_kernel<<<blocks, kBlock, 0, st>>>(scores, w, h, nms, counts, det);
    ++ctx->launches;
    if (orient) {
        moments_kernel<Pixel><<<(total + 127) / 128, 128, 0, st>>>(d_img, w, h, pitch, radius, det, total);
        ++ctx->launches;
    }
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

int launch_detect_u8(clatch_ctx* ctx, const uint8_t* d_img, int w, int h, size_t pitch, double threshold, int nms,
                     int orient, int radius, cudaStream_t st, unsigned* count) {
    return detect_device<uint8_t>(ctx, d_img, w, h, pitch, threshold, nms, orient, radius, st, count);
}

int launch_detect_f64(clatch_ctx* ctx, const double* d_img, int w, int h, size_t pitch, double threshold, int nms,
                      int orient, int radius, cudaStream_t st, unsigned* count) {
    return detect_device<double>(ctx, d_img, w, h, pitch, threshold, nms, orient, radius, st, count);
}

} // namespace clatch
