// LATCH descriptor extraction for sm_100a — bit-exact restatement of the reference's
// fp64 arithmetic (paths relative to /root/reference/proj):
//   extract_window    src/descriptor.cpp:29-49    oriented 64x64 bilinear resample
//   sample_bilinear   src/image.cpp:109-126       top/bottom/blend, each op rounded
//   triplet_bit       src/descriptor.cpp:51-77    two sequential weighted SSD chains, strict >
//   describe          src/descriptor.cpp:79-88    LSB-first bit packing
//
// Numerical contract: every multiply/add is an individually rounded
// fp64 operation (__dmul_rn/__dadd_rn/__dsub_rn never contract into FMA), the
// accumulation order inside one SSD chain is the reference's row-major order, and
// cos/sin arrive from the host's libm. No tree reductions anywhere.
//
// Kernels in this file (all persistent, one CTA per SM unless noted), oldest to newest:
//   extract_fast_kernel     one fp64 window per CTA, 4 CTAs/SM                     (extract_variant 0)
//   extract_quad_kernel     four fp64 windows per CTA, conflict-free 64-bit loads  (1; also every non-u8-valued image)
//   extract_filt_kernel     four split (fp32 + low word) windows; every bit decided by an fp32 estimate with a
//                           proven error bound, exact fp64 chains only for undecided bits     (2)
//   extract_pipe_kernel     the same estimate with double-buffered planes, texture-unit footprints and resampling
//                           overlapped with the estimate (every warp does both halves)       (3)
//   extract_roles_kernel    variant 3 with dedicated producer / consumer warps; the default for u8-valued images (4)
//   extract_generic_kernel  any T % 8 == 0, 1 <= K <= 64, real weights: (w*e)*e literally
// Common shape: (1) the <=92x92 footprint of a keypoint reaches the SM (u8 tile in shared memory, or
// tex2Dgather on a u8 CUDA array), (2) the 4096 window samples are resampled in unfused fp64, (3) each
// thread owns whole triplets and reads the window with immediate-offset shared loads, (4) predicate
// bits are packed with __ballot_sync and stored as 32-bit words.

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "clatch_internal.cuh"
#include "slot_assign.hpp"

namespace clatch {

namespace {

constexpr int kThreads = 256;

struct ExtractParams {
    const void* img;
    int width, height;
    size_t pitch;              // elements
    const double* xycs;        // M x {x, y, cos, sin}
    unsigned long long M;
    uint8_t* out;              // M x T/8
    const ushort4* slots;      // fast kernel: T x {a, b, c, bit}
    const ushort4* slots_sw;   // packed-plane kernel: the one-window placement (fp64 window, stride kWinStride) of its window-wide pass
    const short* triplets;     // generic kernel: T x 6
    const double* weights;     // generic kernel: K x K mask weights (per-context device copy; warp-uniform reads)
    int T, K;
    const int* flags;          // optional device flags (f64 promotion), may be null
    int run_if_flag;           // run only when flags[0] == run_if_flag (if flags != null)
    unsigned long long* stats; // optional {triplets recomputed exactly, warps that took the exact pass}
    uint2* route;              // optional, host-mapped: per CTA {windows that took the exact pass, windows} of this launch
    cudaTextureObject_t tex;   // pipelined kernel: the u8 image as a gather-enabled CUDA array
    cudaTextureObject_t texn;  // packed-plane kernel: the same array read as texel / 255 (cudaReadModeNormalizedFloat)
    unsigned two23;            // packed-plane kernel: 0x4B000000, see ssd_estimate_h16_2
    int dbg;                   // diagnostics (CLATCH_EX_DEBUG): 1 = skip the estimate, 2 = skip the resampling (timing only, wrong bits)
    const unsigned* out_index; // optional: descriptor of record j goes to row out_index[j] (quad / pipelined kernels)
    unsigned* tickets;         // packed-plane kernel: {next quad ticket, CTAs finished}, both 0 between launches (nullptr: static round-robin)
    unsigned long long* trace; // optional (CLATCH_EX_TRACE=1): kExTrace globaltimer stamps per CTA of the default kernel
};

constexpr int kFlagBlockBytes = 64;   // classification flag + pixel range of a float64 image, see classify_convert_kernel
constexpr int kExTrace = 128;   // [0] entry, [1] texture array complete, [2 + i] end of pipeline iteration i - 1 (bit 63: exact pass)

__device__ __forceinline__ unsigned long long ex_global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Exact u8 -> f64 without the 16-lane/clk conversion pipe (I2F.F64 runs at 16/clk/SM on
// B200, profiles/r1a_pipe_peaks.json): splice the byte into the mantissa of 2^52 and
// subtract 2^52 — one DADD on the 64-lane fp64 pipe, result exactly v.
__device__ __forceinline__ double u8_to_f64(unsigned v) {
    return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(v)), 4503599627370496.0);
}

// floor() of a double in (0, 2^31) as both int and double, again without F2I/I2F:
// adding 2^52 + 2^51 with round-toward-minus-infinity leaves magic + floor(s) exactly (the
// ulp is 1 at that magnitude), the integer sits in the low mantissa word, and subtracting
// the magic is exact. So fx = s - floor(s) is bit-identical to the reference's `x - x0`
// (src/image.cpp:113,121) at two DADDs instead of two 16-lane/clk conversions.
__device__ __forceinline__ void floor_exact(double s, int& i, double& f) {
    const double kMagic = 6755399441055744.0;
    const double t = __dadd_rd(s, kMagic);
    i = __double2loint(t);
    f = __dsub_rn(t, kMagic);
}

// One bilinear sample with the reference's exact operation order (src/image.cpp:121-125).
__device__ __forceinline__ double blend(double fx, double fy, double p00, double p10, double p01,
                                        double p11) {
    const double gx = __dsub_rn(1.0, fx);
    const double gy = __dsub_rn(1.0, fy);
    const double top = __dadd_rn(__dmul_rn(gx, p00), __dmul_rn(fx, p10));
    const double bottom = __dadd_rn(__dmul_rn(gx, p01), __dmul_rn(fx, p11));
    return __dadd_rn(__dmul_rn(gy, top), __dmul_rn(fy, bottom));
}

// Stage rows [ty0, ty0+92) x 16-byte-aligned columns [ax0, ax0+112) of a u8 image.
template <int kGroup = kThreads>
__device__ __forceinline__ void stage_tile_u8(uint8_t* tile, const uint8_t* img, size_t pitch,
                                              int height, int ax0, int ty0, bool aligned, int tid = threadIdx.x) {
    if (aligned) {
        constexpr int kChunks = kTileW / 16;
        for (int i = tid; i < kTileH * kChunks; i += kGroup) {
            const int r = i / kChunks, c = i - r * kChunks;
            const int gx = ax0 + 16 * c;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (static_cast<size_t>(gx) < pitch && ty0 + r < height)
                v = __ldg(reinterpret_cast<const uint4*>(img + static_cast<size_t>(ty0 + r) * pitch + gx));
            *reinterpret_cast<uint4*>(tile + r * kTileW + 16 * c) = v;
        }
    } else {
        for (int i = tid; i < kTileH * kTileW; i += kGroup) {
            const int r = i / kTileW, c = i - r * kTileW;
            const int gx = ax0 + c;
            uint8_t v = 0;
            if (static_cast<size_t>(gx) < pitch && ty0 + r < height)
                v = __ldg(img + static_cast<size_t>(ty0 + r) * pitch + gx);
            tile[i] = v;
        }
    }
}

// Phase A: resample the oriented window (src/descriptor.cpp:35-47). Thread -> column
// u = tid & 63, rows v = (tid >> 6) + 4k; sx = (x + c*du) - s*dv, sy = (y + s*du) + c*dv.
template <bool kU8>
__device__ __forceinline__ void build_window(double* win, const uint8_t* tile, int ax0, int ty0,
                                             const double* img64, size_t pitch, double x, double y,
                                             double c, double s, int tid = threadIdx.x) {
    const int u = tid & 63;
    const double du = static_cast<double>(u) - 31.5;
    const double xa = __dadd_rn(x, __dmul_rn(c, du));
    const double ya = __dadd_rn(y, __dmul_rn(s, du));
#pragma unroll 4
    for (int v = tid >> 6; v < kWindow; v += kThreads / 64) {
        const double dv = static_cast<double>(v) - 31.5;
        const double sx = __dsub_rn(xa, __dmul_rn(s, dv));
        const double sy = __dadd_rn(ya, __dmul_rn(c, dv));
        int x0, y0;                           // inside the margin: 1 <= x0 <= width-3, no clamps fire
        double x0f, y0f;
        floor_exact(sx, x0, x0f);
        floor_exact(sy, y0, y0f);
        const double fx = __dsub_rn(sx, x0f);
        const double fy = __dsub_rn(sy, y0f);
        double p00, p10, p01, p11;
        if (kU8) {
            const uint8_t* p = tile + (y0 - ty0) * kTileW + (x0 - ax0);
            p00 = u8_to_f64(p[0]);
            p10 = u8_to_f64(p[1]);
            p01 = u8_to_f64(p[kTileW]);
            p11 = u8_to_f64(p[kTileW + 1]);
        } else {
            const double* p = img64 + static_cast<size_t>(y0) * pitch + x0;
            p00 = __ldg(p);
            p10 = __ldg(p + 1);
            p01 = __ldg(p + pitch);
            p11 = __ldg(p + pitch + 1);
        }
        win[v * kWinStride + u] = blend(fx, fy, p00, p10, p01, p11);
    }
}

// Same resampling with the per-row products s*dv and c*dv read from a 2 x 64 shared table
// (filled once per keypoint; all lanes of a warp share v, so the reads broadcast).
template <bool kU8>
__device__ __forceinline__ void build_window_tab(double* win, const uint8_t* tile, int ax0, int ty0,
                                                 const double* img64, size_t pitch, double x, double y,
                                                 double c, double s, const double* tab, int tid) {
    const int u = tid & 63;
    const double du = static_cast<double>(u) - 31.5;
    const double xa = __dadd_rn(x, __dmul_rn(c, du));
    const double ya = __dadd_rn(y, __dmul_rn(s, du));
#pragma unroll 4
    for (int v = tid >> 6; v < kWindow; v += kThreads / 64) {
        const double sx = __dsub_rn(xa, tab[v]);
        const double sy = __dadd_rn(ya, tab[kWindow + v]);
        int x0, y0;
        double x0f, y0f;
        floor_exact(sx, x0, x0f);
        floor_exact(sy, y0, y0f);
        const double fx = __dsub_rn(sx, x0f);
        const double fy = __dsub_rn(sy, y0f);
        double p00, p10, p01, p11;
        if (kU8) {
            const uint8_t* p = tile + (y0 - ty0) * kTileW + (x0 - ax0);
            p00 = u8_to_f64(p[0]);
            p10 = u8_to_f64(p[1]);
            p01 = u8_to_f64(p[kTileW]);
            p11 = u8_to_f64(p[kTileW + 1]);
        } else {
            const double* p = img64 + static_cast<size_t>(y0) * pitch + x0;
            p00 = __ldg(p);
            p10 = __ldg(p + 1);
            p01 = __ldg(p + pitch);
            p11 = __ldg(p + pitch + 1);
        }
        win[v * kWinStride + u] = blend(fx, fy, p00, p10, p01, p11);
    }
}

// Phase B (specialised): one triplet = two independent 49-term chains over the
// 7x7 live pixels of the 8x8 patch, row-major (src/descriptor.cpp:61-75 with the
// zero-weight terms skipped — exact because w*e*e is +0.0 there and d + 0.0 == d).
// `ob`/`oc` are the companions in LOAD order; the slot planner (slot_assign.hpp) may have
// swapped them to dodge a bank conflict, in which case the caller tests d2 > d1.
__device__ __forceinline__ bool triplet_bit_7x7(const double* win, int oa, int ob, int oc, bool swapped) {
    const double* pa = win + oa;
    const double* pb = win + ob;
    const double* pc = win + oc;
    double d1 = 0.0, d2 = 0.0;
#pragma unroll
    for (int r = 0; r < 7; ++r) {
#pragma unroll
        for (int c = 0; c < 7; ++c) {
            const int o = r * kWinStride + c;
            const double a = pa[o];
            const double e1 = __dsub_rn(a, pb[o]);
            const double e2 = __dsub_rn(a, pc[o]);
            d1 = __dadd_rn(d1, __dmul_rn(e1, e1));
            d2 = __dadd_rn(d2, __dmul_rn(e2, e2));
        }
    }
    return swapped ? d2 > d1 : d1 > d2;
}

template <bool kU8>
__global__ void __launch_bounds__(kThreads, 4) extract_fast_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;

    __shared__ __align__(16) double s_win[kWindow * kWinStride];
    __shared__ __align__(16) uint8_t s_tile[kU8 ? kTileH * kTileW : 16];
    __shared__ uint8_t s_bits[kFastT];

    const int tid = threadIdx.x;
    // Slots tid and tid + 256 stay in registers for the whole persistent loop.
    const ushort4 slot0 = __ldg(p.slots + tid);
    const ushort4 slot1 = __ldg(p.slots + tid + kThreads);
    const bool aligned = kU8 && (reinterpret_cast<uintptr_t>(p.img) % 16 == 0) && (p.pitch % 16 == 0);

    for (unsigned long long kp = blockIdx.x; kp < p.M; kp += gridDim.x) {
        const double x = __ldg(p.xycs + 4 * kp + 0);
        const double y = __ldg(p.xycs + 4 * kp + 1);
        const double c = __ldg(p.xycs + 4 * kp + 2);
        const double s = __ldg(p.xycs + 4 * kp + 3);
        int ax0 = 0, ty0 = 0;
        if (kU8) {
            // Footprint: columns floor(x)-45 .. floor(x)+46, same for rows (|offset| <= 44.55 px).
            const int tx0 = __double2int_rd(x) - 45;
            ty0 = __double2int_rd(y) - 45;
            ax0 = aligned ? (tx0 & ~15) : tx0;
            stage_tile_u8(s_tile, static_cast<const uint8_t*>(p.img), p.pitch, p.height, ax0, ty0,
                          aligned);
        }
        __syncthreads();   // tile ready; previous keypoint's window/bit readers are done
        build_window<kU8>(s_win, s_tile, ax0, ty0, static_cast<const double*>(p.img), p.pitch, x, y,
                          c, s);
        __syncthreads();
        s_bits[slot0.w & 0x7fff] = triplet_bit_7x7(s_win, slot0.x, slot0.y, slot0.z, slot0.w >> 15);
        s_bits[slot1.w & 0x7fff] = triplet_bit_7x7(s_win, slot1.x, slot1.y, slot1.z, slot1.w >> 15);
        __syncthreads();
        // Bit t -> byte t>>3, bit t&7 == bit t of the little-endian 32-bit word t>>5.
        const unsigned w0 = __ballot_sync(0xffffffffu, s_bits[tid] != 0);
        const unsigned w1 = __ballot_sync(0xffffffffu, s_bits[tid + kThreads] != 0);
        if ((tid & 31) == 0) {
            unsigned* out32 = reinterpret_cast<unsigned*>(p.out + kp * (kFastT / 8));
            out32[tid >> 5] = w0;
            out32[(tid >> 5) + kThreads / 32] = w1;
        }
    }
}


// ---- quad kernel: four keypoints per CTA iteration, conflict-free SSD loads ----------------
// Same arithmetic as extract_fast_kernel; what changes is who sits next to whom. The CTA
// (1024 threads, one per SM) keeps four windows in shared memory, window w displaced by
// 4*w bank pairs (kQuadWinPitch % 16 == 4). In the SSD phase each half-warp holds 4 triplets x
// 4 keypoints (lane = 4*i + w): the four lanes of a triplet land on residues r, r+4, r+8,
// r+12, so the half-warp is conflict-free whenever its 4 triplets differ mod 4 in each load —
// which plan_slots_quad arranges for all but ~7 % of the (half-warp, load) pairs.
constexpr int kQuad = 4;
constexpr int kQuadThreads = kQuad * kThreads;                       // 1024
constexpr int kQuadWinPitch = 4164;                                  // doubles; 4164 % 16 == 4
constexpr int kQuadTileBytes = kTileH * kTileW;                      // 10304
constexpr int kQuadSmemBytes = kQuad * kQuadWinPitch * 8             // windows
                               + 2 * kQuad * kQuadTileBytes          // double-buffered u8 tiles
                               + kQuad * kFastT                      // predicate bytes
                               + kQuad * 2 * kWindow * 8;            // s*dv, c*dv tables

// Footprint origin of keypoint (x, y): rows floor(y)-45.., 16-byte aligned columns.
__device__ __forceinline__ void tile_origin(double x, double y, bool aligned, int& ax0, int& ty0) {
    int xi, yi;
    double unused;
    floor_exact(x, xi, unused);
    floor_exact(y, yi, unused);
    ty0 = yi - 45;
    ax0 = aligned ? ((xi - 45) & ~15) : (xi - 45);
}

// Asynchronous (LDGSTS) staging of one keypoint's tile by a 256-thread group.
__device__ __forceinline__ void stage_tile_async(uint8_t* tile, const uint8_t* img, size_t pitch, int height,
                                                 int ax0, int ty0, int gt) {
    constexpr int kChunks = kTileW / 16;
    for (int i = gt; i < kTileH * kChunks; i += kThreads) {
        const int r = i / kChunks, c = i - r * kChunks;
        const int gx = ax0 + 16 * c;
        const bool in = static_cast<size_t>(gx) < pitch && ty0 + r < height;
        const uint8_t* src = in ? img + static_cast<size_t>(ty0 + r) * pitch + gx : img;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(tile + r * kTileW + 16 * c));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(in ? 16 : 0) : "memory");
    }
}

template <bool kU8>
__global__ void __launch_bounds__(kQuadThreads, 1) extract_quad_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;

    extern __shared__ __align__(16) uint8_t s_quad[];
    double* const s_win = reinterpret_cast<double*>(s_quad);
    uint8_t* const s_tile = s_quad + kQuad * kQuadWinPitch * 8;
    uint8_t* const s_bits = s_tile + 2 * kQuad * kQuadTileBytes;
    double* const s_tab = reinterpret_cast<double*>(s_bits + kQuad * kFastT);

    const int tid = threadIdx.x;
    // staging / resampling: thread group `grp` (256 threads) owns keypoint `grp` of the quad
    const int grp = tid >> 8, gt = tid & (kThreads - 1);
    // SSD: half-warp hw holds triplet slots 4*hw .. 4*hw+3 (and +256) for keypoints 0..3
    const int hw = tid >> 4, j = tid & 15, kb = j & 3, ti = j >> 2;
    const ushort4 slot0 = __ldg(p.slots + 4 * hw + ti);
    const ushort4 slot1 = __ldg(p.slots + 4 * hw + ti + kFastT / 2);
    const double* const my_win = s_win + kb * kQuadWinPitch;
    uint8_t* const my_bits = s_bits + kb * kFastT;
    double* const my_tab = s_tab + grp * 2 * kWindow;
    const uint8_t* const img8 = static_cast<const uint8_t*>(p.img);
    const bool aligned = kU8 && (reinterpret_cast<uintptr_t>(p.img) % 16 == 0) && (p.pitch % 16 == 0);
    const unsigned long long quads = (p.M + kQuad - 1) / kQuad;

    // Prefetch the first quad's tiles; later quads are prefetched under the SSD phase.
    if (kU8 && aligned) {
        const unsigned long long kp = static_cast<unsigned long long>(blockIdx.x) * kQuad + grp;
        if (blockIdx.x < quads && kp < p.M) {
            int ax0, ty0;
            tile_origin(__ldg(p.xycs + 4 * kp), __ldg(p.xycs + 4 * kp + 1), true, ax0, ty0);
            stage_tile_async(s_tile + grp * kQuadTileBytes, img8, p.pitch, p.height, ax0, ty0, gt);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }

    int buf = 0;
    for (unsigned long long quad = blockIdx.x; quad < quads; quad += gridDim.x, buf ^= 1) {
        const unsigned long long kp = quad * kQuad + grp;
        const bool valid = kp < p.M;
        double x = 0, y = 0, c = 0, s = 0;
        int ax0 = 0, ty0 = 0;
        uint8_t* const tile = s_tile + (buf * kQuad + grp) * kQuadTileBytes;
        if (valid) {
            x = __ldg(p.xycs + 4 * kp + 0);
            y = __ldg(p.xycs + 4 * kp + 1);
            c = __ldg(p.xycs + 4 * kp + 2);
            s = __ldg(p.xycs + 4 * kp + 3);
            if (kU8) {
                tile_origin(x, y, aligned, ax0, ty0);
                if (!aligned) stage_tile_u8<kThreads>(tile, img8, p.pitch, p.height, ax0, ty0, false, gt);
            }
            if (gt < kWindow) {   // per-row products of extract_window (src/descriptor.cpp:44-45)
                const double dv = static_cast<double>(gt) - 31.5;
                my_tab[gt] = __dmul_rn(s, dv);
                my_tab[kWindow + gt] = __dmul_rn(c, dv);
            }
        }
        if (kU8 && aligned) asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();   // tiles + tables ready; the previous quad's window / bit readers are done
        if (valid)
            build_window_tab<kU8>(s_win + grp * kQuadWinPitch, tile, ax0, ty0, static_cast<const double*>(p.img),
                                  p.pitch, x, y, c, s, my_tab, gt);
        __syncthreads();
        if (kU8 && aligned) {   // next quad's tiles stream in while the SSD phase runs
            const unsigned long long nq = quad + gridDim.x, nkp = nq * kQuad + grp;
            if (nq < quads && nkp < p.M) {
                int nax0, nty0;
                tile_origin(__ldg(p.xycs + 4 * nkp), __ldg(p.xycs + 4 * nkp + 1), true, nax0, nty0);
                stage_tile_async(s_tile + ((buf ^ 1) * kQuad + grp) * kQuadTileBytes, img8, p.pitch, p.height, nax0,
                                 nty0, gt);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        my_bits[slot0.w & 0x7fff] = triplet_bit_7x7(my_win, slot0.x, slot0.y, slot0.z, slot0.w >> 15);
        my_bits[slot1.w & 0x7fff] = triplet_bit_7x7(my_win, slot1.x, slot1.y, slot1.z, slot1.w >> 15);
        __syncthreads();
        const unsigned w0 = __ballot_sync(0xffffffffu, s_bits[grp * kFastT + gt] != 0);
        const unsigned w1 = __ballot_sync(0xffffffffu, s_bits[grp * kFastT + gt + kThreads] != 0);
        if ((tid & 31) == 0 && valid) {
            const unsigned long long row = p.out_index ? p.out_index[kp] : kp;
            unsigned* out32 = reinterpret_cast<unsigned*>(p.out + row * (kFastT / 8));
            out32[gt >> 5] = w0;
            out32[(gt >> 5) + kThreads / 32] = w1;
        }
    }
}

// ---- filtered kernel: fp32 estimate of every SSD pair, exact fp64 only where it is needed ----
// The reference's bit is sign(d1 - d2) of two 49-term fp64 sums; almost always |d1 - d2| is
// many orders of magnitude above anything rounding could change. So each window is kept as
// two 32-bit planes instead of one 64-bit one:
//   F  plane: f = cvt.rz.f32.f64(v)   (v truncated to 24 significant bits, 0 <= v - f < 2^-16)
//   LO plane: the low word of v
// and v is recovered exactly from the pair (hi word = (f >> 3) + 0x38000000 for f != 0: same
// exponent after re-biasing, f's top 20 mantissa bits; u8 images give 0 or 2^-106 <= v <= 255,
// always normal in fp32). The SSD phase reads ONLY the F plane — half the shared-memory
// wavefronts of the 64-bit window, fp32 FMAs instead of unfused fp64 — and proves its answer:
//   |d_ref - d_f| <= 14*2^-16*sqrt(d_f) + 49*2^-32   (truncated inputs, Cauchy-Schwarz over 49 terms)
//                    + 52*2^-24*d_f                   (fp32 subtraction + 49 fused accumulations)
//                    + 6e-15*d_f                      (the reference's own fp64 roundings)
// per chain; if |d1_f - d2_f| exceeds the sum of both chains' bounds (constants rounded up by
// >= 3 %) the sign is the reference's. Otherwise — exact ties in flat regions, or sums closer than
// ~2 parts in 10^5 — the lane recomputes both chains exactly from (F, LO) in the reference's order,
// with the same unfused fp64 arithmetic as the other kernels. The decision is never approximate.
//
// Lanes: warp = 8 triplets x 4 keypoints (lane = 4*i + w), plane w displaced by 8*w banks, so a
// 32-bit load is conflict-free when the 8 triplets differ mod 8 (plan_slots_grouped(8, 8)).
constexpr int kPlanePitch = 4168;                                    // words; 64 x 65 + 8; % 32 == 8
constexpr int kFiltSmemBytes = 2 * kQuad * kPlanePitch * 4           // F planes, LO planes
                               + 2 * kQuad * kQuadTileBytes          // double-buffered u8 tiles
                               + kQuad * kFastT                      // predicate bytes
                               + kQuad * 2 * kWindow * 8;            // s*dv, c*dv tables
constexpr int kLoPlane = kQuad * kPlanePitch;                        // word offset F plane -> LO plane

__device__ __forceinline__ void build_window_split(float* fpl, const uint8_t* tile, int ax0, int ty0, double x,
                                                   double y, double c, double s, const double* tab, int tid) {
    const int u = tid & 63;
    const double du = static_cast<double>(u) - 31.5;
    const double xa = __dadd_rn(x, __dmul_rn(c, du));
    const double ya = __dadd_rn(y, __dmul_rn(s, du));
#pragma unroll 4
    for (int v = tid >> 6; v < kWindow; v += kThreads / 64) {
        const double sx = __dsub_rn(xa, tab[v]);
        const double sy = __dadd_rn(ya, tab[kWindow + v]);
        int x0, y0;
        double x0f, y0f;
        floor_exact(sx, x0, x0f);
        floor_exact(sy, y0, y0f);
        const double fx = __dsub_rn(sx, x0f);
        const double fy = __dsub_rn(sy, y0f);
        const uint8_t* p = tile + (y0 - ty0) * kTileW + (x0 - ax0);
        const double val = blend(fx, fy, u8_to_f64(p[0]), u8_to_f64(p[1]), u8_to_f64(p[kTileW]),
                                 u8_to_f64(p[kTileW + 1]));
        fpl[v * kWinStride + u] = __double2float_rz(val);
        reinterpret_cast<int*>(fpl)[kLoPlane + v * kWinStride + u] = __double2loint(val);
    }
}

// fp32 estimate of both chains of two slots at once (four independent accumulators).
__device__ __forceinline__ void ssd_estimate_2(const float* win, const ushort4 s0, const ushort4 s1, float& d1a,
                                               float& d2a, float& d1b, float& d2b) {
    const float* pa0 = win + s0.x;
    const float* pb0 = win + s0.y;
    const float* pc0 = win + s0.z;
    const float* pa1 = win + s1.x;
    const float* pb1 = win + s1.y;
    const float* pc1 = win + s1.z;
    // Packed fp32x2 arithmetic (sm_100 FFMA2): component 0 = slot 0, component 1 = slot 1.
    // a - b is fma(b, -1, a): one rounding, the same value as a subtraction.
    const float2 neg1 = make_float2(-1.0f, -1.0f);
    float2 d1 = make_float2(0.0f, 0.0f), d2 = d1;
#pragma unroll
    for (int r = 0; r < 7; ++r) {
#pragma unroll
        for (int c = 0; c < 7; ++c) {
            const int o = r * kWinStride + c;
            const float2 a = make_float2(pa0[o], pa1[o]);
            const float2 e1 = __ffma2_rn(make_float2(pb0[o], pb1[o]), neg1, a);
            const float2 e2 = __ffma2_rn(make_float2(pc0[o], pc1[o]), neg1, a);
            d1 = __ffma2_rn(e1, e1, d1);
            d2 = __ffma2_rn(e2, e2, d2);
        }
    }
    d1a = d1.x;
    d1b = d1.y;
    d2a = d2.x;
    d2b = d2.y;
}

// True when sign(d1 - d2) of the fp32 estimate is provably the reference's (bound above).
__device__ __forceinline__ bool estimate_decides(float d1, float d2, float& diff) {
    float r1, r2;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d1));
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(d2));
    diff = d1 - d2;
    const float bound = __fmaf_rn(2.2e-4f, r1 + r2, __fmaf_rn(3.3e-6f, d1 + d2, 3.0e-8f));
    return fabsf(diff) > bound;
}

__device__ __forceinline__ double plane_value_at(const float* p, int lo_off) {
    const unsigned f = __float_as_uint(p[0]);
    const int lo = __float_as_int(p[lo_off]);
    const unsigned hi = f ? (f >> 3) + 0x38000000u : 0u;
    return __hiloint2double(static_cast<int>(hi), lo);
}

__device__ __forceinline__ double plane_value(const float* p) { return plane_value_at(p, kLoPlane); }

// The exact chains (same arithmetic and order as triplet_bit_7x7) from the split planes.
__device__ __noinline__ bool triplet_bit_7x7_planes(const float* win, int oa, int ob, int oc, bool swapped) {
    const float* pa = win + oa;
    const float* pb = win + ob;
    const float* pc = win + oc;
    double d1 = 0.0, d2 = 0.0;
#pragma unroll
    for (int r = 0; r < 7; ++r) {
#pragma unroll
        for (int c = 0; c < 7; ++c) {
            const int o = r * kWinStride + c;
            const double a = plane_value(pa + o);
            const double e1 = __dsub_rn(a, plane_value(pb + o));
            const double e2 = __dsub_rn(a, plane_value(pc + o));
            d1 = __dadd_rn(d1, __dmul_rn(e1, e1));
            d2 = __dadd_rn(d2, __dmul_rn(e2, e2));
        }
    }
    return swapped ? d2 > d1 : d1 > d2;
}

__global__ void __launch_bounds__(kQuadThreads, 1) extract_filt_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;

    extern __shared__ __align__(16) uint8_t s_quad[];
    float* const s_f = reinterpret_cast<float*>(s_quad);
    uint8_t* const s_tile = s_quad + 2 * kQuad * kPlanePitch * 4;
    uint8_t* const s_bits = s_tile + 2 * kQuad * kQuadTileBytes;
    double* const s_tab = reinterpret_cast<double*>(s_bits + kQuad * kFastT);

    const int tid = threadIdx.x;
    const int grp = tid >> 8, gt = tid & (kThreads - 1);         // staging / resampling: group -> keypoint
    const int warp = tid >> 5, lane = tid & 31, kb = lane & 3, ti = lane >> 2;   // SSD: 8 triplets x 4 keypoints
    const ushort4 slot0 = __ldg(p.slots + 8 * warp + ti);
    const ushort4 slot1 = __ldg(p.slots + 8 * warp + ti + kFastT / 2);
    const float* const my_win = s_f + kb * kPlanePitch;
    uint8_t* const my_bits = s_bits + kb * kFastT;
    double* const my_tab = s_tab + grp * 2 * kWindow;
    const uint8_t* const img8 = static_cast<const uint8_t*>(p.img);
    const bool aligned = (reinterpret_cast<uintptr_t>(p.img) % 16 == 0) && (p.pitch % 16 == 0);
    const unsigned long long quads = (p.M + kQuad - 1) / kQuad;
    unsigned n_flagged = 0, n_warps = 0;

    if (aligned) {
        const unsigned long long kp = static_cast<unsigned long long>(blockIdx.x) * kQuad + grp;
        if (blockIdx.x < quads && kp < p.M) {
            int ax0, ty0;
            tile_origin(__ldg(p.xycs + 4 * kp), __ldg(p.xycs + 4 * kp + 1), true, ax0, ty0);
            stage_tile_async(s_tile + grp * kQuadTileBytes, img8, p.pitch, p.height, ax0, ty0, gt);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }

    int buf = 0;
    for (unsigned long long quad = blockIdx.x; quad < quads; quad += gridDim.x, buf ^= 1) {
        const unsigned long long kp = quad * kQuad + grp;
        const bool valid = kp < p.M;
        double x = 0, y = 0, c = 0, s = 0;
        int ax0 = 0, ty0 = 0;
        uint8_t* const tile = s_tile + (buf * kQuad + grp) * kQuadTileBytes;
        if (valid) {
            x = __ldg(p.xycs + 4 * kp + 0);
            y = __ldg(p.xycs + 4 * kp + 1);
            c = __ldg(p.xycs + 4 * kp + 2);
            s = __ldg(p.xycs + 4 * kp + 3);
            tile_origin(x, y, aligned, ax0, ty0);
            if (!aligned) stage_tile_u8<kThreads>(tile, img8, p.pitch, p.height, ax0, ty0, false, gt);
            if (gt < kWindow) {   // per-row products of extract_window (src/descriptor.cpp:44-45)
                const double dv = static_cast<double>(gt) - 31.5;
                my_tab[gt] = __dmul_rn(s, dv);
                my_tab[kWindow + gt] = __dmul_rn(c, dv);
            }
        }
        if (aligned) asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();   // tiles + tables ready; the previous quad's plane / bit readers are done
        if (valid) build_window_split(s_f + grp * kPlanePitch, tile, ax0, ty0, x, y, c, s, my_tab, gt);
        __syncthreads();
        if (aligned) {     // next quad's tiles stream in while the SSD phase runs
            const unsigned long long nq = quad + gridDim.x, nkp = nq * kQuad + grp;
            if (nq < quads && nkp < p.M) {
                int nax0, nty0;
                tile_origin(__ldg(p.xycs + 4 * nkp), __ldg(p.xycs + 4 * nkp + 1), true, nax0, nty0);
                stage_tile_async(s_tile + ((buf ^ 1) * kQuad + grp) * kQuadTileBytes, img8, p.pitch, p.height, nax0,
                                 nty0, gt);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        float d1a, d2a, d1b, d2b, diff0, diff1;
        ssd_estimate_2(my_win, slot0, slot1, d1a, d2a, d1b, d2b);
        const bool sure0 = estimate_decides(d1a, d2a, diff0);
        const bool sure1 = estimate_decides(d1b, d2b, diff1);
        bool bit0 = (slot0.w >> 15) ? diff0 < 0.0f : diff0 > 0.0f;
        bool bit1 = (slot1.w >> 15) ? diff1 < 0.0f : diff1 > 0.0f;
        // A keypoint past the end of the list leaves a stale window: never worth an exact pass.
        const bool live = quad * kQuad + kb < p.M;
        const unsigned undecided = __ballot_sync(0xffffffffu, live && !(sure0 && sure1));
        if (undecided) {
            if (live && !sure0) bit0 = triplet_bit_7x7_planes(my_win, slot0.x, slot0.y, slot0.z, slot0.w >> 15);
            if (live && !sure1) bit1 = triplet_bit_7x7_planes(my_win, slot1.x, slot1.y, slot1.z, slot1.w >> 15);
            n_flagged += (live && !sure0) + (live && !sure1);
            n_warps += lane == 0;
        }
        my_bits[slot0.w & 0x7fff] = bit0;
        my_bits[slot1.w & 0x7fff] = bit1;
        __syncthreads();
        const unsigned w0 = __ballot_sync(0xffffffffu, s_bits[grp * kFastT + gt] != 0);
        const unsigned w1 = __ballot_sync(0xffffffffu, s_bits[grp * kFastT + gt + kThreads] != 0);
        if ((tid & 31) == 0 && valid) {
            unsigned* out32 = reinterpret_cast<unsigned*>(p.out + kp * (kFastT / 8));
            out32[gt >> 5] = w0;
            out32[(gt >> 5) + kThreads / 32] = w1;
        }
    }
    if (p.stats != nullptr) {   // exact-pass counters (diagnostics; off unless asked for)
        n_flagged = __reduce_add_sync(0xffffffffu, n_flagged);
        if (lane == 0 && (n_flagged | n_warps)) {
            atomicAdd(p.stats + 0, static_cast<unsigned long long>(n_flagged));
            atomicAdd(p.stats + 1, static_cast<unsigned long long>(n_warps));
        }
    }
}

// ---- pipelined kernel: resampling and SSD run side by side ----------------------------------
// The filtered kernel alternates two phases that starve each other's pipes: resampling is
// fp64-bound (LSU half idle), the SSD estimate is LSU-bound (fp64 idle). Here the F planes are
// double-buffered and the two phases of consecutive quads overlap: in iteration `it` every
// thread resamples its 16 samples of quad it+1 into F[next] AND estimates its 2 triplet slots
// of quad it from F[cur] — half of the warps (two per SM sub-partition and parity) in that
// order, the other half in the opposite order, so at any moment about half of the SM is on
// the fp64 pipe and half on the LSU, with equal work per warp by construction and a single
// __syncthreads per quad. Footprints come from the texture unit (tex2Dgather on a u8 CUDA
// array: the four texels of a bilinear footprint in one instruction — no tile staging, no LSU
// traffic), software-pipelined four samples deep so the gather latency hides behind the warp's
// own fp64 work. Eight F planes and four LO planes fit in shared memory (200 KB) because LO
// planes are no longer written up front: when some lane could not decide a bit, the whole CTA
// re-resamples just that window's LO plane after the barrier (same exact arithmetic, same
// texels) and the undecided lanes run the exact chains as in the filtered kernel. On textured
// images that happens for ~1 % of the windows.
constexpr int kPipePlanes = 12;                                      // F[2][4] + LO[4]
constexpr int kPipeRows = kQuadThreads / kWindow;                    // 16: thread -> rows v0 + 16k
constexpr int kPipePer = kWindow / kPipeRows;                        // 4 samples per thread per window
constexpr int kPipeBits = kFastT + 16;   // predicate bytes per window; +4 banks so the 4 lanes of a triplet differ
constexpr int kPipeSmemBytes = kPipePlanes * kPlanePitch * 4         // planes
                               + 2 * kQuad * kPipeBits               // predicate bytes [2][4][512 + pad]
                               + 2 * kQuad * kWindow * 16            // {s*dv, c*dv} rows [2][4][64]
                               + 2 * kQuad * 4 * 8                   // keypoint records [2][4][4]
                               + 64;                                 // undecided-window masks [3], deferred-queue tail
// Deferred exact bits (roles kernel): undecided (keypoint, triplet) items parked in shared memory and recomputed by
// whole warps after the pipeline has drained, instead of stalling it (see extract_roles_kernel).
constexpr int kQueueCap = 1024;          // items per CTA
constexpr int kDeferMax = 48;            // a quad with more undecided triplets than this takes the window-wide pass
struct DeferredBit {
    ushort4 slot;                        // {a, b, c, bit | swapped << 15} as in the slot table
    unsigned kp;                         // keypoint record index
};
constexpr int kRolesSmemBytes = kPipeSmemBytes + kQueueCap * static_cast<int>(sizeof(DeferredBit));

// The 2x2 footprint whose top-left texel is (x0, y0): gather at the footprint's centre, half a
// texel away from every selection boundary (tools/tex_probe.cu checks the component order):
// w = (x0,y0), z = (x0+1,y0), x = (x0,y0+1), y = (x0+1,y0+1).
__device__ __forceinline__ uint4 footprint(cudaTextureObject_t tex, int x0, int y0) {
    // (2^23 + x0) - (2^23 - 1) = x0 + 1 exactly, without an integer->float conversion
    const float fx = __uint_as_float(0x4B000000u | static_cast<unsigned>(x0)) - 8388607.0f;
    const float fy = __uint_as_float(0x4B000000u | static_cast<unsigned>(y0)) - 8388607.0f;
    return tex2Dgather<uint4>(tex, fx, fy, 0);   // u8 texels arrive zero-extended: no masking
}

// One window sample, exactly as extract_window / sample_bilinear compute it.
__device__ __forceinline__ double sample_exact(cudaTextureObject_t tex, double xa, double ya, double sdv,
                                               double cdv) {
    const double sx = __dsub_rn(xa, sdv);
    const double sy = __dadd_rn(ya, cdv);
    int x0, y0;
    double x0f, y0f;
    floor_exact(sx, x0, x0f);
    floor_exact(sy, y0, y0f);
    const double fx = __dsub_rn(sx, x0f);
    const double fy = __dsub_rn(sy, y0f);
    const uint4 g = footprint(tex, x0, y0);
    return blend(fx, fy, u8_to_f64(g.w), u8_to_f64(g.z), u8_to_f64(g.x), u8_to_f64(g.y));
}

// The same sample from a float64 image in global memory (what extract_quad_kernel<false> computes).
__device__ __forceinline__ double sample_exact_f64(const double* img, size_t pitch, double xa, double ya, double sdv, double cdv) {
    const double sx = __dsub_rn(xa, sdv);
    const double sy = __dadd_rn(ya, cdv);
    int x0, y0;
    double x0f, y0f;
    floor_exact(sx, x0, x0f);
    floor_exact(sy, y0, y0f);
    const double fx = __dsub_rn(sx, x0f);
    const double fy = __dsub_rn(sy, y0f);
    const double* q = img + static_cast<size_t>(y0) * pitch + x0;
    return blend(fx, fy, __ldg(q), __ldg(q + 1), __ldg(q + pitch), __ldg(q + pitch + 1));
}

__device__ __noinline__ bool triplet_bit_7x7_planes_at(const float* win, int lo_off, int oa, int ob, int oc,
                                                       bool swapped) {
    const float* pa = win + oa;
    const float* pb = win + ob;
    const float* pc = win + oc;
    double d1 = 0.0, d2 = 0.0;
#pragma unroll
    for (int r = 0; r < 7; ++r) {
#pragma unroll
        for (int c = 0; c < 7; ++c) {
            const int o = r * kWinStride + c;
            const double a = plane_value_at(pa + o, lo_off);
            const double e1 = __dsub_rn(a, plane_value_at(pb + o, lo_off));
            const double e2 = __dsub_rn(a, plane_value_at(pc + o, lo_off));
            d1 = __dadd_rn(d1, __dmul_rn(e1, e1));
            d2 = __dadd_rn(d2, __dmul_rn(e2, e2));
        }
    }
    return swapped ? d2 > d1 : d1 > d2;
}

// One quad iteration of one thread, resampling half: its 16 samples of the next quad (4 windows x 4
// rows) into F[next]. Four gathers stay in flight: the gather of sample i + 4 is issued before sample
// i is blended, so the texture latency hides behind the warp's own fp64 work.
// (Interleaving this stream with the estimate's loads and FMAs in one straight-line block was
// measured slower than phase-staggered warps: an LSU queue stall then also blocks the fp64 chain.)
struct PipeStep {
    cudaTextureObject_t tex;
    const double2* tab;   // {s*dv, c*dv} rows of the next quad, already offset by this thread's v0
    const double* kpr;    // keypoint records of the next quad
    float* fbase;         // F[next] + this thread's (v0, u)
    double du;
};

__device__ __forceinline__ void resample_step(const PipeStep& st) {
    constexpr int kDepth = 4, kTotal = kQuad * kPipePer;
    double pfx[kDepth], pfy[kDepth], xa = 0.0, ya = 0.0;
    uint4 pg[kDepth];
#pragma unroll
    for (int i = 0; i < kTotal + kDepth; ++i) {
        if (i >= kDepth) {
            const int j = i - kDepth, sl = j % kDepth;
            const uint4 g = pg[sl];
            const double val = blend(pfx[sl], pfy[sl], u8_to_f64(g.w), u8_to_f64(g.z), u8_to_f64(g.x),
                                     u8_to_f64(g.y));
            st.fbase[(j / kPipePer) * kPlanePitch + (j % kPipePer) * kPipeRows * kWinStride] = __double2float_rz(val);
        }
        if (i < kTotal) {
            const int w = i / kPipePer, sl = i % kDepth;
            if (i % kPipePer == 0) {
                xa = __dadd_rn(st.kpr[4 * w + 0], __dmul_rn(st.kpr[4 * w + 2], st.du));
                ya = __dadd_rn(st.kpr[4 * w + 1], __dmul_rn(st.kpr[4 * w + 3], st.du));
            }
            const double2 row = st.tab[w * kWindow + (i % kPipePer) * kPipeRows];   // {s*dv, c*dv}
            const double sx = __dsub_rn(xa, row.x);
            const double sy = __dadd_rn(ya, row.y);
            int x0, y0;
            double x0f, y0f;
            floor_exact(sx, x0, x0f);
            floor_exact(sy, y0, y0f);
            pfx[sl] = __dsub_rn(sx, x0f);
            pfy[sl] = __dsub_rn(sy, y0f);
            pg[sl] = footprint(st.tex, x0, y0);
        }
    }
}

// Keypoint records and per-row products {s*dv, c*dv} of extract_window (src/descriptor.cpp:44-45)
// for the four windows of the quad that starts at keypoint kp0, by threads 0..255. A keypoint past
// the end repeats the last one (its window is computed and never used).
__device__ __forceinline__ void stage_quad_rows(const ExtractParams& p, unsigned long long kp0, double2* tab,
                                                double* kpr, int tid) {
    if (tid < kQuad * kWindow) {
        const int w = tid >> 6, row = tid & 63;
        const unsigned long long kp = min(kp0 + w, p.M - 1);
        const double c = __ldg(p.xycs + 4 * kp + 2), sn = __ldg(p.xycs + 4 * kp + 3);
        const double dv = static_cast<double>(row) - 31.5;
        tab[tid] = make_double2(__dmul_rn(sn, dv), __dmul_rn(c, dv));
        if (row < 4) kpr[4 * w + row] = __ldg(p.xycs + 4 * kp + row);
    }
}

__global__ void __launch_bounds__(kQuadThreads, 1) extract_pipe_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;

    extern __shared__ __align__(16) uint8_t s_quad[];
    float* const s_f = reinterpret_cast<float*>(s_quad);                              // F[2][4], then LO[4]
    uint8_t* const s_bits = s_quad + kPipePlanes * kPlanePitch * 4;                   // [2][4][512]
    double2* const s_tab = reinterpret_cast<double2*>(s_bits + 2 * kQuad * kPipeBits);   // [2][4][64]
    double* const s_kp = reinterpret_cast<double*>(s_tab + 2 * kQuad * kWindow);      // [2][4][x, y, cos, sin]
    int* const s_mask = reinterpret_cast<int*>(s_kp + 2 * kQuad * 4);                 // [3] windows needing LO

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool ssd_first = (warp >> 2) & 1;                  // per sub-partition: 4 warps each way
    const int u = tid & 63, v0 = tid >> 6;                   // resampling: column u, rows v0 + 16k
    const double du = static_cast<double>(u) - 31.5;
    const int kb = lane & 3, ti = lane >> 2;                 // SSD: 8 triplets x 4 keypoints per warp
    const ushort4 slot0 = __ldg(p.slots + 8 * warp + ti);
    const ushort4 slot1 = __ldg(p.slots + 8 * warp + ti + kFastT / 2);
    const unsigned long long quads = (p.M + kQuad - 1) / kQuad;
    const long long nq = blockIdx.x < quads ? static_cast<long long>((quads - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
    unsigned n_flagged = 0, n_windows = 0;
    if (tid < 3) s_mask[tid] = 0;
    stage_quad_rows(p, static_cast<unsigned long long>(blockIdx.x) * kQuad, s_tab, s_kp, tid);
    __syncthreads();

    for (long long it = -1; it <= nq; ++it) {
        const int cur = static_cast<int>(it & 1), nxt = cur ^ 1;
        const int mslot = static_cast<int>((it + 3) % 3);
        const unsigned long long kp0 = (blockIdx.x + it * gridDim.x) * kQuad;   // quad `it` (when it >= 0)
        const bool consume = it >= 0 && it < nq, produce = it + 1 < nq;
        if (tid == 0) s_mask[(mslot + 1) % 3] = 0;           // quad it-2's mask: every reader is past it
        if (it + 2 < nq)                                      // rows for quad it+2 -> buffer [cur]
            stage_quad_rows(p, (blockIdx.x + (it + 2) * gridDim.x) * kQuad, s_tab + cur * kQuad * kWindow,
                            s_kp + cur * kQuad * 4, tid);
        if (it >= 1) {   // pack the bits of quad it-1 (buffer [nxt])
            const unsigned long long kp = (blockIdx.x + (it - 1) * gridDim.x) * kQuad + (tid >> 8);
            const uint8_t* bits = s_bits + (nxt * kQuad + (tid >> 8)) * kPipeBits;
            const int j = tid & 255;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const unsigned w32 = __ballot_sync(0xffffffffu, bits[256 * k + j] != 0);
                if (lane == 0 && kp < p.M) {
                    const unsigned long long row = p.out_index ? p.out_index[kp] : kp;
                    reinterpret_cast<unsigned*>(p.out + row * (kFastT / 8))[8 * k + (j >> 5)] = w32;
                }
            }
        }

        const float* const my_win = s_f + (cur * kQuad + kb) * kPlanePitch;
        unsigned need = 0;
        {
            PipeStep st;
            st.tex = p.tex;
            st.tab = s_tab + nxt * kQuad * kWindow + v0;
            st.kpr = s_kp + nxt * kQuad * 4;
            st.fbase = s_f + nxt * kQuad * kPlanePitch + v0 * kWinStride + u;
            st.du = du;
            float d1a = 0.f, d2a = 0.f, d1b = 0.f, d2b = 0.f;
            // Half of the warps (four per SM sub-partition) estimate first and resample second, the
            // other half the other way round: at any moment about half of the SM is on the LSU and
            // half on the fp64 pipe, with equal work per warp by construction.
#pragma unroll 1
            for (int phase = 0; phase < 2; ++phase) {
                if ((phase == 0) == ssd_first) {
                    if (consume) ssd_estimate_2(my_win, slot0, slot1, d1a, d2a, d1b, d2b);
                } else if (produce) {
                    resample_step(st);
                }
            }
            if (consume) {
                float diff0, diff1;
                const bool sure0 = estimate_decides(d1a, d2a, diff0);
                const bool sure1 = estimate_decides(d1b, d2b, diff1);
                const bool live = kp0 + kb < p.M;   // a keypoint past the end leaves an unused window
                need = (live && !sure0 ? 1u : 0u) | (live && !sure1 ? 2u : 0u);
                if (need) atomicOr(s_mask + mslot, 1 << kb);
                uint8_t* const my_bits = s_bits + (cur * kQuad + kb) * kPipeBits;
                my_bits[slot0.w & 0x7fff] = (slot0.w >> 15) ? diff0 < 0.0f : diff0 > 0.0f;
                my_bits[slot1.w & 0x7fff] = (slot1.w >> 15) ? diff1 < 0.0f : diff1 > 0.0f;
            }
        }
        __syncthreads();

        if (consume) {
            const int mask = *reinterpret_cast<volatile int*>(s_mask + mslot);
            if (mask) {   // block-uniform: some lane could not decide -> exact pass for those windows
                for (int w = 0; w < kQuad; ++w) {
                    if (!((mask >> w) & 1)) continue;
                    const double* const kpr = p.xycs + 4 * (kp0 + w);   // (the staged copy is already quad it+2's)
                    const double c = __ldg(kpr + 2), sn = __ldg(kpr + 3);
                    const double xa = __dadd_rn(__ldg(kpr + 0), __dmul_rn(c, du));
                    const double ya = __dadd_rn(__ldg(kpr + 1), __dmul_rn(sn, du));
                    int* lopl = reinterpret_cast<int*>(s_f) + (2 * kQuad + w) * kPlanePitch + u;
#pragma unroll 2
                    for (int v = v0; v < kWindow; v += kPipeRows) {
                        const double dv = static_cast<double>(v) - 31.5;
                        lopl[v * kWinStride] =
                            __double2loint(sample_exact(p.tex, xa, ya, __dmul_rn(sn, dv), __dmul_rn(c, dv)));
                    }
                    n_windows += tid == 0;
                }
                __syncthreads();
                const int lo_off = (2 - cur) * kQuad * kPlanePitch;          // F[cur][kb] -> LO[kb]
                uint8_t* const my_bits = s_bits + (cur * kQuad + kb) * kPipeBits;
                if (need & 1) {
                    my_bits[slot0.w & 0x7fff] =
                        triplet_bit_7x7_planes_at(my_win, lo_off, slot0.x, slot0.y, slot0.z, slot0.w >> 15);
                    ++n_flagged;
                }
                if (need & 2) {
                    my_bits[slot1.w & 0x7fff] =
                        triplet_bit_7x7_planes_at(my_win, lo_off, slot1.x, slot1.y, slot1.z, slot1.w >> 15);
                    ++n_flagged;
                }
                __syncthreads();   // the next iteration packs these bits
            }
        }
    }
    if (p.stats != nullptr) {   // exact-pass counters (diagnostics; off unless asked for)
        n_flagged = __reduce_add_sync(0xffffffffu, n_flagged);
        if (lane == 0 && (n_flagged | n_windows)) {
            atomicAdd(p.stats + 0, static_cast<unsigned long long>(n_flagged));
            atomicAdd(p.stats + 1, static_cast<unsigned long long>(n_windows));
        }
    }
}

// One deferred bit, by one warp: the 3 x 49 live samples of the triplet's patches are resampled exactly as
// extract_window / sample_bilinear compute them (the same code as the window-wide pass: sample_exact) into
// `scratch` (147 doubles), lanes 0 and 1 run the two 49-term chains in the reference's row-major order, and the
// descriptor word is patched in global memory (the estimate's guess was stored there by this CTA earlier).
// Patch anchor (column, row) of a packed-plane slot offset (slot_assign.hpp: h16_offset).
__device__ __forceinline__ void h16_anchor_dev(unsigned off, int& x, int& y) {
    const int odd = off >= static_cast<unsigned>(kH16CopyWords);
    const int r = static_cast<int>(off) - odd * kH16CopyWords;
    y = r / kH16RowWords;
    x = 2 * (r - y * kH16RowWords) - odd;
}

// kH16: slot offsets are packed-plane word offsets (else row * kWinStride + column, the fp32 planes).
// kF64: the image is float64 in global memory (img64 / pitch64) instead of the u8 texture.
template <bool kH16, bool kF64 = false>
__device__ __noinline__ void recompute_deferred_bit(cudaTextureObject_t tex, const double* xycs, uint8_t* out,
                                                    const unsigned* out_index, const DeferredBit item, double* scratch,
                                                    int lane, const double* img64 = nullptr, size_t pitch64 = 0) {
    const double* const kpr = xycs + 4 * static_cast<unsigned long long>(item.kp);
    const double kx = __ldg(kpr + 0), ky = __ldg(kpr + 1), c = __ldg(kpr + 2), sn = __ldg(kpr + 3);
    const unsigned offs[3] = {item.slot.x, item.slot.y, item.slot.z};
    if (kF64) {
#pragma unroll 1
        for (int i = lane; i < 3 * 49; i += 32) {
            const int patch = i / 49, pix = i - 49 * patch, r = pix / 7, cc = pix - 7 * r;
            const unsigned off = patch == 0 ? offs[0] : (patch == 1 ? offs[1] : offs[2]);
            int v, u;
            h16_anchor_dev(off, u, v);
            const double du = static_cast<double>(u + cc) - 31.5, dv = static_cast<double>(v + r) - 31.5;
            scratch[i] = sample_exact_f64(img64, pitch64, __dadd_rn(kx, __dmul_rn(c, du)), __dadd_rn(ky, __dmul_rn(sn, du)),
                                          __dmul_rn(sn, dv), __dmul_rn(c, dv));
        }
    }
    // Five rounds of 32 samples: all footprints are requested before the first one is blended (issued one by one, each
    // gather's ~700 clk of latency — nothing else runs on the SM at this point — was paid five times in a row).
    double pfx[5], pfy[5];
    uint4 pg[5];
#pragma unroll
    for (int round = 0; round < (kF64 ? 0 : 5); ++round) {
        const int i = min(lane + 32 * round, 3 * 49 - 1);
        const int patch = i / 49, pix = i - 49 * patch, r = pix / 7, cc = pix - 7 * r;
        const unsigned off = patch == 0 ? offs[0] : (patch == 1 ? offs[1] : offs[2]);
        int v, u;
        if (kH16) {
            h16_anchor_dev(off, u, v);
            v += r;
            u += cc;
        } else {
            v = static_cast<int>(off / kWinStride) + r;
            u = static_cast<int>(off % kWinStride) + cc;
        }
        const double du = static_cast<double>(u) - 31.5, dv = static_cast<double>(v) - 31.5;
        const double sx = __dsub_rn(__dadd_rn(kx, __dmul_rn(c, du)), __dmul_rn(sn, dv));   // as sample_exact
        const double sy = __dadd_rn(__dadd_rn(ky, __dmul_rn(sn, du)), __dmul_rn(c, dv));
        int x0, y0;
        double x0f, y0f;
        floor_exact(sx, x0, x0f);
        floor_exact(sy, y0, y0f);
        pfx[round] = __dsub_rn(sx, x0f);
        pfy[round] = __dsub_rn(sy, y0f);
        pg[round] = footprint(tex, x0, y0);
    }
#pragma unroll
    for (int round = 0; round < (kF64 ? 0 : 5); ++round) {
        const int i = lane + 32 * round;
        const uint4 g = pg[round];
        const double val = blend(pfx[round], pfy[round], u8_to_f64(g.w), u8_to_f64(g.z), u8_to_f64(g.x), u8_to_f64(g.y));
        if (i < 3 * 49) scratch[i] = val;
    }
    __syncwarp();
    double d = 0.0;
    if (lane < 2) {
        const double* const other = scratch + 49 * (1 + lane);
#pragma unroll 7
        for (int k = 0; k < 49; ++k) {
            const double e = __dsub_rn(scratch[k], other[k]);
            d = __dadd_rn(d, __dmul_rn(e, e));
        }
    }
    const double d2 = __shfl_sync(0xffffffffu, d, 1);
    if (lane == 0) {
        const bool bit = (item.slot.w >> 15) ? d2 > d : d > d2;
        const unsigned t = item.slot.w & 0x7fffu;
        const unsigned long long row = out_index ? out_index[item.kp] : item.kp;
        unsigned* const word = reinterpret_cast<unsigned*>(out + row * (kFastT / 8)) + (t >> 5);
        if (bit) atomicOr(word, 1u << (t & 31));
        else atomicAnd(word, ~(1u << (t & 31)));
    }
    __syncwarp();
}

// ---- role-split variant of the pipelined kernel (A/B) -----------------------------------------
// Same planes, same texture path, same estimate and exact code as extract_pipe_kernel, but the
// warps specialise: kRW producer warps only resample (quad it+1 -> F[next]) and pack bits, the
// other 32 - kRW consumer warps only estimate (quad it from F[cur]) and own the exact pass. The
// LSU then sees a steady stream from the consumers instead of bursts from whichever half of the
// SM is in its estimate phase. Roles are spread evenly over the four SM sub-partitions.
template <int kRW>
__global__ void __launch_bounds__(kQuadThreads, 1) extract_roles_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;
    constexpr int kSW = 32 - kRW, kRT = kRW * 32, kST = kSW * 32;
    constexpr int kStep = 32 / kSW;                          // every kStep-th group of 4 warps consumes
    constexpr int kRRows = kRT / kWindow;                    // producer thread -> rows v0 + kRRows * k
    constexpr int kRPer = (kWindow + kRRows - 1) / kRRows;   // samples per producer thread per window (max)
    constexpr int kSRows = kST / kWindow;                    // exact pass: consumer thread -> rows v0 + kSRows * k
    constexpr int kSlots = 64 / kSW;                         // groups of 8 triplets per consumer warp
    static_assert(32 % kSW == 0 && 64 % kSW == 0 && kSlots % 2 == 0 && kRT >= 512, "role split");

    extern __shared__ __align__(16) uint8_t s_quad[];
    float* const s_f = reinterpret_cast<float*>(s_quad);                              // F[2][4], then LO[4]
    uint8_t* const s_bits = s_quad + kPipePlanes * kPlanePitch * 4;                   // [2][4][512 + pad]
    double2* const s_tab = reinterpret_cast<double2*>(s_bits + 2 * kQuad * kPipeBits);   // [2][4][64]
    double* const s_kp = reinterpret_cast<double*>(s_tab + 2 * kQuad * kWindow);      // [2][4][x, y, cos, sin]
    int* const s_mask = reinterpret_cast<int*>(s_kp + 2 * kQuad * 4);                 // [2] windows needing LO
    unsigned* const s_qtail = reinterpret_cast<unsigned*>(s_mask + 2);                // deferred bits queued so far
    DeferredBit* const s_queue = reinterpret_cast<DeferredBit*>(s_quad + kPipeSmemBytes);   // [kQueueCap]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, grp = warp >> 2;
    const bool producer = grp % kStep != 0;
    const int rw = (producer ? grp - grp / kStep - 1 : grp / kStep) * 4 + (warp & 3);   // role-local warp
    const int rt = rw * 32 + lane;                                                       // role-local thread
    const int u = rt & 63, v0 = rt >> 6;
    const double du = static_cast<double>(u) - 31.5;
    const int kb = lane & 3, ti = lane >> 2;
    const unsigned long long quads = (p.M + kQuad - 1) / kQuad;
    const long long nq = blockIdx.x < quads ? static_cast<long long>((quads - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
    ushort4 slot[kSlots];
#pragma unroll
    for (int j = 0; j < kSlots; ++j) slot[j] = __ldg(p.slots + 8 * (rw % kSW + kSW * j) + ti);
    unsigned n_flagged = 0, n_windows = 0;
    unsigned long long* const trace = p.trace != nullptr && tid == 0 ? p.trace + static_cast<size_t>(kExTrace) * blockIdx.x : nullptr;
    if (trace) trace[0] = ex_global_ns();
    if (tid == 0) s_mask[0] = s_mask[1] = 0, *s_qtail = 0;
    // Undecided bits are rare on textured images (2e-5 of the triplets on noise), but the window-wide exact pass
    // below stalls the whole CTA for ~4 us each time (one quad in 25 at that rate; the slowest CTA of a 10 k
    // launch took four). So a quad with few of them only PARKS them — {slot, keypoint} in a shared-memory queue —
    // and carries on with the estimate's guess in the descriptor; after the pipeline has drained every warp of
    // the CTA takes parked items and recomputes each bit exactly (recompute_deferred_bit). Dense quads (flat or
    // saturated regions: more than kDeferMax undecided triplets, or a full queue) take the window-wide pass as
    // before. Either way the bit that ends up in the descriptor comes from the exact fp64 chains.
    const bool defer_ok = p.M <= 0xffffffffull;
    unsigned q_prev = 0;                 // queue tail after the previous quad (uniform over the consumers)
    // Producers only resample. The consumers, which have slack, also stage the keypoint records and
    // row products two quads ahead (buffer [quad & 1]) and pack the previous quad's bits.
    stage_quad_rows(p, static_cast<unsigned long long>(blockIdx.x) * kQuad, s_tab, s_kp, tid);
    __syncthreads();
    pdl_wait();   // launched early behind fill_array_kernel: the texture array is complete from here on
    if (trace) trace[1] = ex_global_ns();

    for (long long it = -1; it <= nq; ++it) {
        const int cur = static_cast<int>(it & 1), nxt = cur ^ 1;
        unsigned windows_before = n_windows;
        if (!producer) {
            if (it + 2 < nq)   // rows for quad it+2 -> buffer [cur] (its last readers resampled quad `it`, an iteration ago)
                stage_quad_rows(p, (blockIdx.x + (it + 2) * gridDim.x) * kQuad, s_tab + cur * kQuad * kWindow,
                                s_kp + cur * kQuad * 4, rt);
            if (it >= 1) {   // pack the bits of the quad consumed in the previous iteration
                const unsigned long long kp = (blockIdx.x + (it - 1) * gridDim.x) * kQuad + (rt >> 7);
                const uint8_t* bits = s_bits + (nxt * kQuad + (rt >> 7)) * kPipeBits;
                const int j = rt & 127;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const unsigned w32 = __ballot_sync(0xffffffffu, bits[128 * k + j] != 0);
                    if (lane == 0 && kp < p.M) {
                        const unsigned long long row = p.out_index ? p.out_index[kp] : kp;
                        reinterpret_cast<unsigned*>(p.out + row * (kFastT / 8))[4 * k + (j >> 5)] = w32;
                    }
                }
            }
        }
        if (producer) {
            if (it + 1 < nq) {   // resample the next quad into F[nxt]
                const double2* const tab = s_tab + nxt * kQuad * kWindow;
                const double* const kpr = s_kp + nxt * kQuad * 4;
                constexpr int kDepth = 4, kTotal = kQuad * kRPer;
                double pfx[kDepth], pfy[kDepth], xa = 0.0, ya = 0.0;
                uint4 pg[kDepth];
                float* const fbase = s_f + nxt * kQuad * kPlanePitch + v0 * kWinStride + u;
#pragma unroll
                for (int i = 0; i < kTotal + kDepth; ++i) {
                    if (i >= kDepth) {
                        const int j = i - kDepth, sl = j % kDepth;
                        if (v0 + (j % kRPer) * kRRows < kWindow) {      // warp-uniform
                            const uint4 g = pg[sl];
                            const double val = blend(pfx[sl], pfy[sl], u8_to_f64(g.w), u8_to_f64(g.z), u8_to_f64(g.x),
                                                     u8_to_f64(g.y));
                            fbase[(j / kRPer) * kPlanePitch + (j % kRPer) * kRRows * kWinStride] =
                                __double2float_rz(val);
                        }
                    }
                    if (i < kTotal) {
                        const int w = i / kRPer, sl = i % kDepth;
                        if (i % kRPer == 0) {
                            xa = __dadd_rn(kpr[4 * w + 0], __dmul_rn(kpr[4 * w + 2], du));
                            ya = __dadd_rn(kpr[4 * w + 1], __dmul_rn(kpr[4 * w + 3], du));
                        }
                        const int v = v0 + (i % kRPer) * kRRows;
                        if (v < kWindow) {                               // warp-uniform
                            const double2 row = tab[w * kWindow + v];   // {s*dv, c*dv}
                            const double sx = __dsub_rn(xa, row.x);
                            const double sy = __dadd_rn(ya, row.y);
                            int x0, y0;
                            double x0f, y0f;
                            floor_exact(sx, x0, x0f);
                            floor_exact(sy, y0, y0f);
                            pfx[sl] = __dsub_rn(sx, x0f);
                            pfy[sl] = __dsub_rn(sy, y0f);
                            pg[sl] = footprint(p.tex, x0, y0);
                        }
                    }
                }
            }
        } else if (it >= 0 && it < nq) {
            const unsigned long long kp0 = (blockIdx.x + it * gridDim.x) * kQuad;
            const float* const my_win = s_f + (cur * kQuad + kb) * kPlanePitch;
            const int lo_off = (2 - cur) * kQuad * kPlanePitch;          // F[cur][kb] -> LO[kb]
            const bool live = kp0 + kb < p.M;   // a keypoint past the end leaves an unused window
            if (rt == 0) s_mask[nxt] = 0;
            uint8_t* const my_bits = s_bits + (cur * kQuad + kb) * kPipeBits;
            unsigned need = 0;
#pragma unroll
            for (int j = 0; j < kSlots; j += 2) {
                float d1a, d2a, d1b, d2b, diff0, diff1;
                ssd_estimate_2(my_win, slot[j], slot[j + 1], d1a, d2a, d1b, d2b);
                const bool sure0 = estimate_decides(d1a, d2a, diff0);
                const bool sure1 = estimate_decides(d1b, d2b, diff1);
                need |= (live && !sure0 ? 1u << j : 0u) | (live && !sure1 ? 2u << j : 0u);
                my_bits[slot[j].w & 0x7fff] = (slot[j].w >> 15) ? diff0 < 0.0f : diff0 > 0.0f;
                my_bits[slot[j + 1].w & 0x7fff] = (slot[j + 1].w >> 15) ? diff1 < 0.0f : diff1 > 0.0f;
            }
            if (need) {
                atomicOr(s_mask + cur, 1 << kb);
                if (defer_ok) {
#pragma unroll
                    for (int j = 0; j < kSlots; ++j)
                        if ((need >> j) & 1) {
                            const unsigned at = atomicAdd(s_qtail, 1u);
                            if (at < kQueueCap) s_queue[at] = DeferredBit{slot[j], static_cast<unsigned>(kp0 + kb)};
                        }
                }
            }
            asm volatile("bar.sync 2, %0;" ::"n"(kST) : "memory");
            const int mask = *reinterpret_cast<volatile int*>(s_mask + cur);
            bool window_pass = mask != 0;
            if (mask && defer_ok) {
                const unsigned tail = *reinterpret_cast<volatile unsigned*>(s_qtail);
                if (tail <= kQueueCap && tail - q_prev <= kDeferMax) {   // few: they stay parked
                    q_prev = tail;
                    window_pass = false;
                }
            }
            if (window_pass) {   // uniform over the consumers: some window needs its LO plane
                for (int w = 0; w < kQuad; ++w) {
                    if (!((mask >> w) & 1)) continue;
                    const double* kpr = p.xycs + 4 * (kp0 + w);
                    const double c = __ldg(kpr + 2), sn = __ldg(kpr + 3);
                    const double xa = __dadd_rn(__ldg(kpr + 0), __dmul_rn(c, du));
                    const double ya = __dadd_rn(__ldg(kpr + 1), __dmul_rn(sn, du));
                    int* lopl = reinterpret_cast<int*>(s_f) + (2 * kQuad + w) * kPlanePitch + u;
#pragma unroll 2
                    for (int v = v0; v < kWindow; v += kSRows) {
                        const double dv = static_cast<double>(v) - 31.5;
                        lopl[v * kWinStride] =
                            __double2loint(sample_exact(p.tex, xa, ya, __dmul_rn(sn, dv), __dmul_rn(c, dv)));
                    }
                    n_windows += rt == 0;
                }
                asm volatile("bar.sync 2, %0;" ::"n"(kST) : "memory");
                if (rt == 0) *s_qtail = q_prev;   // this quad's parked items are withdrawn (every consumer has read the tail)
#pragma unroll
                for (int j = 0; j < kSlots; ++j)
                    if ((need >> j) & 1) {
                        my_bits[slot[j].w & 0x7fff] =
                            triplet_bit_7x7_planes_at(my_win, lo_off, slot[j].x, slot[j].y, slot[j].z, slot[j].w >> 15);
                        ++n_flagged;
                    }
            }
        }
        __syncthreads();
        if (trace && it + 3 < kExTrace)
            trace[it + 3] = ex_global_ns() | (n_windows != windows_before ? 1ull << 63 : 0ull);
    }
    // The pipeline has drained (the loop ends on a CTA-wide barrier, every descriptor word of this CTA is in global
    // memory): all 32 warps take the parked bits, the plane memory serves as their scratch.
    {
        const unsigned parked = *reinterpret_cast<volatile unsigned*>(s_qtail);
        double* const scratch = reinterpret_cast<double*>(s_f) + warp * 160;   // 147 doubles per warp
        for (unsigned i = warp; i < parked; i += kQuadThreads / 32) {
            recompute_deferred_bit<false>(p.tex, p.xycs, p.out, p.out_index, s_queue[i], scratch, lane);
            n_flagged += lane == 0;
        }
        if (trace && parked) trace[kExTrace - 1] = ex_global_ns() | static_cast<unsigned long long>(parked) << 48;
    }
    if (p.stats != nullptr) {
        n_flagged = __reduce_add_sync(0xffffffffu, n_flagged);
        if (lane == 0 && (n_flagged | n_windows)) {
            atomicAdd(p.stats + 0, static_cast<unsigned long long>(n_flagged));
            atomicAdd(p.stats + 1, static_cast<unsigned long long>(n_windows));
        }
    }
    // How many of this CTA's windows needed the exact pass: one plain 8-byte store into page-locked host memory per
    // CTA, read by the host before the NEXT launch of this context (extraction routing, launch_extract).
    if (p.route != nullptr && !producer && rt == 0)
        p.route[blockIdx.x] = make_uint2(n_windows, static_cast<unsigned>(nq > 0 ? nq * kQuad : 0));
}

// ---- packed 16-bit planes: extract_h16_kernel (variant 5), extract_h16s_kernel (variant 6) ---------------------
// The role-split pipeline above is bound by two things at once (profiles/r4a_extract_ncu.json): the shared-memory
// pipe (3 431 wavefronts per descriptor, 80 % busy) and the issue slots (10 769 warp instructions per descriptor,
// 67 %), half of which are the producers' unfused fp64 resampling. But the planes only feed the ESTIMATE — every bit
// the estimate cannot prove is recomputed from the image by the exact code (recompute_deferred_bit, or the
// window-wide pass below) — so nothing in them has to be the reference's value, only provably close to it:
//   * a window is stored as 16-bit fixed point, A = round(65280 * b) with b the bilinear sample of the image scaled
//     to [0, 1] (8.8 fixed point of the grey level), TWICE: copy E with sample (v, u) in halfword 66 v + u, copy O in
//     halfword 66 v + u + 1. The 7 live pixels of a patch row starting at any column are then four aligned 32-bit
//     words of one copy: 28 loads per patch instead of 49, half the bytes, no misaligned pairs.
//   * the estimate unpacks a halfword with one PRMT into the mantissa of 2^23 (0x4B00hhhh = 2^23 + A as a float):
//     differences of two such floats are exact, and the packed FFMA2 sums of squares run as before.
//   * the resampler works in fp32: sample coordinates in 9.23 fixed point (start value from the keypoint's fp64
//     record, one integer add per row step), footprints through a second texture object on the same array that
//     returns texel / 255 as floats (no conversions), three fused lerps, one FFMA that rounds 65280 * b into the
//     mantissa of 2^23. No fp64 pipe, no row tables, ~24 instructions per sample instead of ~40. A lane owns the
//     column pair (2 lane, 2 lane + 1) of a row, so the two samples leave as ONE 32-bit word of copy E and — with
//     the first sample of the next lane (one shuffle) — one word of copy O: one store instruction per sample.
// Error budget, in units of the stored integers (1 = 2^-8 grey levels). Per stored sample, against the true
// bilinear value: rounding to an integer 0.5; coordinates (start value rounded once, column step once, row step
// rounded once and added <= 15 times: <= 8.5 * 2^-23 px per axis, slope <= 1 per axis in [0,1] units: 2.0e-6),
// texel / 255 in fp32 (<= 2^-23; the unit returns the correctly rounded quotient for all 256 levels, tools/tex_probe.cu
// -> profiles/r4g_tex_probe.json) and six fp32 roundings in the lerps (3.6e-7): <= 2.5e-6 * 65280 = 0.16. So
// |A - true| <= 0.66 and a difference of two samples is off by at most eta = 1.32. Per chain, d_f the fp32 sum:
//   |65536 d_ref - d_f| <= 2 eta sum|e| + 49 eta^2      (sum|e| <= 7 sqrt(d) over the 49 terms)
//                          + 52 * 2^-24 d_f              (49 fused accumulations; the differences are exact)
//                          + 6e-15 d_f                   (the reference's own fp64 roundings)
// The kernels test |d1_f - d2_f| > 19.1 (sqrt d1_f + sqrt d2_f) + 3.3e-6 (d1_f + d2_f) + 180 (constants rounded up
// >= 3 %): on noise images 9e-4 of the bits stay undecided (the fp32 planes: 2e-5) — half a bit per descriptor,
// parked and recomputed exactly by whole warps after the pipeline has drained.
// Schedules: variant 5 keeps dedicated producer / consumer warps (16 + 16), variant 6 lets every warp do both
// halves of an iteration, half of the warps of each SM sub-partition in one order and half in the other.
constexpr int kHRow = kH16RowWords;                                  // 33 words per plane row
constexpr int kHCopy = kH16CopyWords;                                // 2112 words: copy E, then copy O
constexpr int kHPitch = 2 * kHCopy + 8;                              // words per window; % 32 == 8
constexpr int kHRecDoubles = 10;                                     // per-window record, see stage_quad_h16
constexpr int kH16PlaneBytes = 2 * kQuad * kHPitch * 4;              // [2][4] windows
constexpr int kH16ExactBytes = kWindow * kWinStride * 8;             // one fp64 window for the window-wide exact pass
constexpr int kH16SmemBytes = kH16PlaneBytes + kH16ExactBytes
                              + 2 * kQuad * kPipeBits                // predicate bytes [2][4][512 + pad]
                              + 2 * kQuad * kHRecDoubles * 8         // window records [2][4]
                              + 64                                   // undecided-window masks, deferred-queue tail
                              + kQueueCap * static_cast<int>(sizeof(DeferredBit));
static_assert(kHPitch % 32 == 8 && kH16SmemBytes <= 227 * 1024, "packed-plane layout");

// The exact chains as a call (rare path: keeps the pipelined loop's code small).
__device__ __noinline__ bool triplet_bit_7x7_cold(const double* win, int oa, int ob, int oc, bool swapped) {
    return triplet_bit_7x7(win, oa, ob, oc, swapped);
}

// The exact bit of a packed-plane slot from an fp64 window (stride kWinStride).
__device__ __forceinline__ bool h16_exact_bit(const double* win, const ushort4 s) {
    int ax, ay, bx, by, cx, cy;
    h16_anchor_dev(s.x, ax, ay);
    h16_anchor_dev(s.y, bx, by);
    h16_anchor_dev(s.z, cx, cy);
    return triplet_bit_7x7_cold(win, ay * kWinStride + ax, by * kWinStride + bx, cy * kWinStride + cx, s.w >> 15);
}

// fp32 estimate of both chains of two slots from the packed planes (component 0 = slot 0, 1 = slot 1).
// kBig = 0x4B000000 (2^23: PRMT drops a halfword into its mantissa) arrives as a kernel PARAMETER: PRMT takes one
// immediate, and when ptxas knows both the selector and this word it keeps the selector in a register that it
// re-materialises with a MOV in front of every PRMT (measured: 380 extra instructions per pass).
__device__ __forceinline__ void ssd_estimate_h16_2(const unsigned* win, const ushort4 s0, const ushort4 s1, const unsigned kBig,
                                                   float& d1a, float& d2a, float& d1b, float& d2b) {
    const unsigned* pa0 = win + s0.x;
    const unsigned* pb0 = win + s0.y;
    const unsigned* pc0 = win + s0.z;
    const unsigned* pa1 = win + s1.x;
    const unsigned* pb1 = win + s1.y;
    const unsigned* pc1 = win + s1.z;
    const float2 neg1 = make_float2(-1.0f, -1.0f);
    float2 d1 = make_float2(0.0f, 0.0f), d2 = d1;
#pragma unroll
    for (int r = 0; r < 7; ++r) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int o = r * kHRow + k;
            const unsigned wa0 = pa0[o], wa1 = pa1[o], wb0 = pb0[o], wb1 = pb1[o], wc0 = pc0[o], wc1 = pc1[o];
#pragma unroll
            for (int h = 0; h < (k < 3 ? 2 : 1); ++h) {
                const unsigned sel = h ? 0x7632u : 0x7610u;
                const float2 a = make_float2(__uint_as_float(__byte_perm(wa0, kBig, sel)), __uint_as_float(__byte_perm(wa1, kBig, sel)));
                const float2 b = make_float2(__uint_as_float(__byte_perm(wb0, kBig, sel)), __uint_as_float(__byte_perm(wb1, kBig, sel)));
                const float2 c = make_float2(__uint_as_float(__byte_perm(wc0, kBig, sel)), __uint_as_float(__byte_perm(wc1, kBig, sel)));
                const float2 e1 = __ffma2_rn(b, neg1, a);   // exact: both are 2^23 + a 16-bit integer
                const float2 e2 = __ffma2_rn(c, neg1, a);
                d1 = __ffma2_rn(e1, e1, d1);
                d2 = __ffma2_rn(e2, e2, d2);
            }
        }
    }
    d1a = d1.x;
    d1b = d1.y;
    d2a = d2.x;
    d2b = d2.y;
}

// True when sign(d1 - d2) of the packed-plane estimate is provably the reference's (budget above).
__device__ __forceinline__ bool estimate_decides_h16(float d1, float d2, float& diff) {
    float r1, r2;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d1));
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(d2));
    diff = d1 - d2;
    const float bound = __fmaf_rn(19.1f, r1 + r2, __fmaf_rn(3.3e-6f, d1 + d2, 180.0f));
    return fabsf(diff) > bound;
}

// Window records of the quad that starts at keypoint kp0, by threads 0..3 of whoever stages: the keypoint
// {x, y, cos, sin}, floor(x), floor(y) as doubles, then eight ints — the texel coordinates of the footprint centre of
// relative cell (0, 0) as floats-to-be {0x4B000000 + floor(x) + 1, 0x4B000000 + floor(y) + 1}, the per-row-step
// increments of the 9.23 fixed-point sample coordinates {round(-sin * rows * 2^23), round(cos * rows * 2^23)} and the
// column step {round(cos * 2^23), round(sin * 2^23)} to the second sample of a lane's pair.
// A keypoint past the end repeats the last one (its window is computed and never used).
struct H16Kp {
    double x, y, c, sn;
};
__device__ __forceinline__ H16Kp h16_kp_load(const ExtractParams& p, unsigned long long kp0, int t) {
    const unsigned long long kp = min(kp0 + t, p.M - 1);
    return H16Kp{__ldg(p.xycs + 4 * kp + 0), __ldg(p.xycs + 4 * kp + 1), __ldg(p.xycs + 4 * kp + 2), __ldg(p.xycs + 4 * kp + 3)};
}
__device__ __forceinline__ void h16_rec_store(const H16Kp k, double* rec, int t, int rows) {
    int xi, yi;
    double xid, yid;
    floor_exact(k.x, xi, xid);
    floor_exact(k.y, yi, yid);
    double* const r = rec + kHRecDoubles * t;
    r[0] = k.x;
    r[1] = k.y;
    r[2] = k.c;
    r[3] = k.sn;
    r[4] = xid;
    r[5] = yid;
    const double one = 8388608.0, step = static_cast<double>(rows) * one;   // 2^23, rows * 2^23
    const double kRound = 6755399441055744.0;                                // 1.5 * 2^52: low word = nearest integer
    int* const ri = reinterpret_cast<int*>(r + 6);
    ri[0] = 0x4B000000 + xi + 1;
    ri[1] = 0x4B000000 + yi + 1;
    ri[2] = __double2loint(__dadd_rn(__dmul_rn(-k.sn, step), kRound));
    ri[3] = __double2loint(__dadd_rn(__dmul_rn(k.c, step), kRound));
    ri[4] = __double2loint(__dadd_rn(__dmul_rn(k.c, one), kRound));
    ri[5] = __double2loint(__dadd_rn(__dmul_rn(k.sn, one), kRound));
    ri[6] = ri[7] = 0;
}
// (Split in two so that the global loads can be issued before an iteration's work and the record written after it:
// done in one piece at the top of an iteration, the ~1 us of load latency sat on the staging warp's critical path.)
__device__ __forceinline__ void stage_quad_h16(const ExtractParams& p, unsigned long long kp0, double* rec, int t, int rows) {
    if (t < kQuad) h16_rec_store(h16_kp_load(p, kp0, t), rec, t, rows);
}

// One thread's share of a quad's resampling: window record `rec`, that window's planes, column pair (2 lane, 2 lane + 1),
// rows v0 + kRows * k. Four gathers stay in flight.
template <int kRows>
__device__ __forceinline__ void h16_resample_pairs(cudaTextureObject_t texn, const double* rec, unsigned* plane, int lane, int v0) {
    constexpr int kPer = kWindow / kRows, kTotal = 2 * kPer, kDepth = 4;
    const double du = static_cast<double>(2 * lane) - 31.5, dv0 = static_cast<double>(v0) - 31.5;
    const double c = rec[2], sn = rec[3];
    const double sx0 = __dsub_rn(__dadd_rn(rec[0], __dmul_rn(c, du)), __dmul_rn(sn, dv0));
    const double sy0 = __dadd_rn(__dadd_rn(rec[1], __dmul_rn(sn, du)), __dmul_rn(c, dv0));
    const int4 k4 = reinterpret_cast<const int4*>(rec + 6)[0];
    const int2 k2 = reinterpret_cast<const int2*>(rec + 8)[0];
    // (s - floor) * 2^23 rounded to an integer: the ulp at 1.5 * 2^29 is 2^-23
    int Xa = __double2loint(__dadd_rn(__dsub_rn(sx0, rec[4]), 805306368.0));
    int Ya = __double2loint(__dadd_rn(__dsub_rn(sy0, rec[5]), 805306368.0));
    int Xb = Xa + k2.x, Yb = Ya + k2.y;
    float pfx[kDepth], pfy[kDepth];
    float4 pg[kDepth];
    unsigned qa = 0;
    unsigned* const ebase = plane + v0 * kHRow + lane;
#pragma unroll
    for (int i = 0; i < kTotal + kDepth; ++i) {
        if (i >= kDepth) {
            const int j = i - kDepth, sl = j % kDepth;
            const float4 g = pg[sl];   // w = (x0,y0), z = (x0+1,y0), x = (x0,y0+1), y = (x0+1,y0+1), each texel / 255
            const float top = __fmaf_rn(pfx[sl], g.z - g.w, g.w);
            const float bot = __fmaf_rn(pfx[sl], g.y - g.x, g.x);
            const float val = __fmaf_rn(pfy[sl], bot - top, top);
            const unsigned q = __float_as_uint(__fmaf_rn(val, 65280.0f, 8388608.0f));   // low half: round(65280 * val)
            if (j % 2 == 0) {
                qa = q;
            } else {
                const unsigned next = __shfl_down_sync(0xffffffffu, qa, 1);   // sample 2 lane + 2 (lane 31: a word nobody reads)
                unsigned* const dst = ebase + (j / 2) * kRows * kHRow;
                dst[0] = __byte_perm(qa, q, 0x5410);                          // copy E: samples (2 lane, 2 lane + 1)
                dst[kHCopy + 1] = __byte_perm(q, next, 0x5410);               // copy O: samples (2 lane + 1, 2 lane + 2)
            }
        }
        if (i < kTotal) {
            const int sl = i % kDepth;
            const int X = i % 2 ? Xb : Xa, Y = i % 2 ? Yb : Ya;
            const float tx = __int_as_float(k4.x + (X >> 23)) - 8388608.0f;   // floor + 1: the footprint's centre
            const float ty = __int_as_float(k4.y + (Y >> 23)) - 8388608.0f;
            pfx[sl] = __int_as_float((X & 0x7fffff) | 0x3f800000) - 1.0f;
            pfy[sl] = __int_as_float((Y & 0x7fffff) | 0x3f800000) - 1.0f;
            pg[sl] = tex2Dgather<float4>(texn, tx, ty, 0);
            if (i % 2) {
                Xa += k4.z;
                Ya += k4.w;
                Xb += k4.z;
                Yb += k4.w;
            }
        }
    }
}

// Pack 512 predicate bytes of one window (two ballots per thread of a 256-thread group) into the descriptor row.
__device__ __forceinline__ void h16_pack_bits(const ExtractParams& p, const uint8_t* bits, unsigned long long kp, int j, int lane) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const unsigned w32 = __ballot_sync(0xffffffffu, bits[256 * k + j] != 0);
        if (lane == 0 && kp < p.M) {
            const unsigned long long row = p.out_index ? p.out_index[kp] : kp;
            reinterpret_cast<unsigned*>(p.out + row * (kFastT / 8))[8 * k + (j >> 5)] = w32;
        }
    }
}

// Diagnostics (clatch_estimate_planes_u8_dev): the stored samples of the default kernel's estimate planes — the same
// resampler, one CTA of 16 warps per quad — as M x 64 x 64 uint16 (row-major, copy E), so that a test can hold
// every sample against the reference's fp64 window and the error budget above (|A - 256 v| <= 0.66).
__global__ void __launch_bounds__(512, 1) h16_planes_kernel(ExtractParams p, unsigned short* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t s_quad[];
    unsigned* const s_h = reinterpret_cast<unsigned*>(s_quad);                        // [4] windows
    double* const s_rec = reinterpret_cast<double*>(s_quad + kQuad * kHPitch * 4);    // [4][10]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned long long quads = (p.M + kQuad - 1) / kQuad;
    for (unsigned long long q = blockIdx.x; q < quads; q += gridDim.x) {
        stage_quad_h16(p, q * kQuad, s_rec, tid, 4);
        __syncthreads();
        h16_resample_pairs<4>(p.texn, s_rec + (warp >> 2) * kHRecDoubles, s_h + (warp >> 2) * kHPitch, lane, warp & 3);
        __syncthreads();
        for (int i = tid; i < kQuad * kWindow * kWindow; i += blockDim.x) {
            const int w = i >> 12, v = (i >> 6) & 63, u = i & 63;
            if (q * kQuad + w < p.M)
                out[(q * kQuad + w) * (kWindow * kWindow) + v * kWindow + u] =
                    reinterpret_cast<const unsigned short*>(s_h + w * kHPitch)[v * (2 * kHRow) + u];
        }
        __syncthreads();
    }
}

// kF64: a float64 image whose pixels are not all u8 values. The planes then come from a float texture of the image
// scaled to [0, 1] over its own range (fill_array_f32_kernel; the estimate and its bound only see that texture, and
// bilinear sampling commutes with the affine map), the exact paths sample the doubles in global memory.
template <int kRW, bool kF64>
__global__ void __launch_bounds__(kQuadThreads, 1) extract_h16_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;
    constexpr int kSW = 32 - kRW, kST = kSW * 32;
    constexpr int kStep = 32 / kSW;                          // every kStep-th group of 4 warps consumes
    constexpr int kRRows = kRW / kQuad;                      // a producer warp owns rows v0 + kRRows * k of one window
    constexpr int kSRows = kST / kWindow;                    // exact pass: consumer thread -> rows v0 + kSRows * k
    constexpr int kSlots = 64 / kSW;                         // groups of 8 triplets per consumer warp
    static_assert(32 % kSW == 0 && 64 % kSW == 0 && kSlots % 2 == 0 && kRW % kQuad == 0 && kWindow % kRRows == 0 && kST == 512,
                  "role split");

    extern __shared__ __align__(16) uint8_t s_quad[];
    unsigned* const s_h = reinterpret_cast<unsigned*>(s_quad);                                   // packed planes [2][4]
    double* const s_exact = reinterpret_cast<double*>(s_quad + kH16PlaneBytes);                  // one fp64 window
    uint8_t* const s_bits = s_quad + kH16PlaneBytes + kH16ExactBytes;                            // [2][4][512 + pad]
    double* const s_rec = reinterpret_cast<double*>(s_bits + 2 * kQuad * kPipeBits);             // [2][4][10]
    int* const s_mask = reinterpret_cast<int*>(s_rec + 2 * kQuad * kHRecDoubles);                // [2] windows needing the exact pass
    unsigned* const s_qtail = reinterpret_cast<unsigned*>(s_mask + 2);                           // deferred bits queued so far
    unsigned* const s_qid = reinterpret_cast<unsigned*>(s_mask + 4);                             // [8] quad of pipeline iteration it at [it & 7]
    DeferredBit* const s_queue = reinterpret_cast<DeferredBit*>(s_mask + 16);                    // [kQueueCap]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, grp = warp >> 2;
    const bool producer = grp % kStep != 0;
    const int rw = (producer ? grp - grp / kStep - 1 : grp / kStep) * 4 + (warp & 3);   // role-local warp
    const int rt = rw * 32 + lane;                                                       // role-local thread
    const int u = rt & 63, v0 = rt >> 6;                     // window-wide exact pass (consumers)
    const double du = static_cast<double>(u) - 31.5;
    const int kb = lane & 3, ti = lane >> 2;
    // Quads are handed out dynamically (ExtractParams::tickets: a device counter the last CTA to finish resets): a CTA's
    // first three quads are the round-robin ones (every CTA draws at the same moment at the start: 148 atomics on one word
    // take 4 us, which only a full pipeline iteration hides), every further one a ticket drawn three iterations ahead. On images whose
    // flat or saturated regions send some windows through the window-wide exact pass (6 us each against 1.9 us for the
    // estimate alone) a static round-robin left the launch waiting for the unluckiest CTA (span 226 us, mean 160).
    const unsigned nquads = static_cast<unsigned>(min((p.M + kQuad - 1) / kQuad, 0xffffffffull));   // also "no quad"
    ushort4 slot[kSlots];
#pragma unroll
    for (int j = 0; j < kSlots; ++j) slot[j] = __ldg(p.slots + 8 * (rw % kSW + kSW * j) + ti);
    unsigned n_flagged = 0, n_windows = 0;
    unsigned long long* const trace = p.trace != nullptr && tid == 0 ? p.trace + static_cast<size_t>(kExTrace) * blockIdx.x : nullptr;
    if (trace) trace[0] = ex_global_ns();
    if (tid == 0) {
        s_mask[0] = s_mask[1] = 0, *s_qtail = 0;
        for (unsigned i = 0; i < 3; ++i) s_qid[i] = min(blockIdx.x + i * gridDim.x, nquads);
    }
    // Sparse undecided bits are parked ({slot, keypoint} in a shared-memory queue) and recomputed exactly by whole warps
    // after the pipeline has drained; a quad with more than kDeferMax of them (flat or saturated footprints), or a full
    // queue, takes the window-wide exact pass instead. See extract_roles_kernel.
    const bool defer_ok = p.M <= 0xffffffffull;
    unsigned q_prev = 0;                 // queue tail after the previous quad (uniform over the consumers)
    unsigned quads_done = 0;
    bool prev_live = false;              // consumers: the previous iteration's quad existed
    bool checked_out = false;            // producer thread 0: this CTA has drawn its last ticket
    stage_quad_h16(p, static_cast<unsigned long long>(blockIdx.x) * kQuad, s_rec, tid, kRRows);
    __syncthreads();
    pdl_wait();   // launched early behind fill_array_kernel: the texture array is complete from here on
    if (trace) trace[1] = ex_global_ns();

    for (int it = -1;; ++it) {
        const int cur = it & 1, nxt = cur ^ 1;
        const unsigned windows_before = n_windows;
        // Each role reads only the ring entries it needs, where it needs them (the consumers one per iteration). Both leave
        // the loop in the iteration after the one whose quad did not exist: tickets only grow, so nothing is in flight then.
        if (producer) {
            const unsigned q_done = it >= 1 ? s_qid[(it - 1) & 7] : nquads;   // its bits are complete: packed and stored now
            if (it >= 1 && q_done >= nquads) break;
            const unsigned q_stage = s_qid[(it + 2) & 7];
            unsigned ticket = nquads;   // drawn now, stored at the end of the iteration: the round trip hides behind the resampling
            if (rt == 0 && it >= 0 && q_stage < nquads)   // (after pdl_wait: the previous launch's rewind of the counter is visible)
                ticket = p.tickets != nullptr ? 3 * gridDim.x + atomicAdd(p.tickets, 1u) : q_stage + gridDim.x;
            // The producers, which have slack (they resample a quad in half the time the consumers need to estimate one),
            // also pack the previous quad's bits and stage the window records two quads ahead (buffer [quad & 1]; its last
            // readers resampled quad `it`, an iteration ago): the consumers' critical path is the estimate alone.
            if (q_done < nquads) {
                const int w = rt >> 7, j = rt & 127;
                const uint8_t* bits = s_bits + (nxt * kQuad + w) * kPipeBits;
                const unsigned long long kp = static_cast<unsigned long long>(q_done) * kQuad + w;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const unsigned w32 = __ballot_sync(0xffffffffu, bits[128 * k + j] != 0);
                    if (lane == 0 && kp < p.M) {
                        const unsigned long long row = p.out_index ? p.out_index[kp] : kp;
                        reinterpret_cast<unsigned*>(p.out + row * (kFastT / 8))[4 * k + (j >> 5)] = w32;
                    }
                }
            }
            if (s_qid[(it + 1) & 7] < nquads && !(p.dbg & 2))   // resample the next quad into the planes [nxt]: this warp's window, its rows
                h16_resample_pairs<kRRows>(p.texn, s_rec + (nxt * kQuad + rw / kRRows) * kHRecDoubles,
                                           s_h + (nxt * kQuad + rw / kRRows) * kHPitch, lane, rw % kRRows);
            if (q_stage < nquads)
                stage_quad_h16(p, static_cast<unsigned long long>(q_stage) * kQuad, s_rec + cur * kQuad * kHRecDoubles, rt, kRRows);
            if (rt == 0 && it >= 0) {
                s_qid[(it + 3) & 7] = ticket < nquads ? ticket : nquads;
                // This CTA's first ticket past the end is its last draw: it checks out here, inside the producers' slack, and
                // the last CTA to do so rewinds the counter for the next launch on this stream (nothing draws any more).
                if (ticket >= nquads && !checked_out) {
                    checked_out = true;
                    if (p.tickets != nullptr && atomicInc(p.tickets + 1, gridDim.x - 1) == gridDim.x - 1) p.tickets[0] = 0;
                }
            }
        } else {
            if (it >= 1 && !prev_live) break;
            const unsigned q_now = it >= 0 ? s_qid[it & 7] : nquads;          // estimated now
            const unsigned long long kp0 = static_cast<unsigned long long>(q_now) * kQuad;   // first keypoint of quad `it`
            prev_live = q_now < nquads;
            if (prev_live) {
                ++quads_done;
                const unsigned* const my_win = s_h + (cur * kQuad + kb) * kHPitch;
                const bool live = kp0 + kb < p.M;   // a keypoint past the end leaves an unused window
                if (rt == 0) s_mask[nxt] = 0;
                uint8_t* const my_bits = s_bits + (cur * kQuad + kb) * kPipeBits;
                unsigned need = 0;
#pragma unroll
                for (int j = 0; j < kSlots; j += 2) {
                    float d1a = 1.f, d2a = 2e9f, d1b = 1.f, d2b = 2e9f, diff0, diff1;
                    if (!(p.dbg & 1)) ssd_estimate_h16_2(my_win, slot[j], slot[j + 1], p.two23, d1a, d2a, d1b, d2b);
                    const bool sure0 = estimate_decides_h16(d1a, d2a, diff0);
                    const bool sure1 = estimate_decides_h16(d1b, d2b, diff1);
                    need |= (live && !sure0 ? 1u << j : 0u) | (live && !sure1 ? 2u << j : 0u);
                    my_bits[slot[j].w & 0x7fff] = (slot[j].w >> 15) ? diff0 < 0.0f : diff0 > 0.0f;
                    my_bits[slot[j + 1].w & 0x7fff] = (slot[j + 1].w >> 15) ? diff1 < 0.0f : diff1 > 0.0f;
                }
                if (need) {
                    atomicOr(s_mask + cur, 1 << kb);
                    if (defer_ok) {
#pragma unroll
                        for (int j = 0; j < kSlots; ++j)
                            if ((need >> j) & 1) {
                                const unsigned at = atomicAdd(s_qtail, 1u);
                                if (at < kQueueCap) s_queue[at] = DeferredBit{slot[j], static_cast<unsigned>(kp0 + kb)};
                            }
                    }
                }
                asm volatile("bar.sync 2, %0;" ::"n"(kST) : "memory");
                const int mask = *reinterpret_cast<volatile int*>(s_mask + cur);
                bool window_pass = mask != 0;
                if (mask && defer_ok) {
                    const unsigned tail = *reinterpret_cast<volatile unsigned*>(s_qtail);
                    if (tail <= kQueueCap && tail - q_prev <= kDeferMax) {   // few: they stay parked
                        q_prev = tail;
                        window_pass = false;
                    }
                }
                if (window_pass) {   // uniform over the consumers: dense undecided bits (flat / saturated footprints)
                    for (int w = 0; w < kQuad; ++w) {
                        if (!((mask >> w) & 1)) continue;
                        // the consumers resample window w exactly (fp64, the reference's operation order) ...
                        const double* kpr = p.xycs + 4 * (kp0 + w);
                        const double c = __ldg(kpr + 2), sn = __ldg(kpr + 3);
                        const double xa = __dadd_rn(__ldg(kpr + 0), __dmul_rn(c, du));
                        const double ya = __dadd_rn(__ldg(kpr + 1), __dmul_rn(sn, du));
#pragma unroll 2
                        for (int v = v0; v < kWindow; v += kSRows) {
                            const double dv = static_cast<double>(v) - 31.5;
                            s_exact[v * kWinStride + u] =
                                kF64 ? sample_exact_f64(static_cast<const double*>(p.img), p.pitch, xa, ya, __dmul_rn(sn, dv), __dmul_rn(c, dv))
                                     : sample_exact(p.tex, xa, ya, __dmul_rn(sn, dv), __dmul_rn(c, dv));
                        }
                        n_windows += rt == 0;
                        asm volatile("bar.sync 2, %0;" ::"n"(kST) : "memory");
                        if (rt == 0) *s_qtail = q_prev;   // this quad's parked items are withdrawn (every consumer has read the tail)
                        // ... and the 512 consumer threads run the exact chains of ALL 512 triplets of that window, one
                        // each, in the one-window lane placement (bank pairs planned for a single fp64 window): with only
                        // the undecided lanes of the packed-plane placement at work — a quarter of the lanes, their
                        // patches colliding 4-8-way in the fp64 window — a flat window took 13 us, this way ~6.
                        {
                            const ushort4 sw = __ldg(p.slots_sw + rt);
                            s_bits[(cur * kQuad + w) * kPipeBits + (sw.w & 0x7fff)] = triplet_bit_7x7_cold(s_exact, sw.x, sw.y, sw.z, sw.w >> 15);
                            ++n_flagged;
                        }
                        asm volatile("bar.sync 2, %0;" ::"n"(kST) : "memory");   // the next window overwrites the scratch
                    }
                }
            }
        }
        __syncthreads();
        if (trace && it + 3 < kExTrace - 2)
            trace[it + 3] = ex_global_ns() | (n_windows != windows_before ? 1ull << 63 : 0ull);
    }
    // The pipeline has drained: all 32 warps take the parked bits, the plane memory serves as their scratch.
    {
        const unsigned parked = *reinterpret_cast<volatile unsigned*>(s_qtail);
        double* const scratch = reinterpret_cast<double*>(s_h) + warp * 160;   // 147 doubles per warp
        for (unsigned i = warp; i < parked; i += kQuadThreads / 32) {
            recompute_deferred_bit<true, kF64>(p.tex, p.xycs, p.out, p.out_index, s_queue[i], scratch, lane,
                                               static_cast<const double*>(p.img), p.pitch);
            n_flagged += lane == 0;
        }
        if (trace && parked) trace[kExTrace - 1] = (ex_global_ns() & 0xffffffffffffull) | static_cast<unsigned long long>(parked) << 48;
        if (trace) trace[kExTrace - 2] = quads_done;
    }
    if (p.stats != nullptr) {
        n_flagged = __reduce_add_sync(0xffffffffu, n_flagged);
        if (lane == 0 && (n_flagged | n_windows)) {
            atomicAdd(p.stats + 0, static_cast<unsigned long long>(n_flagged));
            atomicAdd(p.stats + 1, static_cast<unsigned long long>(n_windows));
        }
    }
    if (p.route != nullptr && !producer && rt == 0)
        p.route[blockIdx.x] = make_uint2(n_windows, quads_done * kQuad);
}

__global__ void __launch_bounds__(kQuadThreads, 1) extract_h16s_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;
    constexpr int kRows = kQuadThreads / 32 / kQuad;         // 8: a warp owns rows v0 + 8k of one window

    extern __shared__ __align__(16) uint8_t s_quad[];
    unsigned* const s_h = reinterpret_cast<unsigned*>(s_quad);                                   // packed planes [2][4]
    double* const s_exact = reinterpret_cast<double*>(s_quad + kH16PlaneBytes);                  // one fp64 window
    uint8_t* const s_bits = s_quad + kH16PlaneBytes + kH16ExactBytes;                            // [2][4][512 + pad]
    double* const s_rec = reinterpret_cast<double*>(s_bits + 2 * kQuad * kPipeBits);             // [2][4][10]
    int* const s_mask = reinterpret_cast<int*>(s_rec + 2 * kQuad * kHRecDoubles);                // [3] windows needing the exact pass
    unsigned* const s_qtail = reinterpret_cast<unsigned*>(s_mask + 3);                           // deferred bits queued so far
    DeferredBit* const s_queue = reinterpret_cast<DeferredBit*>(s_mask + 16);                    // [kQueueCap]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool ssd_first = (warp >> 2) & 1;                  // per sub-partition: 4 warps each way
    const int rwin = warp >> 3, rv0 = warp & 7;              // resampling: window of the quad, first row
    const int u = tid & 63, v0 = tid >> 6;                   // window-wide exact pass: column u, rows v0 + 16k
    const double du = static_cast<double>(u) - 31.5;
    const int kb = lane & 3, ti = lane >> 2;                 // estimate: 8 triplets x 4 keypoints per warp
    const ushort4 slot0 = __ldg(p.slots + 8 * warp + ti);
    const ushort4 slot1 = __ldg(p.slots + 8 * warp + ti + kFastT / 2);
    const unsigned long long quads = (p.M + kQuad - 1) / kQuad;
    const int nq = blockIdx.x < quads ? static_cast<int>((quads - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
    const unsigned long long kp_step = static_cast<unsigned long long>(gridDim.x) * kQuad;
    unsigned n_flagged = 0, n_windows = 0;
    unsigned long long* const trace = p.trace != nullptr && tid == 0 ? p.trace + static_cast<size_t>(kExTrace) * blockIdx.x : nullptr;
    if (trace) trace[0] = ex_global_ns();
    if (tid < 4) s_mask[tid] = 0;   // three masks and the queue tail
    const bool defer_ok = p.M <= 0xffffffffull;
    unsigned q_prev = 0;            // queue tail after the previous quad (uniform over the CTA)
    unsigned long long kp0 = static_cast<unsigned long long>(blockIdx.x) * kQuad - kp_step;   // first keypoint of quad `it`
    int mslot = 2;                  // (it + 3) % 3
    stage_quad_h16(p, static_cast<unsigned long long>(blockIdx.x) * kQuad, s_rec, tid, kRows);
    __syncthreads();
    pdl_wait();   // launched early behind fill_array_kernel: the texture array is complete from here on
    if (trace) trace[1] = ex_global_ns();

    for (int it = -1; it <= nq; ++it, kp0 += kp_step, mslot = mslot == 2 ? 0 : mslot + 1) {
        const int cur = it & 1, nxt = cur ^ 1;
        const bool consume = it >= 0 && it < nq, produce = it + 1 < nq;
        const unsigned windows_before = n_windows;
        if (tid == 0) s_mask[mslot == 2 ? 0 : mslot + 1] = 0;   // quad it-2's mask: every reader is past it
        if (it + 2 < nq) stage_quad_h16(p, kp0 + 2 * kp_step, s_rec + cur * kQuad * kHRecDoubles, tid, kRows);   // -> buffer [cur]
        if (it >= 1)   // pack the bits of quad it-1 (buffer [nxt])
            h16_pack_bits(p, s_bits + (nxt * kQuad + (tid >> 8)) * kPipeBits, kp0 - kp_step + (tid >> 8), tid & 255, lane);

        const unsigned* const my_win = s_h + (cur * kQuad + kb) * kHPitch;
        uint8_t* const my_bits = s_bits + (cur * kQuad + kb) * kPipeBits;
        unsigned need = 0;
        {
            float d1a = 0.f, d2a = 0.f, d1b = 0.f, d2b = 0.f;
#pragma unroll 1
            for (int phase = 0; phase < 2; ++phase) {
                if ((phase == 0) == ssd_first) {
                    if (consume) ssd_estimate_h16_2(my_win, slot0, slot1, p.two23, d1a, d2a, d1b, d2b);
                } else if (produce) {
                    h16_resample_pairs<kRows>(p.texn, s_rec + (nxt * kQuad + rwin) * kHRecDoubles,
                                              s_h + (nxt * kQuad + rwin) * kHPitch, lane, rv0);
                }
            }
            if (consume) {
                float diff0, diff1;
                const bool sure0 = estimate_decides_h16(d1a, d2a, diff0);
                const bool sure1 = estimate_decides_h16(d1b, d2b, diff1);
                const bool live = kp0 + kb < p.M;   // a keypoint past the end leaves an unused window
                need = (live && !sure0 ? 1u : 0u) | (live && !sure1 ? 2u : 0u);
                my_bits[slot0.w & 0x7fff] = (slot0.w >> 15) ? diff0 < 0.0f : diff0 > 0.0f;
                my_bits[slot1.w & 0x7fff] = (slot1.w >> 15) ? diff1 < 0.0f : diff1 > 0.0f;
                if (need) {
                    atomicOr(s_mask + mslot, 1 << kb);
                    if (defer_ok) {
                        if (need & 1) {
                            const unsigned at = atomicAdd(s_qtail, 1u);
                            if (at < kQueueCap) s_queue[at] = DeferredBit{slot0, static_cast<unsigned>(kp0 + kb)};
                        }
                        if (need & 2) {
                            const unsigned at = atomicAdd(s_qtail, 1u);
                            if (at < kQueueCap) s_queue[at] = DeferredBit{slot1, static_cast<unsigned>(kp0 + kb)};
                        }
                    }
                }
            }
        }
        __syncthreads();

        if (consume) {
            const int mask = *reinterpret_cast<volatile int*>(s_mask + mslot);
            bool window_pass = mask != 0;
            if (mask && defer_ok) {
                const unsigned tail = *reinterpret_cast<volatile unsigned*>(s_qtail);
                if (tail <= kQueueCap && tail - q_prev <= kDeferMax) {   // few: they stay parked
                    q_prev = tail;
                    window_pass = false;
                }
            }
            if (window_pass) {   // block-uniform: dense undecided bits (flat / saturated footprints)
                for (int w = 0; w < kQuad; ++w) {
                    if (!((mask >> w) & 1)) continue;
                    // the CTA resamples window w exactly (fp64, the reference's operation order) ...
                    const double* kpr = p.xycs + 4 * (kp0 + w);   // (the staged copy is already quad it+2's)
                    const double c = __ldg(kpr + 2), sn = __ldg(kpr + 3);
                    const double xa = __dadd_rn(__ldg(kpr + 0), __dmul_rn(c, du));
                    const double ya = __dadd_rn(__ldg(kpr + 1), __dmul_rn(sn, du));
#pragma unroll 2
                    for (int v = v0; v < kWindow; v += kQuadThreads / kWindow) {
                        const double dv = static_cast<double>(v) - 31.5;
                        s_exact[v * kWinStride + u] = sample_exact(p.tex, xa, ya, __dmul_rn(sn, dv), __dmul_rn(c, dv));
                    }
                    n_windows += tid == 0;
                    __syncthreads();
                    if (tid == 0) *s_qtail = q_prev;   // this quad's parked items are withdrawn (every thread has read the tail;
                                                       // the next additions come after the barrier below)
                    // ... and the lanes of that window run the exact chains of their undecided triplets
                    if (kb == w && need) {
                        if (need & 1) {
                            my_bits[slot0.w & 0x7fff] = h16_exact_bit(s_exact, slot0);
                            ++n_flagged;
                        }
                        if (need & 2) {
                            my_bits[slot1.w & 0x7fff] = h16_exact_bit(s_exact, slot1);
                            ++n_flagged;
                        }
                    }
                    __syncthreads();   // the next window overwrites the scratch; the next iteration packs these bits
                }
            }
        }
        if (trace && it + 3 < kExTrace)
            trace[it + 3] = ex_global_ns() | (n_windows != windows_before ? 1ull << 63 : 0ull);
    }
    __syncthreads();
    // The pipeline has drained: every warp takes parked bits, the plane memory serves as their scratch.
    {
        const unsigned parked = *reinterpret_cast<volatile unsigned*>(s_qtail);
        double* const scratch = reinterpret_cast<double*>(s_h) + warp * 160;   // 147 doubles per warp
        for (unsigned i = warp; i < parked; i += kQuadThreads / 32) {
            recompute_deferred_bit<true>(p.tex, p.xycs, p.out, p.out_index, s_queue[i], scratch, lane);
            n_flagged += lane == 0;
        }
        if (trace && parked) trace[kExTrace - 1] = ex_global_ns() | static_cast<unsigned long long>(parked) << 48;
    }
    if (p.stats != nullptr) {
        n_flagged = __reduce_add_sync(0xffffffffu, n_flagged);
        if (lane == 0 && (n_flagged | n_windows)) {
            atomicAdd(p.stats + 0, static_cast<unsigned long long>(n_flagged));
            atomicAdd(p.stats + 1, static_cast<unsigned long long>(n_windows));
        }
    }
    if (p.route != nullptr && tid == 0)
        p.route[blockIdx.x] = make_uint2(n_windows, static_cast<unsigned>(nq > 0 ? nq * kQuad : 0));
}

// Generic pattern: any T (multiple of 8), 1 <= K <= 64, arbitrary non-negative weights.
// d += (w*e)*e exactly as the reference writes it (src/descriptor.cpp:70-71).
template <bool kU8>
__global__ void __launch_bounds__(kThreads, 2) extract_generic_kernel(ExtractParams p) {
    if (p.flags != nullptr && p.flags[0] != p.run_if_flag) return;

    __shared__ __align__(16) double s_win[kWindow * kWinStride];
    __shared__ __align__(16) uint8_t s_tile[kU8 ? kTileH * kTileW : 16];
    extern __shared__ uint8_t s_dynbits[];   // T bytes

    const int tid = threadIdx.x;
    const int K = p.K, T = p.T;
    const bool aligned = kU8 && (reinterpret_cast<uintptr_t>(p.img) % 16 == 0) && (p.pitch % 16 == 0);

    for (unsigned long long kp = blockIdx.x; kp < p.M; kp += gridDim.x) {
        const double x = __ldg(p.xycs + 4 * kp + 0);
        const double y = __ldg(p.xycs + 4 * kp + 1);
        const double c = __ldg(p.xycs + 4 * kp + 2);
        const double s = __ldg(p.xycs + 4 * kp + 3);
        int ax0 = 0, ty0 = 0;
        if (kU8) {
            const int tx0 = __double2int_rd(x) - 45;
            ty0 = __double2int_rd(y) - 45;
            ax0 = aligned ? (tx0 & ~15) : tx0;
            stage_tile_u8(s_tile, static_cast<const uint8_t*>(p.img), p.pitch, p.height, ax0, ty0,
                          aligned);
        }
        __syncthreads();
        build_window<kU8>(s_win, s_tile, ax0, ty0, static_cast<const double*>(p.img), p.pitch, x, y,
                          c, s);
        __syncthreads();
        for (int t = tid; t < T; t += kThreads) {
            const short* tr = p.triplets + 6 * t;
            const double* pa = s_win + tr[1] * kWinStride + tr[0];
            const double* pb = s_win + tr[3] * kWinStride + tr[2];
            const double* pc = s_win + tr[5] * kWinStride + tr[4];
            double d1 = 0.0, d2 = 0.0;
            for (int r = 0; r < K; ++r) {
                for (int col = 0; col < K; ++col) {
                    const double w = __ldg(p.weights + r * K + col);
                    const double a = pa[col];
                    const double e1 = __dsub_rn(a, pb[col]);
                    const double e2 = __dsub_rn(a, pc[col]);
                    d1 = __dadd_rn(d1, __dmul_rn(__dmul_rn(w, e1), e1));
                    d2 = __dadd_rn(d2, __dmul_rn(__dmul_rn(w, e2), e2));
                }
                pa += kWinStride;
                pb += kWinStride;
                pc += kWinStride;
            }
            s_dynbits[t] = d1 > d2;
        }
        __syncthreads();
        for (int b = tid; b < T / 8; b += kThreads) {
            unsigned byte = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) byte |= (s_dynbits[8 * b + i] ? 1u : 0u) << i;
            const unsigned long long row = p.out_index ? p.out_index[kp] : kp;
            p.out[row * (T / 8) + b] = static_cast<uint8_t>(byte);
        }
    }
}

// f64 -> u8 promotion: flags[0] = 0 while every pixel seen is an integer in [0, 255]; 1 once some pixel
// is not; 2 once some pixel is NaN, infinite or beyond 2^1000 in magnitude. dst receives the (lossless
// when flags[0]==0) u8 copy. Class 2 matters because the specialised kernels skip the mask's zero-weight
// pixels, which is exact only while every patch difference e is finite (0*e*e = 0): the reference
// multiplies them in (src/descriptor.cpp:66-71), so one NaN or an overflowing a - b under a masked
// pixel poisons its sum. Such images take the generic kernel, which evaluates (w*e)*e literally.
// Rows [row0, row1) only, so an image that arrives in row bands can be classified band by band;
// the flag accumulates ("some pixel seen so far is not a u8 value").
// The flag block (64 bytes): int flags[0] as above; at byte 8 two u64 keys, the smallest and the largest pixel seen as
// order-preserving integers; at byte 24 two doubles {lo, 1 / (hi - lo)} written by range_finalize_kernel.
__host__ __device__ __forceinline__ unsigned long long* flag_keys(int* flags) { return reinterpret_cast<unsigned long long*>(flags + 2); }
__host__ __device__ __forceinline__ double* flag_range(int* flags) { return reinterpret_cast<double*>(flags + 6); }
__device__ __forceinline__ unsigned long long ordered_key(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ordered_value(unsigned long long k) {
    return __longlong_as_double(static_cast<long long>((k >> 63) ? (k ^ 0x8000000000000000ull) : ~k));
}

__global__ void classify_convert_kernel(const double* src, size_t src_pitch, uint8_t* dst,
                                        size_t dst_pitch, int width, int row0, int row1, int* flags) {
    const size_t n = static_cast<size_t>(width) * (row1 - row0);
    int cls = 0;
    double lo = 1.0e308, hi = -1.0e308;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int yy = row0 + static_cast<int>(i / width), xx = static_cast<int>(i % width);
        const double v = src[static_cast<size_t>(yy) * src_pitch + xx];
        const bool ok = (v >= 0.0) && (v <= 255.0) && (v == floor(v));   // NaN/inf fail
        const bool tame = fabs(v) <= 0x1p1000;                            // NaN fails
        cls = max(cls, tame ? (ok ? 0 : 1) : 2);
        dst[static_cast<size_t>(yy) * dst_pitch + xx] = ok ? static_cast<uint8_t>(v) : 0;
        lo = fmin(lo, v);   // (NaN is ignored by fmin / fmax; such an image is class 2 anyway)
        hi = fmax(hi, v);
    }
    cls = __reduce_max_sync(0xffffffffu, cls);
    if (cls != 0 && (threadIdx.x & 31) == 0) atomicMax(flags, cls);
    // the range of ALL pixels (it only matters to the non-u8 route, but which route that is is not known yet)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(flag_keys(flags) + 0, ordered_key(lo));
        atomicMax(flag_keys(flags) + 1, ordered_key(hi));
    }
}

// After the WHOLE image has been classified as "tame, not u8-valued" (flags[0] == 1): if its range is usable —
// 2^-400 <= hi - lo <= 2^400, and no pixel further than 2^20 ranges from zero, so that the reference's own fp64
// roundings (relative to the pixel values) stay below 1e-4 stored units — publish {lo, 1 / (hi - lo)} and move the image to class 3, the
// packed-plane kernel's float64 route. Anything else stays with extract_quad_kernel<false>.
__global__ void range_finalize_kernel(int* flags) {
    if (flags[0] != 1) return;
    const double lo = ordered_value(flag_keys(flags)[0]), hi = ordered_value(flag_keys(flags)[1]);
    // 2^-400 <= r <= 2^400: a squared difference neither overflows nor reaches the denormals in the reference's sums (an
    // image of values around 1e-290 has every bit 0 there: all its squares underflow, which a scale-free estimate cannot see)
    const double r = hi - lo, inv = 1.0 / r;
    if (r >= 0x1p-400 && r <= 0x1p400 && fmax(fabs(lo), fabs(hi)) <= r * 1048576.0) {
        flag_range(flags)[0] = lo;
        flag_range(flags)[1] = inv;
        __threadfence();
        flags[0] = 3;
    }
}

// float64 image -> float CUDA array of (v - lo) / (hi - lo), 4 pixels per thread (class 3 images only).
__global__ void fill_array_f32_kernel(cudaSurfaceObject_t surf, const double* __restrict__ src, size_t pitch, int w, int h,
                                      const int* flags, int run_if_flag) {
    pdl_launch_dependents();
    if (flags[0] != run_if_flag) return;
    const double lo = flag_range(const_cast<int*>(flags))[0], inv = flag_range(const_cast<int*>(flags))[1];
    const int x = (blockIdx.x * blockDim.x + threadIdx.x) * 4, y = blockIdx.y;
    if (x >= w || y >= h) return;
    const double* row = src + static_cast<size_t>(y) * pitch;
    for (int i = x; i < min(w, x + 4); ++i)
        surf2Dwrite(static_cast<float>((row[i] - lo) * inv), surf, i * 4, y);
}

int grid_for(const clatch_ctx* ctx, size_t M, int ctas_per_sm) {
    const size_t cap = static_cast<size_t>(ctx->sm_count) * ctas_per_sm;
    return static_cast<int>(M < cap ? M : cap);
}

// Pitch-linear u8 image -> CUDA array through a surface, 16 pixels per thread (4.6 us for 1920x1080,
// 6.6 us for 3840x2160; cudaMemcpy2DToArrayAsync takes 8.4 / 21 us — tools/tex_probe.cu).
__global__ void fill_array_kernel(cudaSurfaceObject_t surf, const uint8_t* __restrict__ src, size_t pitch, int w, int h,
                                  bool aligned, const int* flags, int run_if_flag) {
    pdl_launch_dependents();   // the extraction kernel's CTAs may load their tables while the array is being filled
    if (flags != nullptr && flags[0] != run_if_flag) return;
    const int x = (blockIdx.x * blockDim.x + threadIdx.x) * 16, y = blockIdx.y;
    if (x >= w || y >= h) return;
    const uint8_t* row = src + static_cast<size_t>(y) * pitch;
    if (aligned && x + 16 <= w) {
        surf2Dwrite(__ldg(reinterpret_cast<const uint4*>(row + x)), surf, x, y);
    } else {
        for (int i = x; i < min(w, x + 16); ++i) surf2Dwrite(row[i], surf, i, y);
    }
}

// One gather-enabled u8 CUDA array + texture object per stream that launches the pipelined
// kernel, re-created when the image size changes.
int tex_image_for(clatch_ctx* ctx, cudaStream_t stream, int width, int height, clatch_ctx::TexImage** out) {
    clatch_ctx::TexImage* ti = nullptr;
    for (auto& t : ctx->tex_images)
        if (t.stream == stream) ti = &t;
    if (!ti) {
        ctx->tex_images.push_back({});
        ti = &ctx->tex_images.back();
        ti->stream = stream;
    }
    if (!ti->tickets) {
        CLATCH_CUDA(cudaMalloc(&ti->tickets, 2 * sizeof(unsigned)));
        CLATCH_CUDA(cudaMemsetAsync(ti->tickets, 0, 2 * sizeof(unsigned), stream));
    }
    if (ti->width != width || ti->height != height) {
        if (ti->tex) {
            CLATCH_CUDA(cudaStreamSynchronize(stream));   // a kernel may still be sampling the old array
            cudaDestroyTextureObject(ti->tex);
            cudaDestroyTextureObject(ti->texn);
            cudaDestroySurfaceObject(ti->surf);
            cudaFreeArray(ti->array);
            ti->tex = 0;
            ti->texn = 0;
            ti->surf = 0;
            ti->array = nullptr;
            ti->width = ti->height = 0;
        }
        const cudaChannelFormatDesc fmt = cudaCreateChannelDesc<unsigned char>();
        CLATCH_CUDA(cudaMallocArray(&ti->array, &fmt, width, height, cudaArrayTextureGather | cudaArraySurfaceLoadStore));
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = ti->array;
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        CLATCH_CUDA(cudaCreateTextureObject(&ti->tex, &rd, &td, nullptr));
        td.readMode = cudaReadModeNormalizedFloat;   // the packed-plane kernel's resampler: texel / 255 as a float
        CLATCH_CUDA(cudaCreateTextureObject(&ti->texn, &rd, &td, nullptr));
        CLATCH_CUDA(cudaCreateSurfaceObject(&ti->surf, &rd));
        ti->width = width;
        ti->height = height;
    }
    *out = ti;
    return CLATCH_OK;
}

// The float companion of a stream's texture image (class 3 float64 images): a gather-enabled float array.
int tex_image_f32_for(clatch_ctx* ctx, clatch_ctx::TexImage* ti, cudaStream_t stream, int width, int height) {
    if (ti->widthf != width || ti->heightf != height) {
        if (ti->texf) {
            CLATCH_CUDA(cudaStreamSynchronize(stream));   // a kernel may still be sampling the old array
            cudaDestroyTextureObject(ti->texf);
            cudaDestroySurfaceObject(ti->surff);
            cudaFreeArray(ti->arrayf);
            ti->texf = 0;
            ti->surff = 0;
            ti->arrayf = nullptr;
            ti->widthf = ti->heightf = 0;
        }
        const cudaChannelFormatDesc fmt = cudaCreateChannelDesc<float>();
        CLATCH_CUDA(cudaMallocArray(&ti->arrayf, &fmt, width, height, cudaArrayTextureGather | cudaArraySurfaceLoadStore));
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = ti->arrayf;
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        CLATCH_CUDA(cudaCreateTextureObject(&ti->texf, &rd, &td, nullptr));
        CLATCH_CUDA(cudaCreateSurfaceObject(&ti->surff, &rd));
        ti->widthf = width;
        ti->heightf = height;
    }
    return CLATCH_OK;
}

// The single-window kernel's placement (16 triplets per half-warp, one million annealing steps)
// is only needed when extract_variant 0 is selected: plan it on first use.
int ensure_single_window_plan(clatch_ctx* ctx) {
    Pattern& pat = ctx->pattern;
    if (pat.slots_planned) return CLATCH_OK;
    const SlotPlan plan = plan_slots(pat.host_triplets.data(), pat.T, kWinStride, 1000000);
    pat.slot_degree = plan.avg_degree;
    pat.slot_degree_identity = plan.avg_degree_identity;
    static_assert(sizeof(SlotEntry) == sizeof(ushort4), "slot layout");
    if (int rc = pat.slots.reserve(sizeof(SlotEntry) * pat.T)) return rc;
    CLATCH_CUDA(cudaMemcpy(pat.slots.ptr, plan.slots.data(), sizeof(SlotEntry) * pat.T, cudaMemcpyHostToDevice));
    pat.slots_planned = true;
    return CLATCH_OK;
}

// The fp32-plane kernels' placement (variants 2-4) for a table other than the built-in one: planned on first use.
int ensure_f8_plan(clatch_ctx* ctx) {
    Pattern& pat = ctx->pattern;
    if (pat.slots_f8_planned) return CLATCH_OK;
    const SlotPlan f8 = plan_slots_grouped(pat.host_triplets.data(), pat.T, kWinStride, 8, 8, 1500000);
    pat.slot_degree_f8 = f8.avg_degree;
    if (int rc = pat.slots_f8.reserve(sizeof(SlotEntry) * pat.T)) return rc;
    CLATCH_CUDA(cudaMemcpy(pat.slots_f8.ptr, f8.slots.data(), sizeof(SlotEntry) * pat.T, cudaMemcpyHostToDevice));
    pat.slots_f8_planned = true;
    return CLATCH_OK;
}

// CLATCH_EX_TRACE=1: where one launch of the default kernel spends its time (stamps of extract_roles_kernel).
void print_extract_trace(const std::vector<unsigned long long>& h, int grid, size_t quads) {
    const unsigned long long kFlag = 1ull << 63;
    unsigned long long t0 = ~0ull, t_end = 0;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[static_cast<size_t>(kExTrace) * c]);
    double entry_max = 0, ready_mean = 0, ready_max = 0, fill_mean = 0, drain_mean = 0, end_mean = 0, end_min = 1e30;
    double steady_sum = 0, exact_sum = 0;
    size_t steady_n = 0, exact_n = 0, parked = 0, parked_ctas = 0;
    double parked_us = 0;
    std::vector<double> ends(grid);
    std::vector<int> exacts(grid, 0);
    std::vector<long long> taken(grid, 0);
    for (int c = 0; c < grid; ++c) {
        const unsigned long long* t = h.data() + static_cast<size_t>(kExTrace) * c;
        const long long nq = t[kExTrace - 2] ? static_cast<long long>(t[kExTrace - 2])   // (quads drawn from the ticket counter)
                                             : static_cast<long long>((quads - c + grid - 1) / grid);
        const long long last = std::min<long long>(nq + 3, kExTrace - 1);   // stamp index of iteration nq
        entry_max = std::max(entry_max, (t[0] - t0) * 1e-3);
        ready_mean += (t[1] - t0) * 1e-3;
        ready_max = std::max(ready_max, (t[1] - t0) * 1e-3);
        fill_mean += ((t[2] & ~kFlag) - t[1]) * 1e-3;
        for (long long i = 3; i < last; ++i) {   // iterations 0 .. nq-1
            const double d = ((t[i] & ~kFlag) - (t[i - 1] & ~kFlag)) * 1e-3;
            if (t[i] & kFlag) {
                exact_sum += d;
                ++exact_n;
                ++exacts[c];
            } else if (i + 1 < last) {
                steady_sum += d;
                ++steady_n;
            } else {
                drain_mean += d;
            }
        }
        double e = ((t[last] & ~kFlag) - t0) * 1e-3;
        if (t[kExTrace - 1]) {   // parked bits recomputed after the pipeline drained
            parked += t[kExTrace - 1] >> 48;
            const double after = ((t[kExTrace - 1] & 0xffffffffffffull) - (t0 & 0xffffffffffffull)) * 1e-3;
            parked_us += after - e;
            ++parked_ctas;
            e = after;
            t_end = std::max(t_end, (t0 & ~0xffffffffffffull) | (t[kExTrace - 1] & 0xffffffffffffull));
        }
        ends[c] = e;
        taken[c] = nq;
        end_mean += e;
        end_min = std::min(end_min, e);
        t_end = std::max(t_end, t[last] & ~kFlag);
    }
    int worst = 0;
    for (int c = 0; c < grid; ++c)
        if (ends[c] > ends[worst]) worst = c;
    std::fprintf(stderr,
                 "[clatch ex trace] ctas=%d quads=%zu span %.1f us | entry max %.1f, texture ready mean %.1f max %.1f, first resample %.1f, "
                 "steady iteration %.2f (n=%zu), iteration with an exact pass %.2f (n=%zu), last estimate %.2f | CTA end mean %.1f min %.1f "
                 "max %.1f (cta %d: %d exact passes, %lld quads) | parked bits %zu in %zu CTAs, %.2f us per such CTA\n",
                 grid, quads, (t_end - t0) * 1e-3, entry_max, ready_mean / grid, ready_max, fill_mean / grid,
                 steady_n ? steady_sum / steady_n : 0.0, steady_n, exact_n ? exact_sum / exact_n : 0.0, exact_n, drain_mean / grid,
                 end_mean / grid, end_min, ends[worst], worst, exacts[worst],
                 taken[worst], parked, parked_ctas,
                 parked_ctas ? parked_us / parked_ctas : 0.0);
}

template <bool kU8>
int launch_extract(clatch_ctx* ctx, const void* d_img, int width, int height, size_t pitch,
                   const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream,
                   const int* flags, int run_if_flag, bool force_generic = false) {
    const Pattern& pat = ctx->pattern;
    ExtractParams p{};
    p.img = d_img;
    p.width = width;
    p.height = height;
    p.pitch = pitch;
    p.xycs = d_xycs;
    p.M = M;
    p.out = d_out;
    p.slots = pat.slots.as<ushort4>();
    p.triplets = pat.triplets.as<short>();
    p.weights = pat.d_weights.as<double>();
    p.T = pat.T;
    p.K = pat.K;
    p.flags = flags;
    p.run_if_flag = run_if_flag;
    p.stats = ctx->extract_stats_on ? ctx->extract_stats.as<unsigned long long>() : nullptr;
    p.out_index = ctx->extract_out_index;   // honoured by the quad and pipelined kernels (extract_supports_out_index)
    // Degenerate input (flat or saturated regions: exact ties, which the fp32 estimate can never decide) makes the
    // estimate-based kernels pay the estimate, a re-resampling and the exact chains — 23 M desc/s on a flat image
    // against 36 M for the all-fp64 quad kernel. The default kernel reports, per launch, how many windows took the
    // exact pass (ExtractParams::route, a host-mapped slot per CTA); when the previous launch of this context saw
    // more than 25 % (35 % for the fp32-plane kernel) the next ones run the quad kernel; the default kernel probes again after
    // 16 launches, then 32, 64, 128 while the probes keep finding the stream degenerate.
    bool quad_routed = false;
    const bool routing = kU8 && pat.fast && ctx->extract_variant >= 4 && ctx->extract_route && !ctx->extract_stats_on &&
                         flags == nullptr && ctx->route_host != nullptr && !force_generic;
    if (routing) {
        if (ctx->route_pending) {   // fold the last probe's slots (its kernel may still be running: then they read 0 / stale, harmless)
            unsigned long long hot = 0, all = 0;
            for (int c = 0; c < ctx->sm_count; ++c) {
                hot += ctx->route_host[c].x;
                all += ctx->route_host[c].y;
            }
            if (all > 0) {
                // measured break-even against the quad kernel (tools/route_perf.py: 36 M desc/s whatever the image): the
                // packed-plane kernel with ticketed quads falls below it at 25 % of the windows in the window-wide pass
                // (18 % for its symmetric, statically scheduled form), the fp32-plane kernel at 35 %
                const bool was = ctx->route_quad;
                ctx->route_quad = hot * 100 > all * (ctx->extract_variant == 5 ? 25u : ctx->extract_variant == 6 ? 18u : 35u);
                ctx->route_pending = false;
                // every probe of a degenerate stream costs a launch at half the quad kernel's rate: the first one comes
                // after 16 launches, each confirming one doubles the distance (up to 128: a flat stream then runs at
                // 36 M desc/s, 34 M with a probe every 16th launch), the first clean one ends the routing
                ctx->route_period = ctx->route_quad && was ? std::min(ctx->route_period * 2, 128u) : 16u;
                if (ctx->route_quad) ctx->route_probe_at = ctx->route_age + ctx->route_period;
            }
        }
        ++ctx->route_age;
        if (ctx->route_quad) {
            if (ctx->route_age != ctx->route_probe_at) quad_routed = true;
            else ctx->route_probe_at += ctx->route_period;   // (this launch probes; its answer is folded a launch or more later)
        }
    }
    if (force_generic) {
        extract_generic_kernel<kU8><<<grid_for(ctx, M, 2), kThreads, pat.T, stream>>>(p);
    } else if (quad_routed) {
        if (!ctx->quad_configured) {   // per-device function attribute
            CLATCH_CUDA(cudaFuncSetAttribute(extract_quad_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kQuadSmemBytes));
            CLATCH_CUDA(cudaFuncSetAttribute(extract_quad_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kQuadSmemBytes));
            ctx->quad_configured = true;
        }
        p.slots = pat.slots_quad.as<ushort4>();
        const size_t quads = (M + kQuad - 1) / kQuad;
        const int grid = static_cast<int>(std::min<size_t>(quads, ctx->sm_count));
        extract_quad_kernel<kU8><<<grid, kQuadThreads, kQuadSmemBytes, stream>>>(p);
    } else if (kU8 && pat.fast && ctx->extract_variant >= 3) {
        if (!ctx->pipe_configured) {   // per-device function attribute
            CLATCH_CUDA(cudaFuncSetAttribute(extract_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kPipeSmemBytes));
            CLATCH_CUDA(cudaFuncSetAttribute(extract_roles_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kRolesSmemBytes));
            CLATCH_CUDA(cudaFuncSetAttribute(extract_h16_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kH16SmemBytes));
            CLATCH_CUDA(cudaFuncSetAttribute(extract_h16_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kH16SmemBytes));
            CLATCH_CUDA(cudaFuncSetAttribute(extract_h16s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kH16SmemBytes));
            ctx->pipe_configured = true;
        }
        // The resampler reads footprints through the texture unit: copy the image into this
        // stream's gather-enabled CUDA array (a surface-write kernel, stream-ordered).
        clatch_ctx::TexImage* ti = nullptr;
        if (int rc = tex_image_for(ctx, stream, width, height, &ti)) return rc;
        {
            const bool al = reinterpret_cast<uintptr_t>(d_img) % 16 == 0 && pitch % 16 == 0;
            const dim3 fgrid((width / 16 + 1 + 127) / 128, height);
            fill_array_kernel<<<fgrid, 128, 0, stream>>>(ti->surf, static_cast<const uint8_t*>(d_img), pitch, width, height,
                                                         al, flags, run_if_flag);
            ++ctx->launches;
        }
        p.tex = ti->tex;
        p.texn = ti->texn;
        p.two23 = 0x4B000000u;
        if (ctx->extract_variant == 5) {
            if (int rc = ensure_single_window_plan(ctx)) return rc;
            p.slots_sw = pat.slots.as<ushort4>();
            static const bool static_quads = std::getenv("CLATCH_EX_STATIC") != nullptr;   // diagnostics: round-robin quads
            p.tickets = static_quads ? nullptr : ti->tickets;
        }
        static const int ex_debug = std::getenv("CLATCH_EX_DEBUG") ? std::atoi(std::getenv("CLATCH_EX_DEBUG")) : 0;
        p.dbg = ex_debug;
        if (ctx->extract_variant < 5)
            if (int rc = ensure_f8_plan(ctx)) return rc;
        p.slots = ctx->extract_variant >= 5 ? pat.slots_h16.as<ushort4>() : pat.slots_f8.as<ushort4>();
        const size_t quads = (M + kQuad - 1) / kQuad;
        const int grid = static_cast<int>(std::min<size_t>(quads, ctx->sm_count));
        // variant 4 (default): dedicated producer / consumer warps, 16 + 16 — 60.1 vs 58.1 M desc/s at 10 k
        // keypoints and 72.3 vs 68.3 M at 50 k against the symmetric schedule of variant 3 (24 + 8 warps
        // measured 48.8 M: eight warps cannot keep the LSU busy)
        // a probe: every default-kernel launch while the stream is degenerate (the 16th, then 32nd, 64th, 128th ones), every 8th one otherwise — the
        // store into host memory at the end of the kernel costs ~2 us per launch
        if (routing && M >= 64 && (ctx->route_quad || (ctx->route_age & 7) == 1)) {
            std::memset(ctx->route_host, 0, sizeof(uint2) * ctx->sm_count);
            p.route = ctx->route_dev;
            ctx->route_pending = true;
        }
        static const bool tracing = std::getenv("CLATCH_EX_TRACE") != nullptr;
        unsigned long long* d_trace = nullptr;
        if (tracing && ctx->extract_variant >= 4) {   // diagnostics: per-CTA timeline of the launch (synchronises)
            CLATCH_CUDA(cudaMalloc(&d_trace, sizeof(unsigned long long) * kExTrace * grid));
            CLATCH_CUDA(cudaMemsetAsync(d_trace, 0, sizeof(unsigned long long) * kExTrace * grid, stream));
            p.trace = d_trace;
        }
        if (ctx->extract_variant == 6)   // packed 16-bit planes, every warp resamples and estimates
            CLATCH_CUDA(launch_kernel(extract_h16s_kernel, dim3(grid), dim3(kQuadThreads), kH16SmemBytes, stream, ctx->pdl, 1, p));
        else if (ctx->extract_variant == 5)   // packed 16-bit planes, fp32 resampling, dedicated roles
            CLATCH_CUDA(launch_kernel(extract_h16_kernel<16, false>, dim3(grid), dim3(kQuadThreads), kH16SmemBytes, stream, ctx->pdl, 1, p));
        else if (ctx->extract_variant == 4)   // may start (tables, first keypoint rows) while fill_array_kernel is still writing
            CLATCH_CUDA(launch_kernel(extract_roles_kernel<16>, dim3(grid), dim3(kQuadThreads), kRolesSmemBytes, stream, ctx->pdl, 1, p));
        else extract_pipe_kernel<<<grid, kQuadThreads, kPipeSmemBytes, stream>>>(p);
        if (d_trace) {
            std::vector<unsigned long long> h(static_cast<size_t>(kExTrace) * grid);
            CLATCH_CUDA(cudaStreamSynchronize(stream));
            CLATCH_CUDA(cudaMemcpy(h.data(), d_trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
            cudaFree(d_trace);
            print_extract_trace(h, grid, quads);
        }
    } else if (kU8 && pat.fast && ctx->extract_variant == 2) {
        if (!ctx->filt_configured) {   // per-device function attribute
            CLATCH_CUDA(cudaFuncSetAttribute(extract_filt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kFiltSmemBytes));
            ctx->filt_configured = true;
        }
        if (int rc = ensure_f8_plan(ctx)) return rc;
        p.slots = pat.slots_f8.as<ushort4>();
        const size_t quads = (M + kQuad - 1) / kQuad;
        const int grid = static_cast<int>(std::min<size_t>(quads, ctx->sm_count));
        extract_filt_kernel<<<grid, kQuadThreads, kFiltSmemBytes, stream>>>(p);
    } else if (pat.fast && ctx->extract_variant >= 1) {   // (variants 2 and 3 are u8-only: other images land here)
        if (!ctx->quad_configured) {   // per-device function attribute
            CLATCH_CUDA(cudaFuncSetAttribute(extract_quad_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kQuadSmemBytes));
            CLATCH_CUDA(cudaFuncSetAttribute(extract_quad_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kQuadSmemBytes));
            ctx->quad_configured = true;
        }
        p.slots = pat.slots_quad.as<ushort4>();
        const size_t quads = (M + kQuad - 1) / kQuad;
        const int grid = static_cast<int>(std::min<size_t>(quads, ctx->sm_count));
        extract_quad_kernel<kU8><<<grid, kQuadThreads, kQuadSmemBytes, stream>>>(p);
    } else if (pat.fast) {
        if (int rc = ensure_single_window_plan(ctx)) return rc;
        p.slots = pat.slots.as<ushort4>();
        extract_fast_kernel<kU8><<<grid_for(ctx, M, 4), kThreads, 0, stream>>>(p);
    } else {
        extract_generic_kernel<kU8><<<grid_for(ctx, M, 2), kThreads, pat.T, stream>>>(p);
    }
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

} // namespace

// Scattered output rows (ExtractParams::out_index) are implemented by the kernels that the banded
// float64 upload can reach: the pipelined kernel (u8-valued image) and the quad kernel (any other).
bool extract_supports_out_index(const clatch_ctx* ctx) {
    return ctx->pattern.fast && ctx->extract_variant >= 3;
}

int launch_estimate_planes_u8(clatch_ctx* ctx, const uint8_t* d_img, int width, int height, size_t pitch,
                              const double* d_xycs, size_t M, uint16_t* d_out, cudaStream_t stream) {
    if (M == 0) return CLATCH_OK;
    constexpr int kSmem = kQuad * kHPitch * 4 + kQuad * kHRecDoubles * 8;
    CLATCH_CUDA(cudaFuncSetAttribute(h16_planes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    clatch_ctx::TexImage* ti = nullptr;
    if (int rc = tex_image_for(ctx, stream, width, height, &ti)) return rc;
    const bool al = reinterpret_cast<uintptr_t>(d_img) % 16 == 0 && pitch % 16 == 0;
    const dim3 fgrid((width / 16 + 1 + 127) / 128, height);
    fill_array_kernel<<<fgrid, 128, 0, stream>>>(ti->surf, d_img, pitch, width, height, al, nullptr, 0);
    ExtractParams p{};
    p.img = d_img;
    p.width = width;
    p.height = height;
    p.pitch = pitch;
    p.xycs = d_xycs;
    p.M = M;
    p.texn = ti->texn;
    const size_t quads = (M + kQuad - 1) / kQuad;
    h16_planes_kernel<<<static_cast<unsigned>(std::min<size_t>(quads, ctx->sm_count)), 512, kSmem, stream>>>(
        p, reinterpret_cast<unsigned short*>(d_out));
    ctx->launches += 2;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

int launch_extract_u8(clatch_ctx* ctx, const uint8_t* d_img, int width, int height, size_t pitch,
                      const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream) {
    if (M == 0) return CLATCH_OK;
    return launch_extract<true>(ctx, d_img, width, height, pitch, d_xycs, M, d_out, stream, nullptr, 0);
}

// f64 images are promoted to u8 on the device when every pixel is an integer in [0,255] (true
// for every PGM-sourced image, src/image.cpp:75-76). Classification and extraction are
// separate steps so that a banded upload can interleave them: classify the rows that have
// arrived, then extract the keypoints whose footprints lie inside them. Both extraction
// kernels are queued and the device flag picks one — no host round trip.
int launch_classify_rows(clatch_ctx* ctx, const double* d_img, int width, int height, size_t pitch, int row0,
                         int row1, bool reset, cudaStream_t stream) {
    const size_t u8_pitch = (static_cast<size_t>(width) + 15) / 16 * 16;
    if (int rc = ctx->img_u8.reserve(u8_pitch * height)) return rc;
    if (int rc = ctx->flags.reserve(kFlagBlockBytes)) return rc;
    int* flags = ctx->flags.as<int>();
    if (reset) {
        if (int rc = scratch_acquire(ctx, stream)) return rc;   // img_u8 / flags may still be read on another stream
        CLATCH_CUDA(cudaMemsetAsync(flags, 0, kFlagBlockBytes, stream));
        CLATCH_CUDA(cudaMemsetAsync(flag_keys(flags), 0xFF, sizeof(unsigned long long), stream));   // the running minimum
    }
    if (row1 <= row0) return CLATCH_OK;
    classify_convert_kernel<<<ctx->sm_count * 8, 256, 0, stream>>>(d_img, pitch, ctx->img_u8.as<uint8_t>(), u8_pitch,
                                                                   width, row0, row1, flags);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

// Class 3 (launch_extract_f64_classified, whole images): the packed-plane kernel over a float texture of the image.
static int launch_extract_h16_f64(clatch_ctx* ctx, const double* d_img, int width, int height, size_t pitch,
                                  const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream, int* flags) {
    const Pattern& pat = ctx->pattern;
    if (!ctx->pipe_configured) {   // per-device function attributes
        CLATCH_CUDA(cudaFuncSetAttribute(extract_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPipeSmemBytes));
        CLATCH_CUDA(cudaFuncSetAttribute(extract_roles_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRolesSmemBytes));
        CLATCH_CUDA(cudaFuncSetAttribute(extract_h16_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kH16SmemBytes));
        CLATCH_CUDA(cudaFuncSetAttribute(extract_h16_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kH16SmemBytes));
        CLATCH_CUDA(cudaFuncSetAttribute(extract_h16s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kH16SmemBytes));
        ctx->pipe_configured = true;
    }
    clatch_ctx::TexImage* ti = nullptr;
    if (int rc = tex_image_for(ctx, stream, width, height, &ti)) return rc;
    if (int rc = tex_image_f32_for(ctx, ti, stream, width, height)) return rc;
    range_finalize_kernel<<<1, 1, 0, stream>>>(flags);
    const dim3 fgrid((width / 4 + 1 + 127) / 128, height);
    fill_array_f32_kernel<<<fgrid, 128, 0, stream>>>(ti->surff, d_img, pitch, width, height, flags, 3);
    ctx->launches += 2;
    ExtractParams p{};
    p.img = d_img;
    p.width = width;
    p.height = height;
    p.pitch = pitch;
    p.xycs = d_xycs;
    p.M = M;
    p.out = d_out;
    p.slots = pat.slots_h16.as<ushort4>();
    p.T = pat.T;
    p.K = pat.K;
    p.flags = flags;
    p.run_if_flag = 3;
    p.stats = ctx->extract_stats_on ? ctx->extract_stats.as<unsigned long long>() : nullptr;
    p.out_index = ctx->extract_out_index;
    p.tex = 0;
    p.texn = ti->texf;
    p.two23 = 0x4B000000u;
    if (int rc = ensure_single_window_plan(ctx)) return rc;
    p.slots_sw = pat.slots.as<ushort4>();
    p.tickets = ti->tickets;
    const size_t quads = (M + kQuad - 1) / kQuad;
    const int grid = static_cast<int>(std::min<size_t>(quads, ctx->sm_count));
    CLATCH_CUDA(launch_kernel(extract_h16_kernel<16, true>, dim3(grid), dim3(kQuadThreads), kH16SmemBytes, stream, ctx->pdl, 1, p));
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

int launch_extract_f64_classified(clatch_ctx* ctx, const double* d_img, int width, int height, size_t pitch,
                                  const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream, bool whole_image) {
    if (M == 0) return CLATCH_OK;
    const size_t u8_pitch = (static_cast<size_t>(width) + 15) / 16 * 16;
    int* flags = ctx->flags.as<int>();
    if (int rc = launch_extract<true>(ctx, ctx->img_u8.ptr, width, height, u8_pitch, d_xycs, M, d_out,
                                      stream, flags, 0))
        return rc;
    // tame but not u8-valued, every row classified, a usable range: class 1 becomes class 3 and takes the packed-plane
    // kernel (extract_f64_h16, on by default with extract_variant 5); otherwise the all-fp64 quad kernel below runs
    if (whole_image && ctx->pattern.fast && ctx->extract_variant == 5 && ctx->extract_f64_h16)
        if (int rc = launch_extract_h16_f64(ctx, d_img, width, height, pitch, d_xycs, M, d_out, stream, flags)) return rc;
    if (int rc = launch_extract<false>(ctx, d_img, width, height, pitch, d_xycs, M, d_out, stream, flags, 1)) return rc;
    // class 2 (non-finite or huge pixels): the literal (w*e)*e kernel, whatever the pattern
    if (int rc = launch_extract<false>(ctx, d_img, width, height, pitch, d_xycs, M, d_out, stream, flags, 2, true)) return rc;
    return scratch_release(ctx, stream);
}

int launch_extract_f64(clatch_ctx* ctx, const double* d_img, int width, int height, size_t pitch,
                       const double* d_xycs, size_t M, uint8_t* d_out, cudaStream_t stream) {
    if (M == 0) return CLATCH_OK;
    if (int rc = launch_classify_rows(ctx, d_img, width, height, pitch, 0, height, true, stream)) return rc;
    return launch_extract_f64_classified(ctx, d_img, width, height, pitch, d_xycs, M, d_out, stream, true);
}

} // namespace clatch
