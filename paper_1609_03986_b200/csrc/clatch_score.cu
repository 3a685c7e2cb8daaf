// Trainer scoring loop for sm_100a ("next" row 4 of SURVEY.md §8f): the bit of every
// candidate triplet on every upright 64x64 training patch — triplet_bits_over,
// src/pattern.cpp:340-346, the parallel body of select_triplets (:397-400). Same arithmetic
// as extraction's SSD phase (triplet_bit, src/descriptor.cpp:51-77: two sequential
// (w*e)*e chains, strict >) with the patch itself as the window (Window64::from_image,
// src/descriptor.cpp:13-21) — no resampling.
//
// score_kernel: persistent CTAs, one patch per iteration: 4096 doubles -> padded shared
// window; each thread evaluates candidates tid, tid+256, ...; a warp's 32 predicates leave as
// one ballot word -> bits[patch][candidate] (row-major by patch). transpose_kernel then turns
// 32x32 bit blocks with ballots into the reference's BitVector orientation
// bits[candidate][patch] (LSB-first).

#include "clatch_internal.cuh"

namespace clatch {

namespace {

constexpr int kScoreThreads = 256;

__constant__ double c_score_weights[kMaxConstWeights];

__global__ void __launch_bounds__(kScoreThreads) score_kernel(const double* __restrict__ windows, unsigned n,
                                                              const short* __restrict__ candidates, unsigned C,
                                                              int K, unsigned words_per_patch,
                                                              unsigned* __restrict__ bits) {
    __shared__ __align__(16) double s_win[kWindow * kWinStride];
    const unsigned c_padded = words_per_patch * 32;
    for (unsigned patch = blockIdx.x; patch < n; patch += gridDim.x) {
        const double* src = windows + static_cast<size_t>(patch) * (kWindow * kWindow);
        __syncthreads();   // previous patch's readers are done
        for (int i = threadIdx.x; i < kWindow * kWindow; i += kScoreThreads)
            s_win[(i >> 6) * kWinStride + (i & 63)] = __ldg(src + i);
        __syncthreads();
        for (unsigned c = threadIdx.x; c < c_padded; c += kScoreThreads) {   // warp-uniform trip count
            bool bit = false;
            if (c < C) {
                const short* tr = candidates + 6 * static_cast<size_t>(c);
                const double* pa = s_win + tr[1] * kWinStride + tr[0];
                const double* pb = s_win + tr[3] * kWinStride + tr[2];
                const double* pc = s_win + tr[5] * kWinStride + tr[4];
                double d1 = 0.0, d2 = 0.0;
                for (int r = 0; r < K; ++r) {
                    for (int col = 0; col < K; ++col) {
                        const double w = c_score_weights[r * K + col];
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
                bit = d1 > d2;
            }
            const unsigned word = __ballot_sync(0xffffffffu, bit);
            if ((threadIdx.x & 31) == 0) bits[static_cast<size_t>(patch) * words_per_patch + (c >> 5)] = word;
        }
    }
}

// in: [n][words_per_patch] (bit c of patch i at word c>>5, bit c&31); out: [C][out_words]
// (bit i of candidate c at word i>>5, bit i&31). One warp per 32-patch x 32-candidate block.
__global__ void transpose_kernel(const unsigned* __restrict__ in, unsigned n, unsigned words_per_patch, unsigned C,
                                 unsigned out_words, unsigned* __restrict__ out) {
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const unsigned cand_word = warp % words_per_patch, patch_block = warp / words_per_patch;
    if (patch_block >= out_words) return;
    const unsigned patch = patch_block * 32 + lane;
    const unsigned w = patch < n ? in[static_cast<size_t>(patch) * words_per_patch + cand_word] : 0u;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
        const unsigned col = __ballot_sync(0xffffffffu, (w >> b) & 1u);
        const unsigned c = cand_word * 32 + b;
        if (lane == 0 && c < C) out[static_cast<size_t>(c) * out_words + patch_block] = col;
    }
}

} // namespace

int launch_triplet_bits(clatch_ctx* ctx, const double* d_windows, size_t n, const short* d_candidates, size_t C, int K,
                        const double* weights, unsigned* d_by_patch, unsigned* d_out, cudaStream_t st) {
    CLATCH_CUDA(cudaMemcpyToSymbolAsync(c_score_weights, weights, sizeof(double) * K * K, 0, cudaMemcpyHostToDevice, st));
    const unsigned words_per_patch = static_cast<unsigned>((C + 31) / 32), out_words = static_cast<unsigned>((n + 31) / 32);
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(n, static_cast<size_t>(ctx->sm_count) * 4));
    score_kernel<<<grid, kScoreThreads, 0, st>>>(d_windows, static_cast<unsigned>(n), d_candidates,
                                                 static_cast<unsigned>(C), K, words_per_patch, d_by_patch);
    const size_t warps = static_cast<size_t>(words_per_patch) * out_words;
    transpose_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(
        d_by_patch, static_cast<unsigned>(n), words_per_patch, static_cast<unsigned>(C), out_words, d_out);
    ctx->launches += 2;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

} // namespace clatch
