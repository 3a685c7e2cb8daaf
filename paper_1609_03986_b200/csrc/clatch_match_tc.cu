// Hamming top-2 matching on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same result as clatch_match.cu (reference: src/match.cpp:14-50 — hamming + knn2), computed as
// an exact integer GEMM: with both descriptor sets expanded to int8 (+1 for a set bit, -1 for
// a clear bit), the dot product of two 512-element rows is D = 512 - 2 * hamming, so the
// nearest neighbour is the largest D and hamming = (512 - D) / 2. Accumulation is int32 in
// TMEM: no rounding anywhere, ties still resolve to the lowest train index.
//
// Why: POPC issues at 16 lanes/clk/SM, which caps the XOR+popcount form at ~3.3e11
// compares/s even with carry-save compression; tcgen05.mma kind::i8 does
// 8192 MAC/clk/SM = 16 compares/clk/SM.
//
// Structure (one CTA = 128 queries x a contiguous range of 256-row train tiles):
//   expand_kernel        bits -> int8, written to HBM directly in the UMMA canonical K-major
//                        SWIZZLE_128B layout (8 rows x 128 B atoms, 16-byte chunk index XOR row),
//                        so every operand tile is one contiguous block in global memory
//   warp 0 (1 thread)    TMA bulk copies (cp.async.bulk + mbarrier expect-tx): A once (64 KiB),
//                        B in 4-stage ring of [256 rows x 128 B of K] = 32 KiB stages
//   warp 1 (1 thread)    tcgen05.mma.cta_group::1.kind::i8, M=128, N=256, K=32 x 16 per tile,
//                        accumulators double-buffered in TMEM (2 x 256 columns);
//                        tcgen05.commit releases smem stages and publishes finished tiles
//   warps 2-9            epilogue: tcgen05.ld 32 columns at a time, running top-2 per query row.
//                        A 3-input max over the 32 values is compared with the row's current
//                        runner-up first; the per-element update only runs when it can change
//                        something (rare once a few thousand rows have been seen).
// Per-split partial results reuse merge_partials_kernel from clatch_match.cu.

#include <algorithm>
#include <climits>

#include "clatch_internal.cuh"

namespace clatch {

namespace {

constexpr int kTcM = 128;                 // queries per CTA (UMMA M)
constexpr int kTcN = 256;                 // train rows per tile (UMMA N)
constexpr int kTcKBlock = 128;            // bytes of K per smem stage = one swizzle-atom row
constexpr int kTcKBlocks = 4;             // 512 / 128
constexpr int kTcStages = 4;
constexpr int kTcABytes = kTcM * 512;             // 65536
constexpr int kTcStageBytes = kTcN * kTcKBlock;   // 32768
constexpr int kTcEpilogueWarps = 8;
constexpr int kTcThreads = 32 * (2 + kTcEpilogueWarps);   // 320
constexpr int kTcSmemBytes = kTcABytes + kTcStages * kTcStageBytes + 1024 /*align*/ + 256 /*barriers*/;

// ---------------------------------------------------------------- expansion ----
// rows_per_tile = 128 (queries, A operand) or 256 (train, B operand). One thread writes one
// 16-byte chunk (16 K-elements) of one row. Rows >= n are zero (masked in the epilogue).
__global__ void expand_kernel(const uint8_t* __restrict__ packed, unsigned long long n,
                              unsigned long long padded_rows, int rows_per_tile, uint8_t* __restrict__ out) {
    const unsigned long long idx = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    const unsigned long long row = idx >> 5;          // 32 chunks per row
    if (row >= padded_rows) return;
    const int chunk = static_cast<int>(idx & 31);     // bits [16*chunk, 16*chunk+16)
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < n) {
        const unsigned bits = *reinterpret_cast<const unsigned short*>(packed + row * 64 + 2 * chunk);
        unsigned w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const unsigned nib = (bits >> (4 * i)) & 0xF;
            // spread 4 bits to 4 bytes (0/1), then 1 -> 0x01 (+1), 0 -> 0xFF (-1)
            const unsigned ones = (nib * 0x00204081u) & 0x01010101u;
            w[i] = ((ones ^ 0x01010101u) * 0xFFu) | ones;   // per byte: 0 -> 0xFF (-1), 1 -> 0x01 (+1)
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
    }
    const unsigned long long tile = row / rows_per_tile;
    const int r = static_cast<int>(row - tile * rows_per_tile);
    const int kb = chunk >> 3, c = chunk & 7, g = r >> 3, ri = r & 7;
    const unsigned long long atom = (tile * kTcKBlocks + kb) * (rows_per_tile / 8) + g;
    *reinterpret_cast<uint4*>(out + atom * 1024 + ri * 128 + ((c ^ ri) << 4)) = v;
}

// ---------------------------------------------------------------- PTX helpers ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TC_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra TC_DONE;\n"
        "bra TC_WAIT;\n"
        "TC_DONE:\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(unsigned bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, int8 x int8 -> int32, M=128, N=256, K=32.
__device__ __forceinline__ void tc_mma_i8(unsigned tmem_d, uint64_t desc_a, uint64_t desc_b, unsigned idesc,
                                          unsigned accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
        : "memory");
}
// K-major, SWIZZLE_128B shared-memory matrix descriptor (cute::UMMA::SmemDescriptor layout):
// start address >> 4 in [0,14), LBO (unused for swizzled K-major) in [16,30), SBO = 1024 B
// between 8-row groups in [32,46), version 1 in [46,48), layout type 2 in [61,64).
__device__ __forceinline__ uint64_t umma_desc(unsigned smem_addr) {
    return static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}
// Instruction descriptor (cute::UMMA::InstrDescriptor): D = S32 (2 @4), A = B = S8 (1 @7, 1 @10),
// both K-major, N >> 3 @17, M >> 4 @24.
constexpr unsigned kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((kTcN >> 3) << 17) | ((kTcM >> 4) << 24);

__device__ __forceinline__ void tmem_ld32(unsigned taddr, int (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- the kernel ----
// grid = (query tiles, splits). Split s owns train tiles [s*tiles_per_split, ...).
__global__ void __launch_bounds__(kTcThreads, 1)
match_tc_kernel(const uint8_t* __restrict__ a_exp_arg, const uint8_t* __restrict__ b_exp_arg, unsigned long long Q_arg,
                unsigned long long N_arg, int total_tiles, int tiles_per_split, Partial* __restrict__ partial,
                int* __restrict__ dump /* optional: raw accumulators of this CTA's first tile, 128 x 256 */,
                const TcItem* __restrict__ items /* optional: one work item per CTA (batched set pairs) */) {
    // Work of this CTA: either derived from (blockIdx.x = query tile, blockIdx.y = train split) or
    // read from the item table (batched matching of many set pairs in one launch).
    const uint8_t* a_exp = a_exp_arg;
    const uint8_t* b_exp = b_exp_arg;
    unsigned long long Q = Q_arg, N = N_arg;
    unsigned qtile = blockIdx.x;
    int tile_begin = blockIdx.y * tiles_per_split;
    int tile_end = min(total_tiles, tile_begin + tiles_per_split);
    int32_t *o_idx = nullptr, *o_best = nullptr, *o_second = nullptr;
    if (items != nullptr) {
        const TcItem it = items[blockIdx.x];
        a_exp = it.a_exp;
        b_exp = it.b_exp;
        Q = it.Q;
        N = it.N;
        qtile = it.qtile;
        tile_begin = 0;
        tile_end = static_cast<int>((it.N + kTcN - 1) / kTcN);
        o_idx = it.best_idx;
        o_best = it.best_dist;
        o_second = it.second_dist;
    }
    extern __shared__ uint8_t smem_raw[];
    const unsigned raw = smem_u32(smem_raw);
    const unsigned base = (raw + 1023u) & ~1023u;              // SWIZZLE_128B atoms need 1024-B alignment
    const unsigned smem_a = base;
    const unsigned smem_b = base + kTcABytes;
    const unsigned bars = smem_b + kTcStages * kTcStageBytes;  // 8-byte mbarriers
    const unsigned bar_a = bars;
    const unsigned bar_full = bars + 8;                        // [kTcStages]
    const unsigned bar_empty = bar_full + 8 * kTcStages;       // [kTcStages]
    const unsigned bar_tfull = bar_empty + 8 * kTcStages;      // [2]
    const unsigned bar_tempty = bar_tfull + 16;                // [2]
    uint8_t* const gen_base = smem_raw + (base - raw);
    volatile unsigned* tmem_slot = reinterpret_cast<volatile unsigned*>(gen_base + kTcABytes + kTcStages * kTcStageBytes + 128);
    int* merge_buf = reinterpret_cast<int*>(gen_base);         // reused after the main loop (A region)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = tile_end - tile_begin;

    if (threadIdx.x == 0) {
        mbar_init(bar_a, 1);
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, kTcEpilogueWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {   // TMEM: all 512 columns (two 256-column accumulators)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(const_cast<unsigned*>(tmem_slot))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== producer =====
        if (lane == 0) {
            mbar_expect_tx(bar_a, kTcABytes);
            bulk_load(smem_a, a_exp + static_cast<unsigned long long>(qtile) * kTcABytes, kTcABytes, bar_a);
            int stage = 0;
            unsigned phase = 0;
            for (int t = 0; t < ntiles; ++t) {
                const uint8_t* src = b_exp + static_cast<unsigned long long>(tile_begin + t) * (kTcKBlocks * kTcStageBytes);
                for (int kb = 0; kb < kTcKBlocks; ++kb) {
                    mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                    mbar_expect_tx(bar_full + 8 * stage, kTcStageBytes);
                    bulk_load(smem_b + stage * kTcStageBytes, src + kb * kTcStageBytes, kTcStageBytes,
                              bar_full + 8 * stage);
                    if (++stage == kTcStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            mbar_wait(bar_a, 0);
            int stage = 0;
            unsigned phase = 0;
            for (int t = 0; t < ntiles; ++t) {
                const int buf = t & 1;
                mbar_wait(bar_tempty + 8 * buf, ((t >> 1) & 1) ^ 1);   // epilogue drained this accumulator
                tc_fence_after();
                const unsigned tmem_d = tmem_base + buf * kTcN;
                for (int kb = 0; kb < kTcKBlocks; ++kb) {
                    mbar_wait(bar_full + 8 * stage, phase);
                    tc_fence_after();
                    const unsigned a_addr = smem_a + kb * (kTcM * kTcKBlock);
                    const unsigned b_addr = smem_b + stage * kTcStageBytes;
#pragma unroll
                    for (int k = 0; k < kTcKBlock / 32; ++k)
                        tc_mma_i8(tmem_d, umma_desc(a_addr + 32 * k), umma_desc(b_addr + 32 * k), kIdesc,
                                  (kb | k) != 0);
                    tc_commit(bar_empty + 8 * stage);      // stage reusable once these MMAs have read it
                    if (++stage == kTcStages) { stage = 0; phase ^= 1; }
                }
                tc_commit(bar_tfull + 8 * buf);            // accumulator complete
            }
        }
    } else {
        // ===== epilogue: warps 2..9 =====
        const int ew = warp - 2;
        const int quarter = warp & 3;                       // TMEM lane quarter this warp may touch
        const int half = ew >> 2;                           // which 128 of the 256 columns
        const unsigned lane_addr = static_cast<unsigned>(quarter * 32) << 16;
        int best = INT_MIN, second = INT_MIN, best_idx = -1;
        for (int t = 0; t < ntiles; ++t) {
            const int buf = t & 1;
            mbar_wait(bar_tfull + 8 * buf, (t >> 1) & 1);
            tc_fence_after();
            const long long col0 = static_cast<long long>(tile_begin + t) * kTcN + half * 128;
            const long long valid = static_cast<long long>(N) - col0;   // columns < valid are real rows
#pragma unroll 1
            for (int chunk = 0; chunk < 4; ++chunk) {
                int v[32];
                tmem_ld32(tmem_base + lane_addr + buf * kTcN + half * 128 + chunk * 32, v);
                if (dump != nullptr && t == 0 && qtile == 0 && blockIdx.y == 0) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        dump[(quarter * 32 + lane) * kTcN + half * 128 + chunk * 32 + i] = v[i];
                }
                const long long cvalid = valid - chunk * 32;
                if (cvalid < 32) {                          // last tile only: mask the zero padding rows
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i >= cvalid) v[i] = INT_MIN;
                }
                int m = v[0];
#pragma unroll
                for (int i = 1; i < 32; i += 2) m = max(m, max(v[i], i + 1 < 32 ? v[i + 1] : INT_MIN));
                if (m > second) {                           // something in this chunk enters the top-2
                    const int cbase = static_cast<int>(col0 - static_cast<long long>(tile_begin) * kTcN) + chunk * 32;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int d = v[i];
                        if (d > best) {                     // strict: earlier (lower) index keeps ties
                            second = best;
                            best = d;
                            best_idx = cbase + i;
                        } else if (d > second) {
                            second = d;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_tempty + 8 * buf);
        }
        // merge the two column halves of each row
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpilogueWarps));   // all MMAs done => A region is free
        const int row = quarter * 32 + lane;
        if (half == 1) {
            merge_buf[row * 4 + 0] = best;
            merge_buf[row * 4 + 1] = second;
            merge_buf[row * 4 + 2] = best_idx;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpilogueWarps));
        if (half == 0) {
            const int ob = merge_buf[row * 4 + 0], os = merge_buf[row * 4 + 1], oi = merge_buf[row * 4 + 2];
            // the halves interleave in index order across tiles, so ties compare indices
            if (ob > best || (ob == best && oi >= 0 && oi < best_idx)) {
                second = max(best, os);
                best = ob;
                best_idx = oi;
            } else {
                second = max(second, ob);
            }
            const unsigned long long qi = static_cast<unsigned long long>(qtile) * kTcM + row;
            if (qi < Q) {
                const int idx = best_idx < 0 ? -1 : tile_begin * kTcN + best_idx;
                const int bd = best == INT_MIN ? 513 : (512 - best) >> 1;
                const int sd = second == INT_MIN ? 513 : (512 - second) >> 1;
                if (items != nullptr) {          // whole train range seen: these are final
                    if (o_idx) o_idx[qi] = idx;
                    if (o_best) o_best[qi] = bd;
                    if (o_second) o_second[qi] = sd;
                } else {
                    Partial r;
                    r.best_idx = idx;
                    r.best_dist = bd;
                    r.second_dist = sd;
                    r.pad = 0;
                    partial[static_cast<unsigned long long>(blockIdx.y) * Q + qi] = r;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

} // namespace

static int configure_tc() {
    static bool configured = false;
    if (!configured) {
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmemBytes));
        configured = true;
    }
    return CLATCH_OK;
}

size_t tc_expanded_bytes(size_t rows, bool as_queries) {
    return as_queries ? (rows + kTcM - 1) / kTcM * kTcABytes
                      : (rows + kTcN - 1) / kTcN * (kTcKBlocks * kTcStageBytes);
}

int launch_tc_expand(clatch_ctx* ctx, const uint8_t* d_packed, size_t n, bool as_queries, uint8_t* d_out,
                     cudaStream_t stream) {
    const int rows_per_tile = as_queries ? kTcM : kTcN;
    const unsigned long long rows = (n + rows_per_tile - 1) / rows_per_tile * rows_per_tile, threads = rows * 32;
    if (rows == 0) return CLATCH_OK;
    expand_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(d_packed, n, rows, rows_per_tile,
                                                                                    d_out);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

int tc_query_tiles(size_t rows) { return static_cast<int>((rows + kTcM - 1) / kTcM); }

int launch_match_tc_items(clatch_ctx* ctx, const TcItem* d_items, size_t count, cudaStream_t stream) {
    if (count == 0) return CLATCH_OK;
    if (int rc = configure_tc()) return rc;
    match_tc_kernel<<<static_cast<unsigned>(count), kTcThreads, kTcSmemBytes, stream>>>(nullptr, nullptr, 0, 0, 0, 0,
                                                                                      nullptr, nullptr, d_items);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

int launch_match_top2_tc(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                         int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second, cudaStream_t stream,
                         int32_t* d_dump) {
    if (int rc = configure_tc()) return rc;
    const size_t qtiles = (Q + kTcM - 1) / kTcM, ttiles = (N + kTcN - 1) / kTcN;
    if (int rc = ctx->exp_q.reserve(qtiles * kTcABytes)) return rc;
    if (int rc = ctx->exp_t.reserve(ttiles * kTcKBlocks * kTcStageBytes)) return rc;
    {
        const unsigned long long rows = qtiles * kTcM, threads = rows * 32;
        expand_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(d_q, Q, rows, kTcM,
                                                                                        ctx->exp_q.as<uint8_t>());
        ++ctx->launches;
    }
    {
        const unsigned long long rows = ttiles * kTcN, threads = rows * 32;
        expand_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(d_t, N, rows, kTcN,
                                                                                        ctx->exp_t.as<uint8_t>());
        ++ctx->launches;
    }
    CLATCH_CUDA(cudaGetLastError());
    // Split the train range over blockIdx.y when there are too few query tiles to fill the
    // SMs. Model: CTAs run in waves of one per SM; a CTA costs (tiles + kOverhead) tile-times
    // (barrier init, TMEM allocation, 64 KiB A load, pipeline fill, merge). Pick the split count with the smallest makespan.
    size_t best_splits = 1, best_per = ttiles;
    {
        const size_t sms = static_cast<size_t>(ctx->sm_count), kOverhead = 8;   // measured: ~8 us of fixed cost per CTA vs ~1 us per tile
        size_t best_cost = ~static_cast<size_t>(0);
        for (size_t s = 1; s <= std::min<size_t>(ttiles, 64); ++s) {
            const size_t per = (ttiles + s - 1) / s, actual = (ttiles + per - 1) / per;
            const size_t waves = (qtiles * actual + sms - 1) / sms;
            const size_t cost = waves * (per + kOverhead);
            if (cost < best_cost) {
                best_cost = cost;
                best_splits = actual;
                best_per = per;
            }
        }
    }
    const size_t splits = best_splits, per_split = best_per;
    if (int rc = ctx->partial.reserve(sizeof(Partial) * splits * Q)) return rc;
    dim3 grid(static_cast<unsigned>(qtiles), static_cast<unsigned>(splits));
    match_tc_kernel<<<grid, kTcThreads, kTcSmemBytes, stream>>>(ctx->exp_q.as<uint8_t>(), ctx->exp_t.as<uint8_t>(), Q,
                                                                N, static_cast<int>(ttiles),
                                                                static_cast<int>(per_split),
                                                                ctx->partial.as<Partial>(), d_dump, nullptr);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    launch_merge_partials(ctx->partial.as<Partial>(), Q, static_cast<int>(splits), 513, d_best_idx, d_best_dist, d_second, stream);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

} // namespace clatch
