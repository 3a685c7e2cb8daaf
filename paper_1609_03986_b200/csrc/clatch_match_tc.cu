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
// Structure (persistent CTAs, one per SM; a work item = 128 queries x a contiguous range of
// 256-row train tiles):
//   expand_kernel        bits -> int8, written to HBM directly in the UMMA canonical K-major
//                        SWIZZLE_128B layout (8 rows x 128 B atoms, 16-byte chunk index XOR row),
//                        128-row tiles, so every operand block is contiguous in global memory and
//                        one expansion of a set serves it as queries and as train rows
//   warp 0 (1 thread)    TMA bulk copies (cp.async.bulk + mbarrier expect-tx): A once per work item
//                        (64 KiB), B in a 4-stage ring of [256 rows x 128 B of K] = 32 KiB stages
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
constexpr int kTcSmemBytes = kTcABytes + kTcStages * kTcStageBytes + 1024 /*align*/ + 256 /*barriers*/ +
                             2048 /*half-merge buffer*/;

// ---------------------------------------------------------------- expansion ----
// One layout serves both operands: 128-row tiles, each [4 K-blocks][16 atoms][1024 B]. A query
// tile (A operand, M = 128) is one 64 KiB block; a train tile (B operand, N = 256) takes, per
// K-block, the 16 KiB of two consecutive 128-row tiles. One thread writes one 16-byte chunk
// (16 K-elements) of one row. Rows >= n (padding up to a multiple of 256) are zero and are
// masked in the epilogue.
__global__ void expand_kernel(const uint8_t* __restrict__ packed, unsigned long long n,
                              unsigned long long padded_rows, uint8_t* __restrict__ out) {
    constexpr int rows_per_tile = kTcM;
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
// The same copy delivered to the same CTA-relative offsets (data and mbarrier) of every CTA in `mask`.
__device__ __forceinline__ void bulk_load_multicast(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                                    unsigned short mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(unsigned bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// ... arriving on the barrier at the same offset in every CTA of `mask`.
__device__ __forceinline__ void tc_commit_multicast(unsigned bar, unsigned short mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"(mask)
                 : "memory");
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
// Persistent: gridDim.x CTAs (one per SM) each walk work items blockIdx.x, +gridDim.x, ...
// A work item = one 128-query tile against a contiguous range of 256-row train tiles. Items
// come either from (query tile, train split) arithmetic (single match; partial results go to
// `partial` and are merged afterwards) or from an item table (batched set pairs; each item
// covers a whole train set and writes final results). Barriers, TMEM and the smem ring are
// set up once per CTA; only the 64 KiB A operand is reloaded per item.
struct TcWork {
    const uint8_t* a;     // expanded query tile (64 KiB)
    const uint8_t* b;     // expanded train set (B form), tile 0
    unsigned long long Q, N;
    unsigned qtile;
    int tile_begin, ntiles, split;
    int32_t *o_idx, *o_best, *o_second;   // final outputs (item-table mode) or null
    bool ghost;           // pair mode: this CTA only keeps its partner's operand stream company (no output)
};

struct TcArgs {
    const uint8_t* a_exp;
    const uint8_t* b_exp;
    unsigned long long Q, N;
    int qtiles, total_tiles, tiles_per_split, num_items;
    int sk_chunks;           // > 0: "stream-K" partition of the (query tile, train tile) units over this many CTAs
    Partial* partial;
    int* dump;               // optional: raw accumulators of item 0's first tile, 128 x 256
    const TcItem* items;     // optional item table
};

// Stream-K partition: chunk c owns units [c*U/G, (c+1)*U/G); the chunk that holds unit x.
__host__ __device__ __forceinline__ unsigned long long tc_sk_chunk_of(unsigned long long x, unsigned long long U,
                                                                      unsigned long long G) {
    unsigned long long c = x * G / U;
    while ((c + 1) * U / G <= x) ++c;
    while (c * U / G > x) --c;
    return c;
}

// kPair: `item` counts PAIR items; the two CTAs of a cluster (rank 0 / 1) take two query tiles that scan the same
// train tiles — table entries 2 * item + rank, or query tiles 2j + rank of one split.
template <bool kPair>
__device__ __forceinline__ TcWork tc_decode(const TcArgs& g, int item, unsigned rank) {
    TcWork w;
    w.ghost = false;
    if (g.items != nullptr) {
        const TcItem it = g.items[kPair ? 2 * item + static_cast<int>(rank) : item];
        w.ghost = it.pad != 0;
        w.a = it.a_exp + static_cast<unsigned long long>(it.qtile) * kTcABytes;
        w.b = it.b_exp;
        w.Q = it.Q;
        w.N = it.N;
        w.qtile = it.qtile;
        w.tile_begin = 0;
        w.ntiles = static_cast<int>((it.N + kTcN - 1) / kTcN);
        w.split = 0;
        w.o_idx = it.best_idx;
        w.o_best = it.best_dist;
        w.o_second = it.second_dist;
    } else if (g.sk_chunks > 0) {
        // Small problems (train set resident in L2): the qtiles x total_tiles units are cut into
        // sk_chunks equal runs, one per CTA, in query-tile-major order; a run that crosses a query
        // tile boundary is several pieces (item = CTA + piece * chunks). Every CTA then carries the
        // same number of tile-times instead of ceil(items / SMs) whole rounds.
        const unsigned long long U = static_cast<unsigned long long>(g.qtiles) * g.total_tiles;
        const unsigned long long G = g.sk_chunks, TT = g.total_tiles;
        const unsigned long long c = static_cast<unsigned long long>(item) % G;
        const int piece = static_cast<int>(item / G);
        unsigned long long u = c * U / G;
        const unsigned long long ue = (c + 1) * U / G;
        unsigned long long q = 0, t0 = 0, n = 0;
        for (int i = 0; i <= piece; ++i, u += n) {
            if (u >= ue) {
                n = 0;
                break;
            }
            q = u / TT;
            t0 = u - q * TT;
            n = min(ue - u, TT - t0);
        }
        w.qtile = static_cast<unsigned>(q);
        w.tile_begin = static_cast<int>(t0);
        w.ntiles = static_cast<int>(n);
        w.split = static_cast<int>(c - tc_sk_chunk_of(q * TT, U, G));   // pieces of a query tile in train order
        w.a = g.a_exp + q * kTcABytes;
        w.b = g.b_exp;
        w.Q = g.Q;
        w.N = g.N;
        w.o_idx = w.o_best = w.o_second = nullptr;
    } else if (kPair) {
        const int pps = (g.qtiles + 1) / 2;                  // pair items per split
        w.split = item / pps;
        int qt = 2 * (item - w.split * pps) + static_cast<int>(rank);
        if (qt >= g.qtiles) {                                // odd tile count: the last pair's second CTA
            qt = g.qtiles - 1;
            w.ghost = true;
        }
        w.qtile = static_cast<unsigned>(qt);
        w.a = g.a_exp + static_cast<unsigned long long>(w.qtile) * kTcABytes;
        w.b = g.b_exp;
        w.Q = g.Q;
        w.N = g.N;
        w.tile_begin = w.split * g.tiles_per_split;
        w.ntiles = min(g.total_tiles, w.tile_begin + g.tiles_per_split) - w.tile_begin;
        w.o_idx = w.o_best = w.o_second = nullptr;
    } else {
        // consecutive CTAs take different query tiles of the SAME split: they stream the same
        // train tiles at the same time, so HBM sees them once and L2 serves the rest
        w.split = item / g.qtiles;
        w.qtile = static_cast<unsigned>(item - w.split * g.qtiles);
        w.a = g.a_exp + static_cast<unsigned long long>(w.qtile) * kTcABytes;
        w.b = g.b_exp;
        w.Q = g.Q;
        w.N = g.N;
        w.tile_begin = w.split * g.tiles_per_split;
        w.ntiles = min(g.total_tiles, w.tile_begin + g.tiles_per_split) - w.tile_begin;
        w.o_idx = w.o_best = w.o_second = nullptr;
    }
    return w;
}

// kPair = true: launched as clusters of two CTAs. Every CTA used to pull the whole train stream out of L2 by
// itself — 64 B/clk/SM at the tensor pipe's pace, 9.5 KB/clk over 148 SMs, which is more than L2 delivers
// (tools/tc_peak.cu: ~4.3-6 KB/clk) and held the kernel at 72-77 % of the MMA rate. Paired CTAs work on two
// query tiles against the SAME train tiles: each loads half of every B stage and multicasts it into both
// CTAs' shared memory (one L2 read feeds two SMs), and a stage is handed back to the producers only when both
// CTAs' MMAs have read it (multicast tcgen05.commit onto both `empty` barriers).
template <bool kPair>
__global__ void __launch_bounds__(kTcThreads, 1) match_tc_kernel(const TcArgs g) {
    const unsigned rank = kPair ? cluster_rank() : 0u;
    const int first_item = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int item_step = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
    extern __shared__ uint8_t smem_raw[];
    const unsigned raw = smem_u32(smem_raw);
    const unsigned base = (raw + 1023u) & ~1023u;              // SWIZZLE_128B atoms need 1024-B alignment
    const unsigned smem_a = base;
    const unsigned smem_b = base + kTcABytes;
    const unsigned bars = smem_b + kTcStages * kTcStageBytes;  // 8-byte mbarriers
    const unsigned bar_a_full = bars;
    const unsigned bar_a_empty = bars + 8;
    const unsigned bar_full = bars + 16;                       // [kTcStages]
    const unsigned bar_empty = bar_full + 8 * kTcStages;       // [kTcStages]
    const unsigned bar_tfull = bar_empty + 8 * kTcStages;      // [2]
    const unsigned bar_tempty = bar_tfull + 16;                // [2]
    uint8_t* const gen_base = smem_raw + (base - raw);
    uint8_t* const tail = gen_base + kTcABytes + kTcStages * kTcStageBytes;
    volatile unsigned* tmem_slot = reinterpret_cast<volatile unsigned*>(tail + 128);
    int* merge_buf = reinterpret_cast<int*>(tail + 256);       // 128 rows x 4 ints

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(bar_a_full, 1);
        mbar_init(bar_a_empty, 1);
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, kPair ? 2 : 1);       // pair mode: both CTAs' MMAs must have read the stage
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
    if (kPair) cluster_sync_all();                             // the partner's barriers exist before anything lands on them
    tc_fence_after();
    const unsigned tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===== producer =====
        if (lane == 0) {
            int stage = 0;
            unsigned phase = 0, a_phase = 0;
            for (int item = first_item; item < g.num_items; item += item_step) {
                const TcWork w = tc_decode<kPair>(g, item, rank);
                if (w.ntiles == 0) continue;                   // (stream-K: this CTA has fewer pieces)
                mbar_wait(bar_a_empty, a_phase ^ 1);           // previous item's MMAs are done with A
                mbar_expect_tx(bar_a_full, kTcABytes);
                bulk_load(smem_a, w.a, kTcABytes, bar_a_full);
                a_phase ^= 1;
                for (int t = 0; t < w.ntiles; ++t) {
                    // train tile = two consecutive 128-row tiles of the expanded set
                    const uint8_t* src = w.b + static_cast<unsigned long long>(w.tile_begin + t) * (2 * kTcABytes);
                    for (int kb = 0; kb < kTcKBlocks; ++kb) {
                        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                        mbar_expect_tx(bar_full + 8 * stage, kTcStageBytes);
                        const unsigned dst = smem_b + stage * kTcStageBytes;
                        if (kPair) {   // this CTA's half of the stage, to both CTAs
                            bulk_load_multicast(dst + rank * (kTcStageBytes / 2),
                                                src + rank * kTcABytes + kb * (kTcStageBytes / 2), kTcStageBytes / 2,
                                                bar_full + 8 * stage, 3);
                        } else {
                            bulk_load(dst, src + kb * (kTcStageBytes / 2), kTcStageBytes / 2, bar_full + 8 * stage);
                            bulk_load(dst + kTcStageBytes / 2, src + kTcABytes + kb * (kTcStageBytes / 2), kTcStageBytes / 2,
                                      bar_full + 8 * stage);
                        }
                        if (++stage == kTcStages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            int stage = 0, tcount = 0;
            unsigned phase = 0, a_phase = 0;
            for (int item = first_item; item < g.num_items; item += item_step) {
                const TcWork w = tc_decode<kPair>(g, item, rank);
                if (w.ntiles == 0) continue;
                mbar_wait(bar_a_full, a_phase);
                a_phase ^= 1;
                for (int t = 0; t < w.ntiles; ++t, ++tcount) {
                    const int buf = tcount & 1;
                    mbar_wait(bar_tempty + 8 * buf, ((tcount >> 1) & 1) ^ 1);   // epilogue drained this accumulator
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
                        if (kPair) tc_commit_multicast(bar_empty + 8 * stage, 3);
                        else tc_commit(bar_empty + 8 * stage);  // stage reusable once these MMAs have read it
                        if (++stage == kTcStages) { stage = 0; phase ^= 1; }
                    }
                    tc_commit(bar_tfull + 8 * buf);            // accumulator complete
                }
                tc_commit(bar_a_empty);                        // every MMA of this item has read A
            }
        }
    } else {
        // ===== epilogue: warps 2..9 =====
        const int ew = warp - 2;
        const int quarter = warp & 3;                       // TMEM lane quarter this warp may touch
        const int half = ew >> 2;                           // which 128 of the 256 columns
        const unsigned lane_addr = static_cast<unsigned>(quarter * 32) << 16;
        const int row = quarter * 32 + lane;
        int tcount = 0;
        for (int item = first_item; item < g.num_items; item += item_step) {
            const TcWork w = tc_decode<kPair>(g, item, rank);
            if (w.ntiles == 0) continue;
            int best = INT_MIN, second = INT_MIN, best_idx = -1;
            for (int t = 0; t < w.ntiles; ++t, ++tcount) {
                const int buf = tcount & 1;
                mbar_wait(bar_tfull + 8 * buf, (tcount >> 1) & 1);
                tc_fence_after();
                const long long col0 = static_cast<long long>(w.tile_begin + t) * kTcN + half * 128;
                const long long valid = static_cast<long long>(w.N) - col0;   // columns < valid are real rows
#pragma unroll 1
                for (int chunk = 0; chunk < 4; ++chunk) {
                    int v[32];
                    tmem_ld32(tmem_base + lane_addr + buf * kTcN + half * 128 + chunk * 32, v);
                    if (g.dump != nullptr && item == 0 && t == 0 && rank == 0) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) g.dump[row * kTcN + half * 128 + chunk * 32 + i] = v[i];
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
                        const int cbase = t * kTcN + half * 128 + chunk * 32;
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
            if (half == 1) {
                merge_buf[row * 4 + 0] = best;
                merge_buf[row * 4 + 1] = second;
                merge_buf[row * 4 + 2] = best_idx;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpilogueWarps) : "memory");
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
                const unsigned long long qi = static_cast<unsigned long long>(w.qtile) * kTcM + row;
                if (qi < w.Q && !w.ghost) {
                    const int idx = best_idx < 0 ? -1 : w.tile_begin * kTcN + best_idx;
                    const int bd = best == INT_MIN ? 513 : (512 - best) >> 1;
                    const int sd = second == INT_MIN ? 513 : (512 - second) >> 1;
                    if (g.items != nullptr) {          // whole train range seen: these are final
                        if (w.o_idx) w.o_idx[qi] = idx;
                        if (w.o_best) w.o_best[qi] = bd;
                        if (w.o_second) w.o_second[qi] = sd;
                    } else {
                        Partial r;
                        r.best_idx = idx;
                        r.best_dist = bd;
                        r.second_dist = sd;
                        r.pad = 0;
                        g.partial[static_cast<unsigned long long>(w.split) * w.Q + qi] = r;
                    }
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpilogueWarps) : "memory");   // merge_buf free again
        }
    }

    tc_fence_before();
    __syncthreads();
    if (kPair) cluster_sync_all();                             // nothing of the partner's is still bound for this CTA
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

} // namespace

namespace {

// Merge of the stream-K pieces: query tile q was cut into the chunks c_first(q) .. c_last(q), whose
// partials sit in slots 0 .. c_last - c_first in ascending train order (same rule as
// merge_partials_kernel: strictly better wins, so the earlier piece keeps ties).
__global__ void merge_partials_sk_kernel(const Partial* __restrict__ partial, unsigned long long Q, int total_tiles,
                                         int qtiles, int chunks, int32_t* __restrict__ best_idx,
                                         int32_t* __restrict__ best_dist, int32_t* __restrict__ second_dist) {
    const unsigned long long qi = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (qi >= Q) return;
    const unsigned long long U = static_cast<unsigned long long>(qtiles) * total_tiles, TT = total_tiles, q = qi / kTcM;
    const int pieces = static_cast<int>(tc_sk_chunk_of((q + 1) * TT - 1, U, chunks) - tc_sk_chunk_of(q * TT, U, chunks)) + 1;
    int best = 513, second = 513, idx = -1;
    for (int s = 0; s < pieces; ++s) {
        const Partial r = partial[static_cast<unsigned long long>(s) * Q + qi];
        if (r.best_dist < best) {
            second = min(best, r.second_dist);
            best = r.best_dist;
            idx = r.best_idx;
        } else {
            second = min(second, r.best_dist);
        }
    }
    if (best_idx) best_idx[qi] = idx;
    if (best_dist) best_dist[qi] = best;
    if (second_dist) second_dist[qi] = second;
}

} // namespace

// The opt-in shared-memory size is a per-device function attribute: remember it per context.
static int configure_tc(clatch_ctx* ctx) {
    if (!ctx->tc_configured) {
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmemBytes));
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmemBytes));
        ctx->tc_configured = true;
    }
    return CLATCH_OK;
}

size_t tc_expanded_bytes(size_t rows) { return (rows + kTcN - 1) / kTcN * (2 * static_cast<size_t>(kTcABytes)); }

int launch_tc_expand(clatch_ctx* ctx, const uint8_t* d_packed, size_t n, uint8_t* d_out, cudaStream_t stream) {
    const unsigned long long rows = (n + kTcN - 1) / kTcN * kTcN, threads = rows * 32;
    if (rows == 0) return CLATCH_OK;
    expand_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(d_packed, n, rows, d_out);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

int tc_query_tiles(size_t rows) { return static_cast<int>((rows + kTcM - 1) / kTcM); }

// Clusters of two CTAs (cudaLaunchKernelEx): the paired form of the kernel.
static int launch_tc_pairs(clatch_ctx* ctx, const TcArgs& g, unsigned ctas, cudaStream_t stream) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas & ~1u);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = kTcSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    CLATCH_CUDA(cudaLaunchKernelEx(&cfg, match_tc_kernel<true>, g));
    ++ctx->launches;
    return CLATCH_OK;
}

int launch_match_tc_items(clatch_ctx* ctx, const TcItem* d_items, size_t count, cudaStream_t stream) {
    if (count == 0) return CLATCH_OK;
    if (int rc = configure_tc(ctx)) return rc;
    TcArgs g{};
    g.items = d_items;
    if (ctx->match_pairs) {   // the table holds entries (2k, 2k + 1) that scan the same train set (tc_items_paired)
        g.num_items = static_cast<int>(count / 2);
        return launch_tc_pairs(ctx, g, static_cast<unsigned>(std::min<size_t>(count, ctx->sm_count)), stream);
    }
    g.num_items = static_cast<int>(count);
    const unsigned grid = static_cast<unsigned>(std::min<size_t>(count, ctx->sm_count));
    match_tc_kernel<false><<<grid, kTcThreads, kTcSmemBytes, stream>>>(g);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

bool tc_items_paired(const clatch_ctx* ctx) { return ctx->match_pairs; }

int launch_match_top2_tc(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                         int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second, cudaStream_t stream,
                         int32_t* d_dump) {
    if (int rc = configure_tc(ctx)) return rc;
    const size_t qtiles = (Q + kTcM - 1) / kTcM, ttiles = (N + kTcN - 1) / kTcN;
    // Both sets go to the tensor cores as int8; a self-match expands its one set once.
    const bool self = d_q == d_t && Q == N;
    if (int rc = ctx->exp_t.reserve(tc_expanded_bytes(N))) return rc;
    if (int rc = launch_tc_expand(ctx, d_t, N, ctx->exp_t.as<uint8_t>(), stream)) return rc;
    const uint8_t* a_exp = ctx->exp_t.as<uint8_t>();
    if (!self) {
        if (int rc = ctx->exp_q.reserve(tc_expanded_bytes(Q))) return rc;
        if (int rc = launch_tc_expand(ctx, d_q, Q, ctx->exp_q.as<uint8_t>(), stream)) return rc;
        a_exp = ctx->exp_q.as<uint8_t>();
    }
    // Split the train range when there are too few query tiles to keep every SM busy. Model: the
    // persistent CTAs run ceil(items / SMs) rounds; an item costs (tiles + kOverhead) tile-times
    // (A reload + pipeline refill). Pick the split count with the smallest makespan.
    size_t splits = 1, per_split = ttiles;
    {
        const size_t sms = static_cast<size_t>(ctx->sm_count);
        const double kOverhead = 1.5;
        double best_cost = 1e300;
        for (size_t s = 1; s <= std::min<size_t>(ttiles, 64); ++s) {
            const size_t per = (ttiles + s - 1) / s, actual = (ttiles + per - 1) / per;
            const size_t rounds = (qtiles * actual + sms - 1) / sms;
            const double cost = rounds * (per + kOverhead);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                splits = actual;
                per_split = per;
            }
        }
    }
    // Stream-K instead, when the expanded train set stays in L2 (every CTA streams it at its own phase)
    // and the equal-share makespan beats whole rounds: U / SMs tile-times + one A reload per piece.
    const size_t sms = static_cast<size_t>(ctx->sm_count);
    const size_t units = qtiles * ttiles, chunks = std::min(units, sms);
    bool streamk = false;
    size_t sk_pieces_per_cta = 1, sk_pieces_per_qtile = 1;
    if (tc_expanded_bytes(N) <= (32u << 20) && units > 0 && ctx->match_streamk) {
        const size_t share = (units + chunks - 1) / chunks;                 // tile-times per CTA
        sk_pieces_per_cta = (share + ttiles - 2) / ttiles + 1;
        sk_pieces_per_qtile = (ttiles + units / chunks - 1) / (units / chunks) + 1;
        const size_t rounds = (qtiles * splits + sms - 1) / sms;
        const double legacy = rounds * (per_split + 1.5), sk = share + 2.0 * sk_pieces_per_cta;   // (measured: tools/sk_perf.py)
        streamk = sk < legacy;
    }
    // Otherwise pairs of CTAs share the train stream (match_tc_kernel<true>): the schedulable unit is a pair of
    // query tiles on a pair of SMs, so the split count is chosen again in those units.
    const bool paired = !streamk && ctx->match_pairs && qtiles >= 2 && sms >= 2;
    if (paired) {
        const size_t pq = (qtiles + 1) / 2, slots2 = sms / 2;
        double best_cost = 1e300;
        for (size_t s = 1; s <= std::min<size_t>(ttiles, 64); ++s) {
            const size_t per = (ttiles + s - 1) / s, actual = (ttiles + per - 1) / per;
            const size_t rounds = (pq * actual + slots2 - 1) / slots2;
            const double cost = rounds * (per + 1.5);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                splits = actual;
                per_split = per;
            }
        }
    }
    const size_t slots = streamk ? sk_pieces_per_qtile : splits;
    if (int rc = ctx->partial.reserve(sizeof(Partial) * slots * Q)) return rc;
    TcArgs g{};
    g.a_exp = a_exp;
    g.b_exp = ctx->exp_t.as<uint8_t>();
    g.Q = Q;
    g.N = N;
    g.qtiles = static_cast<int>(qtiles);
    g.total_tiles = static_cast<int>(ttiles);
    g.tiles_per_split = static_cast<int>(per_split);
    g.num_items = static_cast<int>(streamk ? chunks * sk_pieces_per_cta : qtiles * splits);
    g.sk_chunks = streamk ? static_cast<int>(chunks) : 0;
    g.partial = ctx->partial.as<Partial>();
    g.dump = d_dump;
    if (paired) {
        const size_t pair_items = (qtiles + 1) / 2 * splits;
        g.num_items = static_cast<int>(pair_items);
        if (int rc = launch_tc_pairs(ctx, g, static_cast<unsigned>(std::min<size_t>(2 * pair_items, sms)), stream)) return rc;
    } else {
        const unsigned grid = static_cast<unsigned>(streamk ? chunks : std::min<size_t>(qtiles * splits, ctx->sm_count));
        match_tc_kernel<false><<<grid, kTcThreads, kTcSmemBytes, stream>>>(g);
        ++ctx->launches;
    }
    CLATCH_CUDA(cudaGetLastError());
    if (streamk)
        merge_partials_sk_kernel<<<static_cast<unsigned>((Q + 255) / 256), 256, 0, stream>>>(
            ctx->partial.as<Partial>(), Q, static_cast<int>(ttiles), static_cast<int>(qtiles), static_cast<int>(chunks),
            d_best_idx, d_best_dist, d_second);
    else
        launch_merge_partials(ctx->partial.as<Partial>(), Q, static_cast<int>(splits), 513, d_best_idx, d_best_dist,
                              d_second, stream);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

} // namespace clatch
