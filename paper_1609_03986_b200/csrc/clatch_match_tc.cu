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
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "clatch_internal.cuh"

namespace clatch {

namespace {

constexpr int kTcM = 128;                 // queries per CTA (UMMA M)
constexpr int kTcKBlock = 128;            // bytes of K per smem stage row = one swizzle-atom row
constexpr int kTcStages = 4;
template <class F> __host__ __device__ constexpr int tc_threads() { return 32 * (2 + F::kEpiWarps); }   // 320 / 576

// Two operand forms, same kernel:
//   TcI8  int8 +-1, 512 B per descriptor, kind::i8, int32 accumulators, 256 train rows per tile
//   TcF4  e2m1 +-1.0 (0x2 / 0xA), 256 B per descriptor, kind::mxf4 with every UE8M0 block scale = 2^0, f32
//         accumulators — twice the MACs per clock and half the operand bytes; 240 train rows per tile because
//         the scale factors need TMEM columns too (2 x 240 accumulator columns + 2 x 16 columns of 0x7F bytes).
// Every partial sum is an integer of magnitude <= 512, so f32 accumulation is as exact as int32.
struct TcI8 {
    static constexpr bool kF4 = false;
    static constexpr int kN = 256;             // train rows per tile (UMMA N)
    static constexpr int kKBlocks = 4;         // 128-byte K-blocks per descriptor row (512 B)
    static constexpr bool kParked = false;     // (64 KiB A + 128 KiB ring leave no room for the parking slots)
    static constexpr int kEpiWarps = 8;        // 4 TMEM lane quarters x 2 column halves
};
struct TcF4 {
    static constexpr bool kF4 = true;
    static constexpr int kN = 240;
    static constexpr int kKBlocks = 2;         // 256 B per row
    static constexpr bool kParked = true;      // top-2 bookkeeping by a parked chunk (see the epilogue)
    static constexpr int kEpiWarps = 16;       // 4 TMEM lane quarters x 4 column groups of 64
};
constexpr int kTcAccStride = 256;             // TMEM columns between the two accumulators
constexpr int kTcSfaCol = 240, kTcSfbCol = 496;   // TcF4: 16 columns of scale bytes after each accumulator
// TcF4 epilogue: one parked 32-value chunk per query row and column group (16 warps x 32 lanes x 128 B).
constexpr int kTcParkBytes = 16 * 32 * 128;
constexpr int kTcMergeBytes = 3 * 2048;   // (best, second, index) of up to three column groups, 128 rows x 4 ints each
template <class F> __host__ __device__ constexpr int tc_a_bytes() { return kTcM * kTcKBlock * F::kKBlocks; }   // 64 / 32 KiB
template <class F> __host__ __device__ constexpr int tc_stage_bytes() { return F::kN * kTcKBlock; }            // 32 / 30 KiB
template <class F> __host__ __device__ constexpr int tc_smem_bytes() {
    return tc_a_bytes<F>() + kTcStages * tc_stage_bytes<F>() + 1024 /*align*/ + 512 /*barriers*/ + kTcMergeBytes +
           (F::kParked ? kTcParkBytes : 0);
}

// ---------------------------------------------------------------- expansion ----
// Global layout of an expanded set, both forms: [K-block][8-row atom][1024 B] — the UMMA canonical K-major
// SWIZZLE_128B atom (8 rows x 128 B, 16-byte chunk index XOR row), K-block-major over the WHOLE set, so any run
// of rows (a 128-row query tile, a 240- or 256-row train tile, or half of one) is one contiguous block per
// K-block: plain 1-D TMA bulk copies, no tensor maps. One expansion serves a set as queries and as train rows.
// Rows >= n (padding up to whole tiles) are zero and are masked in the epilogue. One thread writes one 16-byte
// chunk: 16 bits of the descriptor as int8 (0xFF / 0x01), or 32 bits as e2m1 nibbles (0xA / 0x2).
template <class F>
__global__ void expand_kernel(const uint8_t* __restrict__ packed, unsigned long long n,
                              unsigned long long padded_rows, uint8_t* __restrict__ out) {
    constexpr int kChunks = F::kKBlocks * 8;           // 16-byte chunks per row
    pdl_launch_dependents();                           // the matcher's CTAs may start their set-up now
    const unsigned long long idx = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    const unsigned long long row = idx / kChunks;
    if (row >= padded_rows) return;
    const int chunk = static_cast<int>(idx - row * kChunks);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < n) {
        unsigned w[4];
        if (F::kF4) {
            const unsigned bits = *reinterpret_cast<const unsigned*>(packed + row * 64 + 4 * chunk);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                unsigned b = (bits >> (8 * i)) & 0xFFu, nib = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) nib |= ((b >> j) & 1u) << (4 * j + 3);
                w[i] = 0xAAAAAAAAu ^ nib;               // bit j -> nibble j: set 0x2 (+1.0), clear 0xA (-1.0)
            }
        } else {
            const unsigned bits = *reinterpret_cast<const unsigned short*>(packed + row * 64 + 2 * chunk);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const unsigned nib = (bits >> (4 * i)) & 0xF;
                // spread 4 bits to 4 bytes (0/1), then 1 -> 0x01 (+1), 0 -> 0xFF (-1)
                const unsigned ones = (nib * 0x00204081u) & 0x01010101u;
                w[i] = ((ones ^ 0x01010101u) * 0xFFu) | ones;
            }
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
    }
    const int kb = chunk >> 3, c = chunk & 7, ri = static_cast<int>(row & 7);
    const unsigned long long atoms = padded_rows >> 3, atom = static_cast<unsigned long long>(kb) * atoms + (row >> 3);
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
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// One lane of a converged warp (the same one every time on current hardware).
__device__ __forceinline__ bool elect_one() {
    unsigned pred;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.b32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Cluster-wide handshakes of the 2-CTA MMA form: the address of `addr` (an mbarrier of this CTA's layout) in the
// shared memory of CTA `rank`, an arrive on it, and a wait that also acquires what a remote arriver released.
__device__ __forceinline__ unsigned mapa_rank(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(unsigned cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TC_WAITC:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra TC_DONEC;\n"
        "bra TC_WAITC;\n"
        "TC_DONEC:\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
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
constexpr unsigned kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((TcI8::kN >> 3) << 17) | ((kTcM >> 4) << 24);
// Block-scaled descriptor (cute::UMMA::InstrDescriptorBlockScaled): A = B = E2M1 (MXF4Format 1 @7, @10), scale
// format UE8M0 (1 @23), scale-factor ids 0, N >> 3 @17, M >> 4 @24; K = 64 per instruction, D = f32.
constexpr unsigned kIdescF4 = (1u << 7) | (1u << 10) | (1u << 23) | ((TcF4::kN >> 3) << 17) | ((kTcM >> 4) << 24);
// D[tmem] (+)= A[smem] * B[smem]^T, e2m1 x e2m1 -> f32, one UE8M0 scale per 32 K-elements read from TMEM
// (all 0x7F = 2^0 here), M=128, N=240, K=64.
__device__ __forceinline__ void tc_mma_f4(unsigned tmem_d, uint64_t desc_a, uint64_t desc_b, unsigned idesc,
                                          unsigned accumulate, unsigned tmem_sfa, unsigned tmem_sfb) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb)
        : "memory");
}
// The same instruction over a CTA pair (cta_group::2): M = 256, each CTA contributes its 128 rows of A (same shared-
// memory offset in both) and HALF of the B tile (rows [120 rank, 120 rank + 120) at the same offset), each CTA's TMEM
// receives its own 128 accumulator rows; issued by the pair's rank-0 CTA only (tools/tc_pair_probe.cu checks the
// mapping and the rate: 16 382 MAC/clk/SM).
__device__ __forceinline__ void tc_mma_f4_pair(unsigned tmem_d, uint64_t desc_a, uint64_t desc_b, unsigned idesc,
                                               unsigned accumulate, unsigned tmem_sfa, unsigned tmem_sfb) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate), "r"(tmem_sfa), "r"(tmem_sfb)
        : "memory");
}
__device__ __forceinline__ void tc_commit_pair(unsigned bar) {   // ... arrives on `bar` of BOTH CTAs once the pair's MMAs are done
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"(static_cast<unsigned short>(3))
                 : "memory");
}
constexpr unsigned kIdescF4Pair = (1u << 7) | (1u << 10) | (1u << 23) | ((TcF4::kN >> 3) << 17) | ((256u >> 4) << 24);
// 16 TMEM columns of this warp's lane quarter <- one 32-bit value.
__device__ __forceinline__ void tmem_fill16(unsigned taddr, unsigned v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v)
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Issue only: the registers are valid after tmem_wait_ld().
__device__ __forceinline__ void tmem_ld32_issue(unsigned taddr, int (&v)[32]) {
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
}
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
    const uint8_t* a;     // expanded query set: K-block 0 of this tile's first atom
    const uint8_t* b;     // expanded train set
    unsigned long long a_kb_stride, b_kb_stride;   // bytes between K-blocks of the two sets (atoms x 1024)
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
    unsigned long long a_atoms, b_atoms;   // 8-row atoms per K-block of the two expanded sets
    int qtiles, total_tiles, tiles_per_split, num_items;
    int sk_chunks;           // > 0: "stream-K" partition of the (query tile, train tile) units over this many CTAs
    Partial* partial;
    int* dump;               // optional: raw accumulators of item 0's first tile, 128 x 256
    unsigned long long* trace;   // optional (CLATCH_TC_TRACE=1): 8 globaltimer stamps per CTA
    int debug;                   // CLATCH_TC_DEBUG bits (wrong results!): 1 = epilogue releases accumulators unread
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
template <class F, bool kPair>
__device__ __forceinline__ TcWork tc_decode(const TcArgs& g, int item, unsigned rank) {
    constexpr int kTcN = F::kN;
    constexpr unsigned long long kTileA = kTcM / 8 * 1024;     // bytes of one query tile inside a K-block
    TcWork w;
    w.ghost = false;
    w.a_kb_stride = g.a_atoms * 1024;
    w.b_kb_stride = g.b_atoms * 1024;
    if (g.items != nullptr) {
        const TcItem it = g.items[kPair ? 2 * item + static_cast<int>(rank) : item];
        w.ghost = it.ghost != 0;
        w.a_kb_stride = static_cast<unsigned long long>(it.a_atoms) * 1024;
        w.b_kb_stride = static_cast<unsigned long long>(it.b_atoms) * 1024;
        w.a = it.a_exp + static_cast<unsigned long long>(it.qtile) * kTileA;
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
        // kPair: the same cut over (query tile PAIR, train tile) units, one run per cluster — both CTAs of a cluster walk
        // the same train tiles for the two query tiles of the pair and share the stream by multicast.
        const unsigned long long QT = kPair ? (g.qtiles + 1) / 2 : g.qtiles;
        const unsigned long long U = QT * g.total_tiles;
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
        w.tile_begin = static_cast<int>(t0);
        w.ntiles = static_cast<int>(n);
        w.split = static_cast<int>(c - tc_sk_chunk_of(q * TT, U, G));   // pieces of a query tile (pair) in train order
        if (kPair) {
            q = 2 * q + rank;
            if (q >= static_cast<unsigned long long>(g.qtiles)) {       // odd tile count: the last pair's second CTA
                q = g.qtiles - 1;
                w.ghost = true;
            }
        }
        w.qtile = static_cast<unsigned>(q);
        w.a = g.a_exp + q * kTileA;
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
        w.a = g.a_exp + static_cast<unsigned long long>(w.qtile) * kTileA;
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
        w.a = g.a_exp + static_cast<unsigned long long>(w.qtile) * kTileA;
        w.b = g.b_exp;
        w.Q = g.Q;
        w.N = g.N;
        w.tile_begin = w.split * g.tiles_per_split;
        w.ntiles = min(g.total_tiles, w.tile_begin + g.tiles_per_split) - w.tile_begin;
        w.o_idx = w.o_best = w.o_second = nullptr;
    }
    return w;
}

// One 32-column chunk of one query row in the parked-chunk epilogue (see match_tc_kernel): `valid` columns of it are
// real train rows; `cb` is its column base inside the work item. Keeps the two largest chunk maxima seen by this lane
// (k1 >= k2 as monotonic integer keys, over distinct chunks, first come first on ties) and parks the raw values of the
// chunk that holds k1 (base c1) in shared memory.
__device__ __forceinline__ void tc_park_chunk(int (&v)[32], const int valid, const int cb, uint4* const my_park, int& k1, int& k2,
                                              int& c1, int* const dump, const int dump_cols) {
    if (dump != nullptr) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i < dump_cols) dump[i] = static_cast<int>(__int_as_float(v[i]));
    }
    if (valid < 32) {     // the set's last tile (zero padding rows) and the columns past the tile width
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i >= valid) v[i] = static_cast<int>(0xFF800000u);   // -inf
    }
    // 3-input integer max as a tree (depth 4), not a chain of 16 dependent steps
    int a[11];
#pragma unroll
    for (int i = 0; i < 10; ++i) a[i] = max(v[3 * i], max(v[3 * i + 1], v[3 * i + 2]));
    a[10] = max(v[30], v[31]);
    const int b0 = max(a[0], max(a[1], a[2])), b1 = max(a[3], max(a[4], a[5])), b2 = max(a[6], max(a[7], a[8])),
              b3 = max(a[9], a[10]);
    int m = max(max(b0, b1), max(b2, b3));
    if (__any_sync(0xffffffffu, m < 0)) {   // rare: a chunk without one non-negative value (or fully masked)
        float fm = __int_as_float(v[0]);
#pragma unroll
        for (int i = 1; i < 32; ++i) fm = fmaxf(fm, __int_as_float(v[i]));
        m = m < 0 ? __float_as_int(fm) : m;
    }
    const int key = m >= 0 ? m : (m ^ 0x7FFFFFFF);   // monotonic in the float value
    if (__any_sync(0xffffffffu, key > k2)) {
        if (key > k1) {                   // a new largest value for this row: its chunk replaces the parked one
#pragma unroll
            for (int i = 0; i < 8; ++i)
                my_park[32 * i] = make_uint4(static_cast<unsigned>(v[4 * i]), static_cast<unsigned>(v[4 * i + 1]),
                                             static_cast<unsigned>(v[4 * i + 2]), static_cast<unsigned>(v[4 * i + 3]));
            k2 = k1;
            k1 = key;
            c1 = cb;
        } else if (key > k2) {
            k2 = key;                     // only its maximum can matter (as the runner-up)
        }
    }
}

// kPair = true: launched as clusters of two CTAs. Every CTA used to pull the whole train stream out of L2 by
// itself — 64 B/clk/SM at the tensor pipe's pace, 9.5 KB/clk over 148 SMs, which is more than L2 delivers
// (tools/tc_peak.cu: ~4.3-6 KB/clk) and held the kernel at 72-77 % of the MMA rate. Paired CTAs work on two
// query tiles against the SAME train tiles: each loads half of every B stage and multicasts it into both
// CTAs' shared memory (one L2 read feeds two SMs), and a stage is handed back to the producers only when both
// CTAs' MMAs have read it (multicast tcgen05.commit onto both `empty` barriers).
// k2Cta (needs kPair and the e2m1 form; set_option "match_2cta", OFF by default): the pair runs ONE MMA stream of M = 256
// (tcgen05 cta_group::2) issued by its rank-0 CTA. Each CTA then loads only HALF of every B stage: per tile 32 KB of A
// reads + 30 KB of B reads + 30 KB of TMA writes = 92 KB through a CTA's shared-memory port instead of 152 KB. Measured
// (20 k x 1 M, profiles/r4g_match_2cta.log): results identical, and with no B traffic at all (CLATCH_TC_DEBUG=3) a tile
// takes 1 100 clk — the M = 256 MMAs and the handshakes are fine — but WITH the TMA stream 2 240 clk (2 500 with the
// epilogue off) against 1 400 for the multicast pairs, whether the ring has four or eight stages and whether the loads
// hit one L2-resident tile or stream the set. What the pair form changes is only WHEN the partner's half of B crosses
// between the SMs — at MMA time instead of as a prefetched multicast write; each SM still takes in 60 KB per tile, and
// the synchronous fetch next to the TMA fills is the slower of the two. Kept for A/B.
// Handshakes across the pair: the rank-1 CTA's MMA warp relays its "A landed" / "stage landed" barriers to rank 0
// (remote arrive), its epilogue warps hand accumulators back on rank 0's barrier, and every commit of the issuer
// arrives on both CTAs' barriers.
template <class F, bool kPair, bool k2Cta = false>
__global__ void __launch_bounds__(tc_threads<F>(), 1) match_tc_kernel(const TcArgs g) {
    static_assert(!k2Cta || (kPair && F::kF4), "the 2-CTA MMA form is built for paired CTAs and e2m1 operands");
    constexpr int kTcEpilogueWarps = F::kEpiWarps;
    constexpr int kTcN = F::kN, kTcKBlocks = F::kKBlocks;
    constexpr int kTcABytes = tc_a_bytes<F>(), kTcStageBytes = tc_stage_bytes<F>();
    const unsigned rank = kPair ? cluster_rank() : 0u;
    const int first_item = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int item_step = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
    extern __shared__ uint8_t smem_raw[];
    unsigned long long* const trace = g.trace ? g.trace + 8 * blockIdx.x : nullptr;
    if (trace && threadIdx.x == 0) trace[0] = global_ns();
    const unsigned raw = smem_u32(smem_raw);
    const unsigned base = (raw + 1023u) & ~1023u;              // SWIZZLE_128B atoms need 1024-B alignment
    const unsigned smem_a = base;
    const unsigned smem_b = base + kTcABytes;
    // The 2-CTA form keeps half a K-block of B per stage and CTA, so the same ring memory holds twice as many stages:
    // the operand loop (TMA latency + relay + MMAs + the commit's way back) is ~2 500 clk long, and with four stages in
    // flight it, not the tensor pipe, set the tile time (measured: 2 240 clk per tile).
    constexpr int kStages = k2Cta ? 2 * kTcStages : kTcStages;
    constexpr int kStageStride = k2Cta ? kTcStageBytes / 2 : kTcStageBytes;
    const unsigned bars = smem_b + kTcStages * kTcStageBytes;  // 8-byte mbarriers (512 bytes; the TMEM slot sits at +128)
    const unsigned bar_a_full = bars;
    const unsigned bar_a_empty = bars + 8;
    const unsigned bar_tfull = bars + 16;                      // [2]
    const unsigned bar_tempty = bars + 32;                     // [2]
    const unsigned bar_peer_a_full = bars + 48;                // 2-CTA form, rank 0: the partner's A tile has landed
    const unsigned bar_full = bars + 136;                      // [kStages]
    const unsigned bar_empty = bar_full + 8 * kStages;         // [kStages]
    const unsigned bar_peer_full = bar_empty + 8 * kStages;    // [kStages] 2-CTA form, rank 0: the partner's half of a stage has landed
    static_assert(136 + 3 * 8 * kStages <= 512, "barrier block");
    uint8_t* const gen_base = smem_raw + (base - raw);
    uint8_t* const tail = gen_base + kTcABytes + kTcStages * kTcStageBytes;
    volatile unsigned* tmem_slot = reinterpret_cast<volatile unsigned*>(tail + 128);
    int* merge_buf = reinterpret_cast<int*>(tail + 512);       // 128 rows x 4 ints
    uint4* const park = reinterpret_cast<uint4*>(tail + 512 + kTcMergeBytes);   // F::kParked: [16 warps][8 pieces][32 lanes] x uint4

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(bar_a_full, 1);
        mbar_init(bar_a_empty, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, kPair && !k2Cta ? 2 : 1);   // pair mode: both CTAs' MMAs must have read the stage
            mbar_init(bar_peer_full + 8 * s, 1);
        }
        mbar_init(bar_peer_a_full, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar_tfull + 8 * b, 1);
            mbar_init(bar_tempty + 8 * b, k2Cta ? 2 * kTcEpilogueWarps : kTcEpilogueWarps);   // 2-CTA form: both CTAs' epilogues
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {   // TMEM: all 512 columns (two 256-column accumulators)
        if (k2Cta) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                smem_u32(const_cast<unsigned*>(tmem_slot))));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                smem_u32(const_cast<unsigned*>(tmem_slot))));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (kPair) cluster_sync_all();                             // the partner's barriers exist before anything lands on them
    tc_fence_after();
    const unsigned tmem_base = *tmem_slot;
    if (F::kF4) {
        // Block scales: every byte of the 16 columns behind each accumulator is UE8M0 0x7F = 2^0, so whichever
        // cells the MMA reads for its 128 A rows and 240 B rows, each 32-element block is scaled by exactly 1.
        if (warp >= 2 && warp < 6) {
            const unsigned lanes = static_cast<unsigned>((warp & 3) * 32) << 16;
            tmem_fill16(tmem_base + lanes + kTcSfaCol, 0x7F7F7F7Fu);
            tmem_fill16(tmem_base + lanes + kTcSfbCol, 0x7F7F7F7Fu);
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }

    pdl_launch_dependents();                                   // (the merge kernel's blocks may take their seats)
    pdl_wait();                                                // the expanded operands are complete and visible
    if (trace && threadIdx.x == 0) trace[1] = global_ns();   // set-up done (barriers, TMEM, scale bytes)
    if (warp == 0) {
        // ===== producer =====
        if (lane == 0) {
            int stage = 0;
            unsigned phase = 0, a_phase = 0;
            for (int item = first_item; item < g.num_items; item += item_step) {
                const TcWork w = tc_decode<F, kPair>(g, item, rank);
                if (w.ntiles == 0) continue;                   // (stream-K: this CTA has fewer pieces)
                mbar_wait(bar_a_empty, a_phase ^ 1);           // previous item's MMAs are done with A
                mbar_expect_tx(bar_a_full, kTcABytes);
                for (int kb = 0; kb < kTcKBlocks; ++kb)        // 128 rows x 128 B of every K-block
                    bulk_load(smem_a + kb * (kTcM * kTcKBlock), w.a + kb * w.a_kb_stride, kTcM * kTcKBlock, bar_a_full);
                a_phase ^= 1;
                for (int t = 0; t < w.ntiles; ++t) {
                    // train tile = kTcN consecutive rows = kTcN / 8 consecutive atoms of every K-block
                    const uint8_t* src = w.b + static_cast<unsigned long long>((g.debug & 4) ? 0 : w.tile_begin + t) * (kTcN / 8 * 1024);   // (debug 4: one tile over and over — timing only)
                    for (int kb = 0; kb < kTcKBlocks; ++kb) {
                        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                        if ((g.debug & 2) || ((g.debug & 8) && (t & 1))) {   // measurement only (wrong results): no B
                                                                                          // traffic at all / for odd tiles (8)
                            mbar_arrive(bar_full + 8 * stage);
                            if (++stage == kStages) { stage = 0; phase ^= 1; }
                            continue;
                        }
                        mbar_expect_tx(bar_full + 8 * stage, k2Cta ? kTcStageBytes / 2 : kTcStageBytes);
                        const unsigned dst = smem_b + stage * kStageStride;
                        if (k2Cta) {   // this CTA's half of the tile's rows, for this CTA alone (the pair's MMA reads both)
                            bulk_load(dst, src + kb * w.b_kb_stride + rank * (kTcStageBytes / 2), kTcStageBytes / 2,
                                      bar_full + 8 * stage);
                        } else if (kPair) {   // this CTA's half of the stage, to both CTAs
                            bulk_load_multicast(dst + rank * (kTcStageBytes / 2),
                                                src + kb * w.b_kb_stride + rank * (kTcStageBytes / 2), kTcStageBytes / 2,
                                                bar_full + 8 * stage, 3);
                        } else {
                            bulk_load(dst, src + kb * w.b_kb_stride, kTcStageBytes, bar_full + 8 * stage);
                        }
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        // The WHOLE warp walks the loop, converged, and one elected lane issues the tensor-core instructions: with
        // warp-uniform control flow the descriptor arithmetic stays on the uniform datapath. Issued from a lone
        // `lane == 0` thread every MMA cost ~20 instructions of register -> uniform-register shuffling, ~250 per tile,
        // and at the ~7 clk per instruction a single warp gets next to four busy epilogue warps on its scheduler that
        // chain (not the tensor pipe, not shared memory) set the tile time: 1 700 clk against 960 clk of MMAs.
        int stage = 0, tcount = 0;
        unsigned phase = 0, a_phase = 0;
        const unsigned sfa = tmem_base + kTcSfaCol, sfb = tmem_base + kTcSfbCol;
        if (k2Cta && rank != 0) {
            // The partner of the issuing CTA: relay "my A tile / my half of a stage has landed" to rank 0.
            const unsigned r_a = mapa_rank(bar_peer_a_full, 0), r_full = mapa_rank(bar_peer_full, 0);
            for (int item = first_item; item < g.num_items; item += item_step) {
                const TcWork w = tc_decode<F, kPair>(g, item, rank);
                if (w.ntiles == 0) continue;
                mbar_wait(bar_a_full, a_phase);
                a_phase ^= 1;
                if (lane == 0) mbar_arrive_cluster(r_a);
                for (int t = 0; t < w.ntiles; ++t, ++tcount) {
#pragma unroll
                    for (int kb = 0; kb < kTcKBlocks; ++kb) {
                        mbar_wait(bar_full + 8 * stage, phase);
                        if (lane == 0) mbar_arrive_cluster(r_full + 8 * stage);
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                }
                __syncwarp();
            }
        } else
        for (int item = first_item; item < g.num_items; item += item_step) {
            const TcWork w = tc_decode<F, kPair>(g, item, rank);
            if (w.ntiles == 0) continue;
            mbar_wait(bar_a_full, a_phase);
            if (k2Cta) mbar_wait_cluster(bar_peer_a_full, a_phase);
            a_phase ^= 1;
            for (int t = 0; t < w.ntiles; ++t, ++tcount) {
                const int buf = tcount & 1;
                if (k2Cta) mbar_wait_cluster(bar_tempty + 8 * buf, ((tcount >> 1) & 1) ^ 1);   // both CTAs' epilogues drained it
                else mbar_wait(bar_tempty + 8 * buf, ((tcount >> 1) & 1) ^ 1);   // epilogue drained this accumulator
                tc_fence_after();
                const unsigned tmem_d = tmem_base + buf * kTcAccStride;
#pragma unroll
                for (int kb = 0; kb < kTcKBlocks; ++kb) {
                    mbar_wait(bar_full + 8 * stage, phase);
                    if (k2Cta) mbar_wait_cluster(bar_peer_full + 8 * stage, phase);
                    if (trace && tcount == 0 && kb == 0 && lane == 0) trace[2] = global_ns();   // first operand stage has landed
                    tc_fence_after();
                    const uint64_t a_desc = umma_desc(smem_a + kb * (kTcM * kTcKBlock));
                    const uint64_t b_desc = umma_desc(smem_b + stage * kStageStride);
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < kTcKBlock / 32; ++k) {   // 32 bytes of K per instruction: 32 int8 or 64 e2m1
                            // (start address field counts 16-byte units: + 2 per 32 bytes of K)
                            if (k2Cta) tc_mma_f4_pair(tmem_d, a_desc + 2 * k, b_desc + 2 * k, kIdescF4Pair, (kb | k) != 0, sfa, sfb);
                            else if (F::kF4) tc_mma_f4(tmem_d, a_desc + 2 * k, b_desc + 2 * k, kIdescF4, (kb | k) != 0, sfa, sfb);
                            else tc_mma_i8(tmem_d, a_desc + 2 * k, b_desc + 2 * k, kIdescI8, (kb | k) != 0);
                        }
                        if (k2Cta) tc_commit_pair(bar_empty + 8 * stage);
                        else if (kPair) tc_commit_multicast(bar_empty + 8 * stage, 3);
                        else tc_commit(bar_empty + 8 * stage);  // stage reusable once these MMAs have read it
                        if (kb == kTcKBlocks - 1) {             // accumulator complete (in both CTAs' TMEM)
                            if (k2Cta) tc_commit_pair(bar_tfull + 8 * buf);
                            else tc_commit(bar_tfull + 8 * buf);
                        }
                    }
                    __syncwarp();
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
            if (elect_one()) {                                 // every MMA of this item has read A
                if (k2Cta) tc_commit_pair(bar_a_empty);
                else tc_commit(bar_a_empty);
            }
            __syncwarp();
        }
        if (trace && lane == 0) {
            trace[3] = global_ns();   // last MMA issued
            trace[6] = static_cast<unsigned long long>(tcount);
        }
    } else {
        // ===== epilogue: warps 2.. =====
        const int ew = warp - 2;
        // hand an accumulator back to the MMA issuer — which, in the 2-CTA form, is the pair's rank-0 CTA
        const unsigned r_tempty = k2Cta ? mapa_rank(bar_tempty, 0) : 0u;
        auto tempty_arrive = [&](int buf) {
            if (k2Cta) mbar_arrive_cluster(r_tempty + 8 * buf);
            else mbar_arrive(bar_tempty + 8 * buf);
        };
        const int quarter = warp & 3;                       // TMEM lane quarter this warp may touch
        const int half = ew >> 2;                           // int8 form: which 128 of the 256 columns
        const unsigned lane_addr = static_cast<unsigned>(quarter * 32) << 16;
        const int row = quarter * 32 + lane;
        int tcount = 0;
        for (int item = first_item; item < g.num_items; item += item_step) {
            const TcWork w = tc_decode<F, kPair>(g, item, rank);
            if (w.ntiles == 0) continue;
            int best, second, best_idx = -1;
            if constexpr (F::kParked) {
                // Top-2 by a PARKED CHUNK. Examining 32 accumulators one by one whenever a chunk might change a row's
                // top-2 costs ~160 instructions for the whole warp each time one lane needs it, and with n columns
                // seen a lane needs it with probability ~64/n per chunk: over an 8 000-row train set (an image pair)
                // or a stream-K piece nearly every chunk took that pass. Here a lane tracks only the two largest CHUNK
                // MAXIMA it has seen (k1 >= k2, distinct chunks, first come first on ties) and keeps the 32 raw values
                // of the chunk holding k1 in shared memory (8 predicated 16-byte stores when a chunk's maximum beats
                // k1). Every value outside that chunk is <= k2: the row's largest value is the first maximum of the
                // parked chunk, and its second-largest is k2 or the parked chunk's own runner-up — one exact pass over
                // 32 parked values at the end of the item gives the same (index, best, second) as examining
                // everything. Keys: f32 bits order like signed integers among non-negative values; a negative chunk
                // maximum (all 32 distances above 256) is re-derived with float compares and mapped monotonically.
                // Sixteen epilogue warps (four per scheduler): the epilogue is latency-bound — ~100 instructions per
                // chunk at ~7 clk each — and eight warps needed 1 850 clk per 240-column tile against 960 clk of MMAs.
                const int colgrp = ew >> 2;                                // columns [64 * colgrp, 64 * colgrp + 64)
                int k1 = INT_MIN, k2 = INT_MIN, c1 = -1;
                uint4* const my_park = park + ew * (32 * 8) + lane;   // [warp][16-byte piece i][lane]: a warp's stores of one piece are contiguous
                const bool dumping = g.dump != nullptr && item == 0 && rank == 0;
                for (int t = 0; t < w.ntiles; ++t, ++tcount) {
                    const int buf = tcount & 1;
                    mbar_wait(bar_tfull + 8 * buf, (tcount >> 1) & 1);
                    tc_fence_after();
                    const long long left = static_cast<long long>(w.N) - static_cast<long long>(w.tile_begin + t) * kTcN;
                    const int tile_valid = left < kTcN ? static_cast<int>(left) : kTcN;   // real rows among this tile's columns
                    const unsigned acc = tmem_base + lane_addr + buf * kTcAccStride + colgrp * 64;
                    if (g.debug & 1) {   // measurement only: how fast is everything BUT the epilogue?
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) tempty_arrive(buf);
                        continue;
                    }
#pragma unroll
                    for (int chunk = 0; chunk < 2; ++chunk) {
                        const int ccol = colgrp * 64 + chunk * 32;   // first column of this chunk inside the tile
                        int v[32];
                        tmem_ld32(acc + chunk * 32, v);
                        if (chunk == 1) {   // everything this warp needs of the accumulator has left TMEM
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) tempty_arrive(buf);
                        }
                        tc_park_chunk(v, tile_valid - ccol, t * kTcN + ccol, my_park, k1, k2, c1,
                                      dumping && t == 0 ? g.dump + row * 256 + ccol : nullptr, kTcN - ccol);
                    }
                }
                // the exact pass over the parked chunk
                float fbest = __int_as_float(0xFF800000u), fsecond = fbest;
                if (c1 >= 0) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint4 q = my_park[32 * i];
                        const unsigned e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float f = __uint_as_float(e[j]);
                            if (f > fbest) {                      // strict: the lower index keeps ties
                                fsecond = fbest;
                                fbest = f;
                                best_idx = c1 + 4 * i + j;
                            } else if (f > fsecond) {
                                fsecond = f;
                            }
                        }
                    }
                    if (k2 != INT_MIN) fsecond = fmaxf(fsecond, __int_as_float(k2 >= 0 ? k2 : (k2 ^ 0x7FFFFFFF)));
                }
                best = __float_as_int(fbest);
                second = __float_as_int(fsecond);
            } else {
                // best / second are dot products D = 512 - 2 * hamming, kept as the raw accumulator words: int32, or the
                // bits of an f32 holding that integer. Signed-integer order on f32 bits is the float order among
                // non-negative values and puts every negative value below them, so the per-chunk test (3-input integer
                // max over the 32 words against the runner-up) is exact whenever the runner-up is >= 0 (second_key =
                // its bits); until then second_key = INT_MIN and every chunk takes the full pass, which compares as floats.
                best = F::kF4 ? static_cast<int>(0xFF800000u) : INT_MIN;   // -inf / INT_MIN
                second = best;
                int second_key = INT_MIN;
                for (int t = 0; t < w.ntiles; ++t, ++tcount) {
                    const int buf = tcount & 1;
                    mbar_wait(bar_tfull + 8 * buf, (tcount >> 1) & 1);
                    tc_fence_after();
                    const long long tile_col0 = static_cast<long long>(w.tile_begin + t) * kTcN;
                    const long long tile_valid = min(static_cast<long long>(kTcN), static_cast<long long>(w.N) - tile_col0);
    #pragma unroll 1
                    for (int chunk = 0; chunk < 4; ++chunk) {
                        const int ccol = half * 128 + chunk * 32;   // first column of this chunk inside the tile
                        if (ccol >= kTcN) break;
                        int v[32];
                        tmem_ld32(tmem_base + lane_addr + buf * kTcAccStride + ccol, v);
                        if (g.dump != nullptr && item == 0 && t == 0 && rank == 0) {
    #pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (ccol + i < kTcN)
                                    g.dump[row * 256 + ccol + i] = F::kF4 ? static_cast<int>(__int_as_float(v[i])) : v[i];
                        }
                        const long long cvalid = tile_valid - ccol;
                        if (cvalid < 32) {     // the set's last tile (zero padding rows) and the columns past kTcN
    #pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (i >= cvalid) v[i] = F::kF4 ? static_cast<int>(0xFF800000u) : INT_MIN;   // -inf
                        }
                        int m = v[0];
    #pragma unroll
                        for (int i = 1; i < 32; i += 2) m = max(m, max(v[i], i + 1 < 32 ? v[i + 1] : INT_MIN));
                        if (m > second_key) {                       // something in this chunk may enter the top-2
                            const int cbase = t * kTcN + ccol;
    #pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                const int d = v[i];
                                const bool gt_best = F::kF4 ? __int_as_float(d) > __int_as_float(best) : d > best;
                                const bool gt_second = F::kF4 ? __int_as_float(d) > __int_as_float(second) : d > second;
                                if (gt_best) {                      // strict: earlier (lower) index keeps ties
                                    second = best;
                                    best = d;
                                    best_idx = cbase + i;
                                } else if (gt_second) {
                                    second = d;
                                }
                            }
                            second_key = !F::kF4 ? second : (__int_as_float(second) >= 0.f ? second : INT_MIN);
                        }
                    }
                    // (All four loads in flight at once, with the accumulator handed back to the MMA issuer before the
                    // chunks are examined, was measured 2.5x SLOWER in both forms: 1 M x 1 M 3.06e12 vs 5.12e12 compares/s.)
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) tempty_arrive(buf);
                }
            }
            if (F::kF4) {   // f32 bits -> the integer they hold (-inf: nothing seen)
                best = __int_as_float(best) > -1024.f ? static_cast<int>(__int_as_float(best)) : INT_MIN;
                second = __int_as_float(second) > -1024.f ? static_cast<int>(__int_as_float(second)) : INT_MIN;
            }
            // merge the column groups of each row (two halves, or four groups of 64 in the parked form): the groups
            // interleave in index order across tiles, so ties compare indices
            constexpr int kGroups = kTcEpilogueWarps / 4;
            const int grp = ew >> 2;
            if (grp != 0) {
                int* const mb = merge_buf + (grp - 1) * 512 + row * 4;
                mb[0] = best;
                mb[1] = second;
                mb[2] = best_idx;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(32 * kTcEpilogueWarps) : "memory");
            if (grp == 0) {
#pragma unroll
                for (int o = 1; o < kGroups; ++o) {
                    const int* const mb = merge_buf + (o - 1) * 512 + row * 4;
                    const int ob = mb[0], os = mb[1], oi = mb[2];
                    if (ob > best || (ob == best && oi >= 0 && oi < best_idx)) {
                        second = max(best, os);
                        best = ob;
                        best_idx = oi;
                    } else {
                        second = max(second, ob);
                    }
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

    if (trace && threadIdx.x == 64) trace[4] = global_ns();   // first epilogue warp finished its last item
    tc_fence_before();
    __syncthreads();
    if (trace && threadIdx.x == 0) trace[5] = global_ns();
    if (kPair) cluster_sync_all();                             // nothing of the partner's is still bound for this CTA
    if (warp == 1) {
        tc_fence_after();
        if (k2Cta) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

} // namespace

namespace {

// Merge of the stream-K pieces: query tile q was cut into the chunks c_first(q) .. c_last(q), whose
// partials sit in slots 0 .. c_last - c_first in ascending train order (same rule as
// merge_partials_kernel: strictly better wins, so the earlier piece keeps ties).
__global__ void merge_partials_sk_kernel(const Partial* __restrict__ partial, unsigned long long Q, int total_tiles,
                                         int qtiles, int chunks, int pair_shift, int32_t* __restrict__ best_idx,
                                         int32_t* __restrict__ best_dist, int32_t* __restrict__ second_dist) {
    pdl_wait();                                                // every partial of the GEMM launch is in place
    const unsigned long long qi = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (qi >= Q) return;
    // (pair_shift = 1: the cut ran over query tile PAIRS, `qtiles` counts pairs)
    const unsigned long long U = static_cast<unsigned long long>(qtiles) * total_tiles, TT = total_tiles, q = (qi / kTcM) >> pair_shift;
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
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel<TcI8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<TcI8>()));
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel<TcI8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<TcI8>()));
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel<TcF4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<TcF4>()));
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel<TcF4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<TcF4>()));
        CLATCH_CUDA(cudaFuncSetAttribute(match_tc_kernel<TcF4, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes<TcF4>()));
        ctx->tc_configured = true;
    }
    return CLATCH_OK;
}

static int tc_tile_rows(const clatch_ctx* ctx) { return ctx->match_variant == 4 ? TcF4::kN : TcI8::kN; }
static size_t tc_row_bytes(const clatch_ctx* ctx) { return ctx->match_variant == 4 ? 256 : 512; }

// Rows an expanded set is padded to: whole train tiles AND whole 128-row query tiles of the current form.
size_t tc_padded_rows(const clatch_ctx* ctx, size_t rows) {
    const size_t n = tc_tile_rows(ctx);
    return std::max((rows + n - 1) / n * n, (rows + kTcM - 1) / kTcM * kTcM);
}
size_t tc_expanded_bytes(const clatch_ctx* ctx, size_t rows) { return tc_padded_rows(ctx, rows) * tc_row_bytes(ctx); }
int tc_format(const clatch_ctx* ctx) { return ctx->match_variant == 4 ? 4 : 8; }

int launch_tc_expand(clatch_ctx* ctx, const uint8_t* d_packed, size_t n, uint8_t* d_out, cudaStream_t stream) {
    const unsigned long long rows = tc_padded_rows(ctx, n);
    if (rows == 0) return CLATCH_OK;
    if (ctx->match_variant == 4) {
        const unsigned long long threads = rows * (TcF4::kKBlocks * 8);
        expand_kernel<TcF4><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(d_packed, n, rows, d_out);
    } else {
        const unsigned long long threads = rows * (TcI8::kKBlocks * 8);
        expand_kernel<TcI8><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(d_packed, n, rows, d_out);
    }
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

int tc_query_tiles(size_t rows) { return static_cast<int>((rows + kTcM - 1) / kTcM); }

// One launch of the kernel in the context's operand form; `paired` = clusters of two CTAs; `pdl` = may start while the
// expansion kernel queued just before it is still running (it waits for it after its own set-up).
static int launch_tc(clatch_ctx* ctx, const TcArgs& g, unsigned ctas, bool paired, cudaStream_t stream, bool pdl = false) {
    const bool f4 = ctx->match_variant == 4;
    const dim3 grid(paired ? (ctas & ~1u) : ctas), block(f4 ? tc_threads<TcF4>() : tc_threads<TcI8>());
    const size_t smem = f4 ? tc_smem_bytes<TcF4>() : tc_smem_bytes<TcI8>();
    const unsigned cluster = paired ? 2 : 1;
    pdl = pdl && ctx->pdl;
    cudaError_t e;
    if (f4) e = paired ? (ctx->match_2cta ? launch_kernel(match_tc_kernel<TcF4, true, true>, grid, block, smem, stream, pdl, cluster, g)
                                          : launch_kernel(match_tc_kernel<TcF4, true>, grid, block, smem, stream, pdl, cluster, g))
                       : launch_kernel(match_tc_kernel<TcF4, false>, grid, block, smem, stream, pdl, cluster, g);
    else e = paired ? launch_kernel(match_tc_kernel<TcI8, true>, grid, block, smem, stream, pdl, cluster, g)
                    : launch_kernel(match_tc_kernel<TcI8, false>, grid, block, smem, stream, pdl, cluster, g);
    CLATCH_CUDA(e);
    ++ctx->launches;
    return CLATCH_OK;
}

int launch_match_tc_items(clatch_ctx* ctx, const TcItem* d_items, size_t count, cudaStream_t stream) {
    if (count == 0) return CLATCH_OK;
    if (int rc = configure_tc(ctx)) return rc;
    TcArgs g{};
    g.items = d_items;
    const unsigned ctas = static_cast<unsigned>(std::min<size_t>(count, ctx->sm_count));
    if (ctx->match_pairs) {   // the table holds entries (2k, 2k + 1) that scan the same train set (tc_items_paired)
        g.num_items = static_cast<int>(count / 2);
        return launch_tc(ctx, g, ctas, true, stream);
    }
    g.num_items = static_cast<int>(count);
    return launch_tc(ctx, g, ctas, false, stream);
}

bool tc_items_paired(const clatch_ctx* ctx) { return ctx->match_pairs; }

static int match_top2_tc_impl(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                              int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second, cudaStream_t stream,
                              int32_t* d_dump);

int launch_match_top2_tc(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                         int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second, cudaStream_t stream,
                         int32_t* d_dump) {
    // Operand form per call under match_variant 4 (A/B switch, off by default): before the parked-chunk epilogue the
    // int8 kernel was ~10 % ahead between 8 k and 20 k squared, where top-2 bookkeeping of short runs dominated.
    const int saved = ctx->match_variant;
    const double work = static_cast<double>(Q) * static_cast<double>(N);
    if (saved == 4 && ctx->match_form_auto && work >= 3e7 && work <= 6e8) ctx->match_variant = 3;
    const int rc = match_top2_tc_impl(ctx, d_q, Q, d_t, N, d_best_idx, d_best_dist, d_second, stream, d_dump);
    ctx->match_variant = saved;
    return rc;
}

static int match_top2_tc_impl(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                              int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second, cudaStream_t stream,
                              int32_t* d_dump) {
    if (int rc = configure_tc(ctx)) return rc;
    const size_t kTcN = tc_tile_rows(ctx);
    const size_t qtiles = (Q + kTcM - 1) / kTcM, ttiles = (N + kTcN - 1) / kTcN;
    // Both sets go to the tensor cores in the expanded form; a self-match expands its one set once.
    const bool self = d_q == d_t && Q == N;
    if (int rc = ctx->exp_t.reserve(tc_expanded_bytes(ctx, N))) return rc;
    if (int rc = launch_tc_expand(ctx, d_t, N, ctx->exp_t.as<uint8_t>(), stream)) return rc;
    const uint8_t* a_exp = ctx->exp_t.as<uint8_t>();
    if (!self) {
        if (int rc = ctx->exp_q.reserve(tc_expanded_bytes(ctx, Q))) return rc;
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
    // With CTA pairs (match_pairs) the units are (query tile pair, train tile) and a run belongs to a cluster of two CTAs
    // that share the train stream by multicast: on its own a CTA pulls 60 KB per tile out of L2 and is bound by that
    // (1.17 us per tile at 10 k x 10 k against 0.72 us for paired CTAs at scale).
    const size_t sms = static_cast<size_t>(ctx->sm_count);
    const bool sk_pairs = ctx->match_pairs && ctx->match_streamk_pairs && qtiles >= 2 && sms >= 2;
    const size_t sk_q = sk_pairs ? (qtiles + 1) / 2 : qtiles, sk_slots = sk_pairs ? sms / 2 : sms;
    const size_t units = sk_q * ttiles, chunks = std::min(units, sk_slots);
    bool streamk = false;
    size_t sk_pieces_per_cta = 1, sk_pieces_per_qtile = 1;
    if (tc_expanded_bytes(ctx, N) <= (32u << 20) && units > 0 && ctx->match_streamk) {
        const size_t share = (units + chunks - 1) / chunks;                 // tile-times per CTA
        sk_pieces_per_cta = (share + ttiles - 2) / ttiles + 1;
        sk_pieces_per_qtile = (ttiles + units / chunks - 1) / (units / chunks) + 1;
        const size_t rounds = (qtiles * splits + sms - 1) / sms;
        // (in tile-times of an unpaired CTA; a paired tile takes ~0.65 of one)
        const double legacy = rounds * (per_split + 1.5), sk = (share + 2.0 * sk_pieces_per_cta) * (sk_pairs ? 0.65 : 1.0);   // (measured: tools/sk_perf.py)
        streamk = sk < legacy;
    }
    // Otherwise pairs of CTAs share the train stream (match_tc_kernel<true>): the schedulable unit is a pair of
    // query tiles on a pair of SMs, so the split count is chosen again in those units.
    const bool paired = !streamk && ctx->match_pairs && qtiles >= 2 && sms >= 2;
    const bool sk_paired = streamk && sk_pairs;
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
    g.a_atoms = tc_padded_rows(ctx, self ? N : Q) / 8;
    g.b_atoms = tc_padded_rows(ctx, N) / 8;
    g.qtiles = static_cast<int>(qtiles);
    g.total_tiles = static_cast<int>(ttiles);
    g.tiles_per_split = static_cast<int>(per_split);
    g.num_items = static_cast<int>(streamk ? chunks * sk_pieces_per_cta : qtiles * splits);
    g.sk_chunks = streamk ? static_cast<int>(chunks) : 0;
    g.partial = ctx->partial.as<Partial>();
    g.dump = d_dump;
    static const bool tracing = std::getenv("CLATCH_TC_TRACE") != nullptr;
    static const int debug_bits = std::getenv("CLATCH_TC_DEBUG") ? std::atoi(std::getenv("CLATCH_TC_DEBUG")) : 0;
    g.debug = debug_bits;
    unsigned long long* d_trace = nullptr;
    if (tracing) {
        CLATCH_CUDA(cudaMalloc(&d_trace, sizeof(unsigned long long) * 8 * sms));
        CLATCH_CUDA(cudaMemsetAsync(d_trace, 0, sizeof(unsigned long long) * 8 * sms, stream));
        g.trace = d_trace;
    }
    if (sk_paired) {   // g.num_items = clusters x pieces: item = cluster + piece * clusters
        if (int rc = launch_tc(ctx, g, static_cast<unsigned>(2 * chunks), true, stream, !tracing)) return rc;
    } else if (paired) {
        const size_t pair_items = (qtiles + 1) / 2 * splits;
        g.num_items = static_cast<int>(pair_items);
        if (int rc = launch_tc(ctx, g, static_cast<unsigned>(std::min<size_t>(2 * pair_items, sms)), true, stream, !tracing)) return rc;
    } else {
        const unsigned grid = static_cast<unsigned>(streamk ? chunks : std::min<size_t>(qtiles * splits, ctx->sm_count));
        if (int rc = launch_tc(ctx, g, grid, false, stream, !tracing)) return rc;
    }
    if (tracing) {   // debug: where the time of a launch goes, per CTA (globaltimer, ns)
        std::vector<unsigned long long> h(8 * sms);
        CLATCH_CUDA(cudaStreamSynchronize(stream));
        CLATCH_CUDA(cudaMemcpy(h.data(), d_trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
        cudaFree(d_trace);
        unsigned long long t0 = ~0ull, t_end = 0;
        for (size_t c = 0; c < sms; ++c)
            if (h[8 * c]) t0 = std::min(t0, h[8 * c]), t_end = std::max(t_end, h[8 * c + 5]);
        double sum[6] = {0}, mx[6] = {0};
        size_t n = 0;
        for (size_t c = 0; c < sms; ++c) {
            if (!h[8 * c]) continue;
            ++n;
            for (int k = 0; k < 6; ++k) {
                const double v = (static_cast<double>(h[8 * c + k]) - static_cast<double>(t0)) / 1e3;
                sum[k] += v;
                mx[k] = std::max(mx[k], v);
            }
        }
        std::fprintf(stderr, "[clatch tc trace] %s Q=%zu N=%zu ctas=%zu tiles/cta=%llu total %.1f us | mean (max) us since first CTA start: "
                     "entry %.1f (%.1f), setup done %.1f (%.1f), first stage landed %.1f (%.1f), last MMA issued %.1f (%.1f), "
                     "epilogue done %.1f (%.1f), exit %.1f (%.1f)\n",
                     sk_paired ? "stream-K pairs" : streamk ? "stream-K" : paired ? "paired" : "rounds", Q, N, n, h[6], (t_end - t0) / 1e3, sum[0] / n, mx[0], sum[1] / n,
                     mx[1], sum[2] / n, mx[2], sum[3] / n, mx[3], sum[4] / n, mx[4], sum[5] / n, mx[5]);
    }
    if (streamk)
        CLATCH_CUDA(launch_kernel(merge_partials_sk_kernel, dim3(static_cast<unsigned>((Q + 255) / 256)), dim3(256), 0, stream,
                                  ctx->pdl && !tracing, 1, static_cast<const Partial*>(ctx->partial.as<Partial>()),
                                  static_cast<unsigned long long>(Q), static_cast<int>(ttiles), static_cast<int>(sk_q),
                                  static_cast<int>(chunks), sk_paired ? 1 : 0, d_best_idx, d_best_dist, d_second));
    else
        launch_merge_partials(ctx->partial.as<Partial>(), Q, static_cast<int>(splits), 513, d_best_idx, d_best_dist,
                              d_second, stream, ctx->pdl && !tracing);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

} // namespace clatch
