// Brute-force Hamming top-2 matching for sm_100a — exact restatement of the
// reference (paths relative to /root/reference/proj):
//   hamming   src/match.cpp:14-31   XOR + popcount over the descriptor bytes
//   knn2      src/match.cpp:33-50   best / runner-up, strict '<' => lowest index wins ties,
//                                   sentinel 8*bytes+1
// Pure integer work, so any evaluation order is exact as long as ties resolve
// toward the lowest train index.
//
// Tiled kernel (64-byte descriptors): one query per thread held in 16 registers;
// the train set streams through a double-buffered shared-memory tile filled by the
// TMA bulk-copy engine (cp.async.bulk + mbarrier); every thread reads the same train
// descriptor with four broadcast 128-bit shared loads. POPC issues on the 16-lane/clk XU
// pipe, which the plain XOR+__popc form saturates (profiles/r1a_match_ncu.json: XU 93.7 %
// active, ALU 38 %), so the 16 XOR words are first compressed with carry-save adders
// (two LOP3 each, on the 64-lane ALU pipe) into words of weight 1, 2 (and 4) and only
// those are popcounted: 9 (or 7) POPC per 512-bit compare instead of 16. Top-2 selection
// runs on packed keys (distance << 21 | local index): min/max only, lowest index wins
// ties by construction. The train set is split across blockIdx.y so small query sets still fill 148 SMs; a
// second tiny kernel merges the per-split partial top-2 (splits are ascending index
// ranges, so "earlier split wins ties" keeps the lowest index).

#include <algorithm>

#include "clatch_internal.cuh"

namespace clatch {

namespace {

constexpr int kMatchThreads = 128;   // queries per CTA
constexpr int kTileDesc = 128;       // train descriptors per shared-memory tile (8 KiB)
constexpr int kDescBytes = 64;
constexpr int kDescWords = 16;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_LOOP:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra WAIT_DONE;\n"
        "bra WAIT_LOOP;\n"
        "WAIT_DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine (SASS: UBLKCP).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Carry-save adder: three words of weight w -> one of weight w (sum) + one of weight 2w (carry).
__device__ __forceinline__ void csa(unsigned& sum, unsigned& carry, unsigned a, unsigned b, unsigned c) {
    sum = a ^ b ^ c;                        // LOP3 0x96
    carry = (a & b) | (a & c) | (b & c);    // LOP3 0xE8
}

// Hamming distance of two 512-bit descriptors. kVariant 0: 16 POPC. 1: 7 CSA + 9 POPC.
// 2: 9 CSA + 7 POPC. All exact (integer identities).
template <int kVariant>
__device__ __forceinline__ unsigned hamming16(const unsigned (&q)[kDescWords], const uint4* t) {
    unsigned x[kDescWords];
#pragma unroll
    for (int i = 0; i < kDescWords / 4; ++i) {
        const uint4 v = t[i];   // same address in every lane: one broadcast wavefront
        x[4 * i + 0] = q[4 * i + 0] ^ v.x;
        x[4 * i + 1] = q[4 * i + 1] ^ v.y;
        x[4 * i + 2] = q[4 * i + 2] ^ v.z;
        x[4 * i + 3] = q[4 * i + 3] ^ v.w;
    }
    if (kVariant == 0) {
        unsigned d = 0;
#pragma unroll
        for (int i = 0; i < kDescWords; ++i) d += __popc(x[i]);
        return d;
    }
    unsigned o[7], w2[9];
    csa(o[0], w2[0], x[0], x[1], x[2]);
    csa(o[1], w2[1], x[3], x[4], x[5]);
    csa(o[2], w2[2], x[6], x[7], x[8]);
    csa(o[3], w2[3], x[9], x[10], x[11]);
    csa(o[4], w2[4], x[12], x[13], x[14]);
    csa(o[5], w2[5], o[0], o[1], o[2]);
    csa(o[6], w2[6], o[3], o[4], x[15]);
    const unsigned ones = __popc(o[5]) + __popc(o[6]);
    if (kVariant == 1) {
        const unsigned twos = __popc(w2[0]) + __popc(w2[1]) + __popc(w2[2]) + __popc(w2[3]) +
                              __popc(w2[4]) + __popc(w2[5]) + __popc(w2[6]);
        return ones + 2 * twos;
    }
    unsigned w4[2];
    csa(w2[7], w4[0], w2[0], w2[1], w2[2]);
    csa(w2[8], w4[1], w2[3], w2[4], w2[5]);
    const unsigned twos = __popc(w2[6]) + __popc(w2[7]) + __popc(w2[8]);
    const unsigned fours = __popc(w4[0]) + __popc(w4[1]);
    return ones + 2 * twos + 4 * fours;
}

constexpr int kKeyShift = 21;                       // local train index bits inside a packed key
constexpr unsigned kKeyIndexMask = (1u << kKeyShift) - 1;

// grid = (ceil(Q/128), splits). Split s scans train rows [s*per_split, min(N, (s+1)*per_split)).
template <int kVariant>
__global__ void __launch_bounds__(kMatchThreads) match64_kernel(const uint8_t* __restrict__ queries,
                                                                unsigned long long Q,
                                                                const uint8_t* __restrict__ train,
                                                                unsigned long long N,
                                                                unsigned long long per_split,
                                                                Partial* __restrict__ partial) {
    __shared__ __align__(128) uint4 s_tile[2][kTileDesc * kDescBytes / 16];
    __shared__ __align__(8) uint64_t s_bar[2];

    const int tid = threadIdx.x;
    const unsigned long long qi = static_cast<unsigned long long>(blockIdx.x) * kMatchThreads + tid;
    const unsigned long long n_begin = static_cast<unsigned long long>(blockIdx.y) * per_split;
    const unsigned long long n_end = min(N, n_begin + per_split);
    const int tiles = static_cast<int>((n_end - n_begin + kTileDesc - 1) / kTileDesc);

    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int tile) {   // thread 0 only
        const unsigned long long first = n_begin + static_cast<unsigned long long>(tile) * kTileDesc;
        const unsigned count = static_cast<unsigned>(min(static_cast<unsigned long long>(kTileDesc), n_end - first));
        const unsigned bytes = count * kDescBytes;
        uint64_t* bar = &s_bar[tile & 1];
        mbar_expect_tx(bar, bytes);
        bulk_load(s_tile[tile & 1], train + first * kDescBytes, bytes, bar);
    };
    if (tid == 0 && tiles > 0) issue(0);

    unsigned q[kDescWords];
    {
        const unsigned long long src = qi < Q ? qi : Q - 1;   // tail threads shadow the last query
        const uint4* qp = reinterpret_cast<const uint4*>(queries + src * kDescBytes);
#pragma unroll
        for (int i = 0; i < kDescWords / 4; ++i) {
            const uint4 v = __ldg(qp + i);
            q[4 * i + 0] = v.x;
            q[4 * i + 1] = v.y;
            q[4 * i + 2] = v.z;
            q[4 * i + 3] = v.w;
        }
    }

    // Packed keys: (distance << 21) | index inside this split. Scanning with min/max keeps
    // the two smallest keys; equal distances order by index, so the lowest index wins
    // (knn2's strict '<', src/match.cpp:41-47) and the runner-up may tie the best.
    const unsigned sentinel_key = (static_cast<unsigned>(8 * kDescBytes + 1) << kKeyShift) | kKeyIndexMask;
    unsigned best_key = sentinel_key, second_key = sentinel_key;

    for (int tile = 0; tile < tiles; ++tile) {
        if (tid == 0 && tile + 1 < tiles) issue(tile + 1);   // buffer (tile+1)&1 was released by the
                                                             // __syncthreads closing iteration tile-1
        mbar_wait(&s_bar[tile & 1], (tile >> 1) & 1);
        const int count = static_cast<int>(
            min(static_cast<unsigned long long>(kTileDesc), n_end - n_begin - static_cast<unsigned long long>(tile) * kTileDesc));
        const uint4* t = s_tile[tile & 1];
        const unsigned base = static_cast<unsigned>(tile) * kTileDesc;
#pragma unroll 4
        for (int j = 0; j < count; ++j) {
            const unsigned d = hamming16<kVariant>(q, t + j * (kDescBytes / 16));
            const unsigned key = (d << kKeyShift) + (base + j);
            second_key = min(second_key, max(best_key, key));
            best_key = min(best_key, key);
        }
        __syncthreads();   // everyone is done with this buffer before it is refilled
    }

    if (qi < Q) {
        Partial r;
        r.best_idx = best_key == sentinel_key ? -1 : static_cast<int>(n_begin + (best_key & kKeyIndexMask));
        r.best_dist = static_cast<int>(best_key >> kKeyShift);
        r.second_dist = static_cast<int>(second_key >> kKeyShift);
        r.pad = 0;
        partial[static_cast<unsigned long long>(blockIdx.y) * Q + qi] = r;
    }
}

// Merge per-split partials in ascending split order (== ascending index ranges).
__global__ void merge_partials_kernel(const Partial* __restrict__ partial, unsigned long long Q,
                                      int splits, int sentinel, int32_t* __restrict__ best_idx,
                                      int32_t* __restrict__ best_dist, int32_t* __restrict__ second_dist) {
    pdl_wait();   // (launched early behind the tensor-core matcher: its partials are complete from here on)
    const unsigned long long qi = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (qi >= Q) return;
    int best = sentinel, second = sentinel, idx = -1;
    for (int s = 0; s < splits; ++s) {
        const Partial r = partial[static_cast<unsigned long long>(s) * Q + qi];
        if (r.best_dist < best) {          // strictly better: earlier splits keep ties
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

// Any descriptor length (byte tail included, src/match.cpp:28-29): one query per
// thread, operands straight from global memory through L1. Correctness path for
// non-64-byte descriptors, not a tuned one.
__global__ void match_generic_kernel(const uint8_t* __restrict__ queries, unsigned long long Q,
                                     const uint8_t* __restrict__ train, unsigned long long N, int bytes,
                                     int32_t* __restrict__ best_idx, int32_t* __restrict__ best_dist,
                                     int32_t* __restrict__ second_dist) {
    const unsigned long long qi = blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
    if (qi >= Q) return;
    const uint8_t* q = queries + qi * bytes;
    const int sentinel = 8 * bytes + 1;
    int best = sentinel, second = sentinel, idx = -1;
    for (unsigned long long g = 0; g < N; ++g) {
        const uint8_t* t = train + g * bytes;
        int d = 0;
        for (int i = 0; i < bytes; ++i) d += __popc(static_cast<unsigned>(q[i] ^ __ldg(t + i)));
        if (d < best) {
            second = best;
            best = d;
            idx = static_cast<int>(g);
        } else if (d < second) {
            second = d;
        }
    }
    if (best_idx) best_idx[qi] = idx;
    if (best_dist) best_dist[qi] = best;
    if (second_dist) second_dist[qi] = second;
}

} // namespace

// ---- filter pass of match_brute_force on the device (src/match.cpp:69-79), for batched set pairs ----
// One CTA per pair walks its probes in order: ratio test in double exactly as the reference writes
// it (best < ratio * second, int -> double), inclusive max distance, cross-check against the
// reverse pass; kept rows [probe, gallery, distance, second] are written in ascending probe order
// to the pair's own (worst-case sized) slice, and the count is recorded. A one-block scan and a
// copy kernel then pack the slices back to back, so only the surviving rows cross the bus.
__global__ void __launch_bounds__(256) filter_pairs_kernel(const FilterPair* __restrict__ pairs, int has_ratio,
                                                           double ratio, int has_max, int max_distance,
                                                           int4* __restrict__ rows, unsigned* __restrict__ kept) {
    const FilterPair fp = pairs[blockIdx.x];
    __shared__ unsigned s_warp[8];
    __shared__ unsigned s_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned base = 0;
    int4* const out = rows + fp.out_base;
    for (unsigned p0 = 0; p0 < fp.n; p0 += 256) {
        const unsigned p = p0 + threadIdx.x;
        bool keep = false;
        int best = 0, second = 0, idx = 0;
        if (p < fp.n) {
            best = fp.best_dist[p];
            second = fp.second_dist[p];
            idx = fp.best_idx[p];
            keep = true;
            if (has_ratio && !(static_cast<double>(best) < __dmul_rn(ratio, static_cast<double>(second)))) keep = false;
            if (keep && has_max && best > max_distance) keep = false;
            if (keep && fp.reverse_best != nullptr && fp.reverse_best[idx] != static_cast<int>(p)) keep = false;
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_warp[warp] = __popc(ballot);
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned run = 0;
            for (int w = 0; w < 8; ++w) {
                const unsigned c = s_warp[w];
                s_warp[w] = run;
                run += c;
            }
            s_total = run;
        }
        __syncthreads();
        if (keep) out[base + s_warp[warp] + __popc(ballot & ((1u << lane) - 1u))] = make_int4(static_cast<int>(p), idx, best, second);
        base += s_total;
        __syncthreads();
    }
    if (threadIdx.x == 0) kept[blockIdx.x] = base;
}

// Exclusive scan of the per-pair counts (a few thousand at most): one block, 1024 entries per step.
__global__ void __launch_bounds__(1024) scan_counts_kernel(const unsigned* __restrict__ kept, unsigned count,
                                                           unsigned long long* __restrict__ offsets) {
    __shared__ unsigned s_w[32];
    __shared__ unsigned long long s_run;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_run = 0;
    __syncthreads();
    for (unsigned i0 = 0; i0 < count; i0 += 1024) {
        const unsigned i = i0 + tid;
        const unsigned v = i < count ? kept[i] : 0;
        unsigned x = v;
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned t = s_w[lane];
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, t, d);
                if (lane >= d) t += y;
            }
            s_w[lane] = t;
        }
        __syncthreads();
        const unsigned warp_before = warp ? s_w[warp - 1] : 0;
        const unsigned long long run = s_run;
        if (i < count) offsets[i] = run + warp_before + x - v;
        __syncthreads();   // everyone has read s_run and s_w
        if (tid == 1023) s_run = run + warp_before + x;
        __syncthreads();
    }
    if (tid == 0) offsets[count] = s_run;
}

__global__ void compact_rows_kernel(const FilterPair* __restrict__ pairs, const int4* __restrict__ rows,
                                    const unsigned long long* __restrict__ offsets, int4* __restrict__ out) {
    const FilterPair fp = pairs[blockIdx.x];
    const unsigned long long begin = offsets[blockIdx.x], n = offsets[blockIdx.x + 1] - begin;
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) out[begin + i] = rows[fp.out_base + i];
}

int launch_filter_pairs(clatch_ctx* ctx, const FilterPair* d_pairs, size_t count, int has_ratio, double ratio, int has_max,
                        int max_distance, int32_t* d_rows, unsigned* d_kept, unsigned long long* d_offsets,
                        int32_t* d_out, cudaStream_t stream) {
    if (count == 0) return CLATCH_OK;
    filter_pairs_kernel<<<static_cast<unsigned>(count), 256, 0, stream>>>(d_pairs, has_ratio, ratio, has_max, max_distance,
                                                                           reinterpret_cast<int4*>(d_rows), d_kept);
    scan_counts_kernel<<<1, 1024, 0, stream>>>(d_kept, static_cast<unsigned>(count), d_offsets);
    compact_rows_kernel<<<static_cast<unsigned>(count), 256, 0, stream>>>(d_pairs, reinterpret_cast<const int4*>(d_rows),
                                                                          d_offsets, reinterpret_cast<int4*>(d_out));
    ctx->launches += 3;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

void launch_merge_partials(const Partial* partial, unsigned long long Q, int splits, int sentinel,
                           int32_t* best_idx, int32_t* best_dist, int32_t* second_dist, cudaStream_t stream, bool pdl) {
    launch_kernel(merge_partials_kernel, dim3(static_cast<unsigned>((Q + 255) / 256)), dim3(256), 0, stream, pdl, 1, partial, Q,
                  splits, sentinel, best_idx, best_dist, second_dist);
}

static int match_top2_on(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                         int bytes, int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second,
                         cudaStream_t stream);

// The matcher's operands and partials (exp_q, exp_t, partial) are context scratch: order this use
// behind the previous one when it ran on another stream.
int launch_match_top2(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                      int bytes, int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second,
                      cudaStream_t stream) {
    if (Q == 0) return CLATCH_OK;
    if (int rc = scratch_acquire(ctx, stream)) return rc;
    if (int rc = match_top2_on(ctx, d_q, Q, d_t, N, bytes, d_best_idx, d_best_dist, d_second, stream)) return rc;
    return scratch_release(ctx, stream);
}

static int match_top2_on(clatch_ctx* ctx, const uint8_t* d_q, size_t Q, const uint8_t* d_t, size_t N,
                         int bytes, int32_t* d_best_idx, int32_t* d_best_dist, int32_t* d_second,
                         cudaStream_t stream) {
    const bool tiled = bytes == kDescBytes && reinterpret_cast<uintptr_t>(d_q) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(d_t) % 16 == 0;
    if (!tiled) {
        const unsigned blocks = static_cast<unsigned>((Q + 127) / 128);
        match_generic_kernel<<<blocks, 128, 0, stream>>>(d_q, Q, d_t, N, bytes, d_best_idx, d_best_dist,
                                                         d_second);
        ++ctx->launches;
        CLATCH_CUDA(cudaGetLastError());
        return CLATCH_OK;
    }
    if (ctx->match_variant >= 3)   // 3: int8, 4: e2m1 operands on the tensor cores
        return launch_match_top2_tc(ctx, d_q, Q, d_t, N, d_best_idx, d_best_dist, d_second, stream);
    const size_t qblocks = (Q + kMatchThreads - 1) / kMatchThreads;
    // Enough CTAs for ~8 resident per SM, but never a split shorter than two tiles.
    const size_t want = static_cast<size_t>(ctx->sm_count) * 8;
    size_t splits = std::max<size_t>(1, (want + qblocks - 1) / qblocks);
    const size_t max_splits = std::max<size_t>(1, N / (2 * kTileDesc));
    splits = std::min(splits, std::min<size_t>(max_splits, 65535));
    splits = std::max(splits, (N + kKeyIndexMask - 1) / kKeyIndexMask);   // local index must fit the key
    size_t per_split = (N + splits - 1) / splits;
    per_split = (per_split + kTileDesc - 1) / kTileDesc * kTileDesc;
    splits = (N + per_split - 1) / per_split;

    if (int rc = ctx->partial.reserve(sizeof(Partial) * splits * Q)) return rc;
    Partial* partial = ctx->partial.as<Partial>();
    dim3 grid(static_cast<unsigned>(qblocks), static_cast<unsigned>(splits));
    switch (ctx->match_variant) {
        case 0: match64_kernel<0><<<grid, kMatchThreads, 0, stream>>>(d_q, Q, d_t, N, per_split, partial); break;
        case 2: match64_kernel<2><<<grid, kMatchThreads, 0, stream>>>(d_q, Q, d_t, N, per_split, partial); break;
        default: match64_kernel<1><<<grid, kMatchThreads, 0, stream>>>(d_q, Q, d_t, N, per_split, partial); break;
    }
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    merge_partials_kernel<<<static_cast<unsigned>((Q + 255) / 256), 256, 0, stream>>>(
        partial, Q, static_cast<int>(splits), 8 * bytes + 1, d_best_idx, d_best_dist, d_second);
    ++ctx->launches;
    CLATCH_CUDA(cudaGetLastError());
    return CLATCH_OK;
}

} // namespace clatch
