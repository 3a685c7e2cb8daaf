// tcgen05 cta_group::2 probe for B200 (sm_100a): one block-scaled FP4 MMA of M = 256 over a CTA pair
// (kind::mxf4, e2m1 +-1 operands, unit UE8M0 scales, f32 accumulators), N = 240 with each CTA holding HALF of B.
//   check: operands whose rows are uniform (+1 or -1 everywhere, so neither swizzle nor K order matters) with
//          row-dependent signs -> D[m][n] = 256 * sign_a(m) * sign_b(n); both CTAs read their 128 accumulator rows
//          back and the host verifies which rows / columns landed where.
//   rate:  the leader issues `tiles` x 8 MMAs (two K-blocks of 4) back to back, no epilogue; MACs/clk/SM.
// Prints one JSON object.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t umma_desc(unsigned smem_addr) {
    return static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ bool mbar_wait_bounded(unsigned bar, unsigned parity, long long max_clk) {
    const long long t0 = clock64();
    unsigned ok = 0;
    while (!ok) {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.b32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (!ok && clock64() - t0 > max_clk) return false;
    }
    return true;
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int kN = 240, kNHalf = kN / 2, kSfaCol = 240, kSfbCol = 496;
// block-scaled idesc: A = B = E2M1 (1 @7, 1 @10), UE8M0 scales (1 @23), N >> 3 @17, M >> 4 @24 — M = 256 over the pair
constexpr unsigned kIdesc = (1u << 7) | (1u << 10) | (1u << 23) | ((kN >> 3) << 17) | ((256u >> 4) << 24);

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
pair_probe_kernel(int tiles, float* out /* [2][128][256] */, unsigned long long* cycles, int* status) {
    extern __shared__ uint8_t raw[];
    const unsigned base = (smem_u32(raw) + 1023u) & ~1023u;
    uint8_t* const gen = raw + (base - smem_u32(raw));
    const unsigned smem_a = base, smem_b = base + 2 * 16384, bar = smem_b + 2 * 16384, slot = bar + 16;
    const unsigned rank = cluster_rank();
    // A: 2 K-blocks x 128 rows x 128 B; B half: 2 K-blocks x 120 rows x 128 B (16 KiB apart). Uniform rows.
    for (int i = threadIdx.x; i < 2 * 128 * 8; i += blockDim.x) {        // 16-byte chunks of A
        const int kb = i / (128 * 8), row = (i / 8) % 128;
        const unsigned gm = rank * 128 + row;
        const unsigned v = (gm % 5 == 0) ? 0xAAAAAAAAu : 0x22222222u;
        reinterpret_cast<uint4*>(gen + kb * 16384)[i % (128 * 8)] = make_uint4(v, v, v, v);
    }
    for (int i = threadIdx.x; i < 2 * 128 * 8; i += blockDim.x) {        // ... of B (rows >= 120 unused)
        const int kb = i / (128 * 8), row = (i / 8) % 128;
        const unsigned gn = rank * kNHalf + row;
        const unsigned v = row >= kNHalf ? 0u : (gn % 3 == 0) ? 0xAAAAAAAAu : 0x22222222u;
        reinterpret_cast<uint4*>(gen + 2 * 16384 + kb * 16384)[i % (128 * 8)] = make_uint4(v, v, v, v);
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(slot));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    unsigned tmem;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(slot));
    {   // scale factors: every byte of the 16 columns behind each accumulator = 0x7F (2^0), all 128 lanes, both CTAs
        const unsigned lanes = (threadIdx.x & ~31u) << 16, one = 0x7F7F7F7Fu;
        for (int c = 0; c < 2; ++c) {
            const unsigned addr = tmem + lanes + (c ? kSfbCol : kSfaCol);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr), "r"(one) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();            // both CTAs' operands, barriers and scale bytes are in place
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    long long t0 = 0, t1 = 0;
    if (rank == 0 && threadIdx.x == 0) {
        t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t da = umma_desc(smem_a + (k >> 2) * 16384 + 32 * (k & 3));
                const uint64_t db = umma_desc(smem_b + (k >> 2) * 16384 + 32 * (k & 3));
                const unsigned acc = k != 0;
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                             "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(tmem),
                             "l"(da), "l"(db), "r"(kIdesc), "r"(acc), "r"(tmem + kSfaCol), "r"(tmem + kSfbCol)
                             : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                     "h"(static_cast<unsigned short>(3))
                     : "memory");
    }
    // every thread of both CTAs waits for the commit on its own CTA's barrier
    const bool ok = mbar_wait_bounded(bar, 0, 2000000000ll);
    if (rank == 0 && threadIdx.x == 0) {
        t1 = clock64();
        cycles[blockIdx.x >> 1] = static_cast<unsigned long long>(t1 - t0);
    }
    if (!ok) {
        if (threadIdx.x == 0) atomicExch(status, 1);
    } else if (out != nullptr && blockIdx.x < 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned lanes = (threadIdx.x & ~31u) << 16;
        for (int c0 = 0; c0 < 256; c0 += 16) {
            unsigned v[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
                           "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(tmem + lanes + c0)
                         : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 16; ++i) out[(rank * 128 + threadIdx.x) * 256 + c0 + i] = __uint_as_float(v[i]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount & ~1;
    const int smem = 4 * 16384 + 2048;
    CK(cudaFuncSetAttribute(pair_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float* d_out;
    unsigned long long* d_cyc;
    int* d_status;
    CK(cudaMalloc(&d_out, sizeof(float) * 2 * 128 * 256));
    CK(cudaMalloc(&d_cyc, 8 * sms));
    CK(cudaMalloc(&d_status, 4));
    CK(cudaMemset(d_status, 0, 4));
    CK(cudaMemset(d_out, 0, sizeof(float) * 2 * 128 * 256));
    // 1. correctness: one cluster, one tile
    pair_probe_kernel<<<2, 128, smem>>>(1, d_out, d_cyc, d_status);
    CK(cudaDeviceSynchronize());
    std::vector<float> out(2 * 128 * 256);
    int status = 0;
    CK(cudaMemcpy(out.data(), d_out, sizeof(float) * out.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&status, d_status, 4, cudaMemcpyDeviceToHost));
    long long bad = 0, first_bad = -1;
    for (int gm = 0; gm < 256; ++gm)
        for (int gn = 0; gn < kN; ++gn) {
            const float want = 512.0f * ((gm % 5 == 0) ? -1.f : 1.f) * ((gn % 3 == 0) ? -1.f : 1.f);
            if (out[gm * 256 + gn] != want) {
                if (first_bad < 0) first_bad = gm * 256 + gn;
                ++bad;
            }
        }
    printf("{\"device\": \"%s\", \"timeout\": %d, \"mismatches\": %lld, \"first_bad\": %lld,\n", prop.name, status, bad, first_bad);
    printf(" \"sample\": [%.0f, %.0f, %.0f, %.0f, %.0f, %.0f, %.0f, %.0f],\n", out[0], out[1], out[3], out[119], out[120], out[123],
           out[128 * 256], out[130 * 256 + 121]);
    if (first_bad >= 0)
        printf(" \"first_bad_value\": %.1f, \"first_bad_row\": %lld, \"first_bad_col\": %lld,\n", out[first_bad], first_bad / 256, first_bad % 256);
    // 2. rate: all SMs as pairs
    if (bad == 0 && status == 0) {
        const int tiles = 4000;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
        pair_probe_kernel<<<sms, 128, smem>>>(tiles, nullptr, d_cyc, d_status);
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(e0));
            pair_probe_kernel<<<sms, 128, smem>>>(tiles, nullptr, d_cyc, d_status);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = std::min(best, ms);
        }
        std::vector<unsigned long long> cyc(sms / 2);
        CK(cudaMemcpy(cyc.data(), d_cyc, 8 * (sms / 2), cudaMemcpyDeviceToHost));
        std::sort(cyc.begin(), cyc.end());
        const double macs_pair = static_cast<double>(tiles) * 8 * 256 * kN * 64;   // per CTA pair
        printf(" \"pair_mxf4_tops\": %.1f, \"mac_per_clk_sm\": %.1f, \"ms\": %.3f,\n", 2.0 * macs_pair * (sms / 2) / (best * 1e-3) / 1e12,
               macs_pair / 2 / static_cast<double>(cyc.back()), best);
    }
    printf(" \"how\": \"tools/tc_pair_probe.cu: tcgen05.mma.cta_group::2.kind::mxf4.block_scale, M256 N240 K64, each CTA holds half of B\"}\n");
    return 0;
}
