// tcgen05 issue-rate microbenchmark for B200 (sm_100a): the tensor-pipe roofline the Hamming matcher is
// measured against, with the SM clock recorded next to every figure.
//   kind::i8      int8 x int8 -> int32   (the matcher up to r2c)
//   kind::f8f6f4  e4m3 x e4m3 -> f16 / f32 accumulators
// One CTA per SM; one thread issues M128 N256 K32 MMAs back to back from (zeroed) shared-memory operands in
// the canonical K-major SWIZZLE_128B layout, committing to an mbarrier every 16 (one 512-deep tile), with no
// epilogue at all. Prints one JSON object: T-op/s from CUDA events, MACs/clk/SM from clock64, and the SM clock
// each kernel actually ran at (clock64 ticks / globaltimer ns).
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
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D;\nbra W;\nD:\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// KIND 0: i8 -> s32; 1: f8f6f4 e4m3 -> f16; 2: f8f6f4 e4m3 -> f32; 3: mxf4 (e2m1, UE8M0 block scales = 1.0, K = 64) -> f32
// `stream_src` != nullptr: warp 1 keeps `depth` 16 KiB cp.async.bulk copies (global/L2 -> shared) in flight for the
// whole run — the operand traffic of a real GEMM mainloop (one 32 KiB B stage per 4 MMAs = 64 B/clk) without any
// dependency on it — to show what concurrent TMA writes into shared memory cost the SS-mode MMA stream.
template <int KIND>
__global__ void __launch_bounds__(128, 1) tc_rate_kernel(int tiles, unsigned long long* cycles, unsigned long long* nanos,
                                                          const uint8_t* stream_src, int depth, unsigned long long* copied) {
    extern __shared__ uint8_t raw[];
    const unsigned base = (smem_u32(raw) + 1023u) & ~1023u;
    const unsigned smem_a = base, smem_b = base + 16384, bar = base + 16384 + 32768, slot = bar + 16;
    const unsigned ring = base + 65536, ring_bar = bar + 64;   // 8 x 16 KiB landing buffers + their mbarriers
    volatile unsigned* done_flag = reinterpret_cast<volatile unsigned*>(raw + (bar + 32 - smem_u32(raw)));
    for (unsigned i = threadIdx.x * 16; i < 16384 + 32768; i += blockDim.x * 16)
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + i), "r"(0));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ring_bar + 8 * i));
        *done_flag = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(slot));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    unsigned tmem;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(tmem) : "r"(slot));
    // idesc: D format @4 (0 f16, 1 f32, 2 s32), A/B formats @7/@10 (i8: 1 = s8; f8f6f4: 0 = e4m3), N>>3 @17, M>>4 @24
    constexpr unsigned idesc = (KIND == 0 ? (2u << 4) | (1u << 7) | (1u << 10) : KIND == 1 ? 0u : KIND == 2 ? (1u << 4)
                                : (1u << 7) | (1u << 10) | (1u << 23)) |      // mxf4: A = B = E2M1 (MXF4Format 1), scale format UE8M0
                               ((256u >> 3) << 17) | ((128u >> 4) << 24);
    if (KIND == 3 && threadIdx.x < 128) {   // scale factors: every byte of TMEM columns 256..287 = 0x7F (2^0), whatever the layout
        const unsigned addr = tmem + ((threadIdx.x & ~31u) << 16) + 256;
        const unsigned one = 0x7F7F7F7Fu;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr), "r"(one));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 32 && stream_src != nullptr) {
        unsigned long long n = 0;
        const uint8_t* src = stream_src + static_cast<size_t>(blockIdx.x) * (1u << 20);   // 1 MiB window per CTA: L2 hits
        unsigned phase[8] = {0};
        for (int i = 0; i < depth; ++i) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ring_bar + 8 * i), "r"(16384) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(ring + 16384 * i),
                         "l"(src + 16384 * (n++ & 63)), "r"(16384), "r"(ring_bar + 8 * i)
                         : "memory");
        }
        while (*done_flag == 0) {
            for (int i = 0; i < depth; ++i) {
                mbar_wait(ring_bar + 8 * i, phase[i]);
                phase[i] ^= 1;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ring_bar + 8 * i), "r"(16384) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(ring + 16384 * i),
                             "l"(src + 16384 * (n++ & 63)), "r"(16384), "r"(ring_bar + 8 * i)
                             : "memory");
            }
        }
        for (int i = 0; i < depth; ++i) mbar_wait(ring_bar + 8 * i, phase[i]);
        copied[blockIdx.x] = n * 16384;
    }
    if (threadIdx.x == 0) {
        unsigned long long n0, n1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n0));
        const long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            const unsigned d = KIND == 3 ? tmem : tmem + (t & 1) * 256;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint64_t da = umma_desc(smem_a + 32 * (k & 3)), db = umma_desc(smem_b + 32 * (k & 3));
                const unsigned acc = k != 0;
                if (KIND == 3)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(d),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 272)
                                 : "memory");
                else if (KIND == 0)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc)
                                 : "memory");
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc)
                                 : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
        mbar_wait(bar, 0);
        const long long t1 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n1));
        cycles[blockIdx.x] = t1 - t0;
        nanos[blockIdx.x] = n1 - n0;
        *done_flag = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

struct Res { double tops, mac_per_clk_sm, mhz, ms, copy_bytes_per_clk_sm; };

template <int KIND>
Res run(int sms, int tiles, unsigned long long* d_cyc, unsigned long long* d_ns, const uint8_t* stream_src = nullptr, int depth = 0) {
    const int smem = 65536 + 8 * 16384 + 1024;
    unsigned long long* d_copied;
    CK(cudaMalloc(&d_copied, 8 * sms));
    CK(cudaMemset(d_copied, 0, 8 * sms));
    CK(cudaFuncSetAttribute(tc_rate_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    tc_rate_kernel<KIND><<<sms, 128, smem>>>(tiles, d_cyc, d_ns, stream_src, depth, d_copied);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        tc_rate_kernel<KIND><<<sms, 128, smem>>>(tiles, d_cyc, d_ns, stream_src, depth, d_copied);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    std::vector<unsigned long long> cyc(sms), ns(sms);
    CK(cudaMemcpy(cyc.data(), d_cyc, 8 * sms, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ns.data(), d_ns, 8 * sms, cudaMemcpyDeviceToHost));
    std::sort(cyc.begin(), cyc.end());
    std::vector<double> mhz(sms);
    double cmax = static_cast<double>(cyc.back());
    for (int i = 0; i < sms; ++i) mhz[i] = 0;
    std::vector<unsigned long long> cyc2(sms);
    CK(cudaMemcpy(cyc2.data(), d_cyc, 8 * sms, cudaMemcpyDeviceToHost));
    for (int i = 0; i < sms; ++i) mhz[i] = cyc2[i] * 1e3 / static_cast<double>(ns[i]);
    std::sort(mhz.begin(), mhz.end());
    const double macs = static_cast<double>(tiles) * 16 * 128 * 256 * (KIND == 3 ? 64 : 32);   // per SM
    Res r;
    r.ms = best;
    r.tops = 2.0 * macs * sms / (best * 1e-3) / 1e12;
    r.mac_per_clk_sm = macs / cmax;
    r.mhz = mhz[sms / 2];
    std::vector<unsigned long long> cp(sms);
    CK(cudaMemcpy(cp.data(), d_copied, 8 * sms, cudaMemcpyDeviceToHost));
    r.copy_bytes_per_clk_sm = static_cast<double>(cp[0]) / static_cast<double>(cyc2[0]);
    CK(cudaFree(d_copied));
    return r;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    unsigned long long *d_cyc, *d_ns;
    CK(cudaMalloc(&d_cyc, 8 * sms));
    CK(cudaMalloc(&d_ns, 8 * sms));
    const int tiles = 4000;   // 4000 x 16 MMAs = 8.2 M clk at the 128 clk/MMA floor = 4 ms
    const Res i8 = run<0>(sms, tiles, d_cyc, d_ns);
    const Res f8h = run<1>(sms, tiles, d_cyc, d_ns);
    const Res f8s = run<2>(sms, tiles, d_cyc, d_ns);
    uint8_t* d_src;
    CK(cudaMalloc(&d_src, static_cast<size_t>(sms) << 20));
    CK(cudaMemset(d_src, 0, static_cast<size_t>(sms) << 20));
    Res tr[4];
    const int depths[4] = {1, 2, 4, 8};
    for (int i = 0; i < 4; ++i) tr[i] = run<0>(sms, tiles, d_cyc, d_ns, d_src, depths[i]);
    const Res f4 = run<3>(sms, tiles, d_cyc, d_ns);
    // sustained: ~0.3 s per launch, the length of the 1 M x 1 M match — long enough for the power cap to pull the clock down
    const Res i8_long = run<0>(sms, 75 * tiles, d_cyc, d_ns);
    const Res f4_long = run<3>(sms, 75 * tiles, d_cyc, d_ns);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    printf("{\"device\": \"%s\", \"sm_count\": %d, \"max_sm_mhz\": %.0f,\n", prop.name, sms, khz / 1e3);
    printf(" \"i8_s32_tops\": %.1f, \"i8_s32_mac_per_clk_sm\": %.1f, \"i8_s32_sm_mhz\": %.0f, \"i8_s32_ms\": %.3f,\n", i8.tops,
           i8.mac_per_clk_sm, i8.mhz, i8.ms);
    printf(" \"e4m3_f16_tops\": %.1f, \"e4m3_f16_mac_per_clk_sm\": %.1f, \"e4m3_f16_sm_mhz\": %.0f, \"e4m3_f16_ms\": %.3f,\n", f8h.tops,
           f8h.mac_per_clk_sm, f8h.mhz, f8h.ms);
    printf(" \"e4m3_f32_tops\": %.1f, \"e4m3_f32_mac_per_clk_sm\": %.1f, \"e4m3_f32_sm_mhz\": %.0f, \"e4m3_f32_ms\": %.3f,\n", f8s.tops,
           f8s.mac_per_clk_sm, f8s.mhz, f8s.ms);
    printf(" \"mxf4_f32_tops\": %.1f, \"mxf4_f32_mac_per_clk_sm\": %.1f, \"mxf4_f32_sm_mhz\": %.0f, \"mxf4_f32_ms\": %.3f,\n", f4.tops,
           f4.mac_per_clk_sm, f4.mhz, f4.ms);
    printf(" \"sustained_0.3s\": {\"i8_s32_tops\": %.1f, \"i8_s32_sm_mhz\": %.0f, \"i8_s32_ms\": %.1f, \"mxf4_f32_tops\": %.1f, \"mxf4_f32_sm_mhz\": %.0f, \"mxf4_f32_ms\": %.1f},\n",
           i8_long.tops, i8_long.mhz, i8_long.ms, f4_long.tops, f4_long.mhz, f4_long.ms);
    for (int i = 0; i < 4; ++i)
        printf(" \"i8_s32_with_tma_depth%d\": {\"tops\": %.1f, \"mac_per_clk_sm\": %.1f, \"tma_bytes_per_clk_sm\": %.1f, \"sm_mhz\": %.0f},\n",
               depths[i], tr[i].tops, tr[i].mac_per_clk_sm, tr[i].copy_bytes_per_clk_sm, tr[i].mhz);
    printf(" \"how\": \"tools/tc_peak.cu: %d CTAs (one per SM), one thread issuing %d x 16 tcgen05.mma M128 N256 K32 from shared memory, "
           "no epilogue; T-op/s = 2 x MACs / best-of-5 CUDA-event time; sm_mhz = clock64 ticks / globaltimer ns, median over SMs\"}\n",
           sms, tiles);
    return 0;
}
