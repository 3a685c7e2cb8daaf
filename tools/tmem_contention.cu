// Does the tensor core's accumulator traffic slow down tcgen05.ld? (B200, sm_100a)
// 8 epilogue-like warps loop over tcgen05.ld.32x32b.x32 + wait::ld on accumulator buffer 1 (columns 256..511)
// while one thread issues kind::mxf4 M128 N240 K64 MMAs back to back into buffer 0 (columns 0..239) — and, for
// reference, the same loads with the MMA thread idle. Prints clk per x32 load per warp in both cases and the
// MMA rate with and without the loads.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t umma_desc(unsigned a) {
    return static_cast<uint64_t>((a & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void __launch_bounds__(288, 1) probe(int iters, int mma_on, int ld_on, unsigned long long* ld_cycles,
                                                unsigned long long* mma_cycles, unsigned* sink) {
    extern __shared__ uint8_t raw[];
    const unsigned base = (smem_u32(raw) + 1023u) & ~1023u;
    const unsigned smem_a = base, smem_b = base + 16384, bar = base + 16384 + 32768, slot = bar + 16;
    volatile unsigned* done = reinterpret_cast<volatile unsigned*>(raw + (bar + 32 - smem_u32(raw)));
    for (unsigned i = threadIdx.x * 16; i < 16384 + 32768; i += blockDim.x * 16)
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + i), "r"(0x22222222));   // e2m1 +1.0 everywhere
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        *done = 0;
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
    const int warp = threadIdx.x >> 5;
    if (warp < 4) {   // scale bytes behind accumulator 0
        const unsigned addr = tmem + (static_cast<unsigned>(warp * 32) << 16) + 240;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr), "r"(0x7F7F7F7Fu));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    constexpr unsigned idesc = (1u << 7) | (1u << 10) | (1u << 23) | ((240u >> 3) << 17) | ((128u >> 4) << 24);
    if (threadIdx.x == 256) {
        const long long t0 = clock64();
        long long n = 0;
        if (mma_on) {
            const int total = ld_on ? (1 << 30) : iters * 8;
            for (int t = 0; t < total; ++t) {
                if (ld_on && *done >= 8) break;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint64_t da = umma_desc(smem_a + 32 * (k & 3)), db = umma_desc(smem_b + 32 * (k & 3));
                    const unsigned acc = k != 0;
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n" ::"r"(tmem),
                                 "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(tmem + 240), "r"(tmem + 244)
                                 : "memory");
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
                asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D;\nbra W;\nD:\n}\n" ::"r"(bar), "r"(t & 1) : "memory");
                ++n;
            }
        }
        const long long t1 = clock64();
        mma_cycles[2 * blockIdx.x] = t1 - t0;
        mma_cycles[2 * blockIdx.x + 1] = n;
    } else if (warp < 8 && ld_on) {
        const unsigned lane_addr = static_cast<unsigned>((warp & 3) * 32) << 16;
        unsigned acc = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                unsigned v[32];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),
                      "=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
                    : "r"(tmem + lane_addr + 256 + (warp >> 2) * 128 + c * 32));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                for (int i = 0; i < 32; ++i) acc ^= v[i];
            }
        }
        const long long t1 = clock64();
        if (acc == 0x12345) sink[0] = acc;
        if ((threadIdx.x & 31) == 0) {
            ld_cycles[blockIdx.x * 8 + warp] = t1 - t0;
            atomicAdd(const_cast<unsigned*>(done), 1u);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

int main() {
    unsigned long long *d_ld, *d_mma; unsigned* d_sink;
    CK(cudaMalloc(&d_ld, 8 * 148 * 8)); CK(cudaMalloc(&d_mma, 8 * 148 * 2)); CK(cudaMalloc(&d_sink, 4));
    const int smem = 16384 + 32768 + 2048, iters = 2000;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    printf("{\n");
    for (int mode = 0; mode < 3; ++mode) {   // 0: loads only, 1: loads + MMAs, 2: MMAs only
        const int mma_on = mode != 0, ld_on = mode != 2;
        CK(cudaMemset(d_ld, 0, 8 * 148 * 8)); CK(cudaMemset(d_mma, 0, 8 * 148 * 2));
        probe<<<148, 288, smem>>>(iters, mma_on, ld_on, d_ld, d_mma, d_sink);
        CK(cudaDeviceSynchronize());
        unsigned long long ld[8], mm[2];
        CK(cudaMemcpy(ld, d_ld, sizeof(ld), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(mm, d_mma, sizeof(mm), cudaMemcpyDeviceToHost));
        const char* names[] = {"loads_only", "loads_and_mma", "mma_only"};
        printf(" \"%s\": {\"clk_per_x32_load_per_warp\": %.1f, \"clk_per_240col_tile_of_8_mma\": %.1f},\n", names[mode],
               ld_on ? static_cast<double>(ld[0]) / (iters * 4) : 0.0, mm[1] ? static_cast<double>(mm[0]) / mm[1] : 0.0);
    }
    printf(" \"how\": \"tools/tmem_contention.cu: 8 warps of tcgen05.ld.32x32b.x32 + wait::ld on TMEM columns 256..511 against one thread issuing kind::mxf4 M128 N240 K64 MMAs into columns 0..239 (commit + wait per 8)\"}\n");
    return 0;
}
