// TMEM read-out rate probe (B200, sm_100a): how fast can the epilogue warps pull accumulators out of TMEM?
// 4 or 8 warps (one or two per SM sub-partition) loop over tcgen05.ld.32x32b of their lane quarter:
//   x32      32 columns -> 32 registers
//   x64      64 columns -> 64 registers
//   x32p16   64 columns of 16-bit data -> 32 registers (.pack::16b)
//   x16p16 / x64p16 likewise
// Prints bytes of TMEM cells covered per clk per SM and columns per clk per SM for each form.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int MODE>
__device__ __forceinline__ unsigned ld(unsigned taddr) {
    unsigned acc = 0;
    if (MODE == 0) {   // x32
        unsigned v[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),
              "=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 32; ++i) acc ^= v[i];
    } else if (MODE == 1) {   // x32 pack16: 64 columns
        unsigned v[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),
              "=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 32; ++i) acc ^= v[i];
    } else if (MODE == 2) {   // x16
        unsigned v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 16; ++i) acc ^= v[i];
    } else if (MODE == 3) {   // 16x256b.x8: 16 lanes x 256 bits x 8 = 32 registers, different lane mapping
        unsigned v[32];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]),"=r"(v[1]),"=r"(v[2]),"=r"(v[3]),"=r"(v[4]),"=r"(v[5]),"=r"(v[6]),"=r"(v[7]),"=r"(v[8]),"=r"(v[9]),"=r"(v[10]),"=r"(v[11]),"=r"(v[12]),"=r"(v[13]),"=r"(v[14]),"=r"(v[15]),
              "=r"(v[16]),"=r"(v[17]),"=r"(v[18]),"=r"(v[19]),"=r"(v[20]),"=r"(v[21]),"=r"(v[22]),"=r"(v[23]),"=r"(v[24]),"=r"(v[25]),"=r"(v[26]),"=r"(v[27]),"=r"(v[28]),"=r"(v[29]),"=r"(v[30]),"=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 32; ++i) acc ^= v[i];
    }
    return acc;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) probe(int iters, unsigned long long* cycles, unsigned* sink) {
    __shared__ unsigned slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&slot))));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = slot;
    const int warp = threadIdx.x >> 5;
    const unsigned lane_addr = static_cast<unsigned>((warp & 3) * 32) << 16;
    unsigned acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc ^= ld<MODE>(tmem + lane_addr + (warp >> 2) * 256 + c * 64);
    }
    __syncthreads();
    const long long t1 = clock64();
    if (acc == 0x12345) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int MODE>
void run(const char* name, int warps, int cols_per_ld, unsigned long long* d_cyc, unsigned* d_sink) {
    const int iters = 2000;
    probe<MODE><<<148, warps * 32>>>(iters, d_cyc, d_sink);
    CK(cudaDeviceSynchronize());
    probe<MODE><<<148, warps * 32>>>(iters, d_cyc, d_sink);
    CK(cudaDeviceSynchronize());
    unsigned long long cyc[148];
    CK(cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    for (auto c : cyc) mx = c > mx ? c : mx;
    const double lds = static_cast<double>(iters) * 4 * warps;
    printf(" \"%s_w%d\": {\"clk_per_ld_per_sm\": %.1f, \"columns_x_lanes_per_clk_sm\": %.1f},\n", name, warps, mx / lds,
           lds * cols_per_ld * 32 / mx);
}

int main() {
    unsigned long long* d_cyc; unsigned* d_sink;
    CK(cudaMalloc(&d_cyc, 8 * 148)); CK(cudaMalloc(&d_sink, 4));
    printf("{\n");
    run<0>("x32", 4, 32, d_cyc, d_sink); run<0>("x32", 8, 32, d_cyc, d_sink);
    run<1>("x64_pack16", 4, 64, d_cyc, d_sink); run<1>("x64_pack16", 8, 64, d_cyc, d_sink);
    run<2>("x16", 4, 16, d_cyc, d_sink); run<2>("x16", 8, 16, d_cyc, d_sink);
    run<3>("16x256b_x8", 4, 32, d_cyc, d_sink); run<3>("16x256b_x8", 8, 32, d_cyc, d_sink);
    printf(" \"how\": \"tools/tmem_ld_probe.cu: 148 CTAs, warps looping over tcgen05.ld + wait::ld; clk per load per SM and 32-bit TMEM cells covered per clk per SM\"}\n");
    return 0;
}
