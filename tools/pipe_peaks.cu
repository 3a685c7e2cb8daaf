// Pipe-rate microbenchmark for B200 (sm_100a): the roofline denominators the two CLATCH
// kernels are actually bound by (MEASURED_PEAKS.json only carries HBM and bf16 GEMM).
// Prints one JSON object: absolute G-ops/s (CUDA events) and ops/clk/SM (clock64).
//   popc        POPC.32                      (matcher: 16 per 512-bit compare)
//   lop3        LOP3.LUT                     (XOR / carry-save adders)
//   dadd/dmul   non-fused fp64 add / mul     (extraction: every op individually rounded)
//   dfma        fp64 FMA                     (for context only; never usable bit-exactly)
//   f2i / i2f   F2I.F64.FLOOR / I2F.F64      (floor + int->double in the resampler)
//   lds64       conflict-free 64-bit shared loads, GB/s and B/clk/SM
//   lds64_rand  64-bit shared loads at per-lane random 8-byte slots (bank-conflict model)
//   lds64_hw16  random, but distinct bank pairs inside each half-warp
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kThreads = 512;
constexpr int kIters = 4096;
constexpr int kUnroll = 8;

template <int OP>
__global__ void alu_kernel(unsigned long long* cycles, double* sink, unsigned seed) {
    unsigned long long n0, n1;
    unsigned a[kUnroll];
    double d[kUnroll];
    for (int i = 0; i < kUnroll; ++i) {
        a[i] = seed * (threadIdx.x + 1) + i * 2654435761u;
        d[i] = 1.0 + 1e-9 * (threadIdx.x + i);
    }
    const double m = 1.0 + 1e-12 * seed, c = 1e-13 * seed;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n0));
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kUnroll; ++i) {
            if (OP == 0) a[i] = __popc(a[i]) + seed;                 // POPC (+ IADD on another pipe)
            if (OP == 1) a[i] = (a[i] ^ seed) & (a[i] >> 1 | seed);  // LOP3-ish
            if (OP == 2) d[i] = __dadd_rn(d[i], c);
            if (OP == 3) d[i] = __dmul_rn(d[i], m);
            if (OP == 4) d[i] = __fma_rn(d[i], m, c);
            if (OP == 5) a[i] = __double2int_rd(d[i]) + a[i], d[i] = __dadd_rn(d[i], c);
            if (OP == 6) d[i] = __dadd_rn(static_cast<double>(static_cast<int>(a[i])), d[i]), a[i] += seed;
        }
    }
    const long long t1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n1));
    double s = 0;
    for (int i = 0; i < kUnroll; ++i) s += d[i] + a[i];
    if (s == 12345.678) sink[0] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0, cycles[gridDim.x + blockIdx.x] = n1 - n0;
}

// mode 0: lane-linear (conflict free); 1: random slots; 2: random with distinct bank pairs per half-warp
__global__ void lds_kernel(unsigned long long* cycles, double* sink, const unsigned short* offsets) {
    __shared__ double buf[4160];
    for (int i = threadIdx.x; i < 4160; i += blockDim.x) buf[i] = i;
    __syncthreads();
    unsigned off[kUnroll];
    for (int i = 0; i < kUnroll; ++i) off[i] = offsets[threadIdx.x * kUnroll + i];
    double acc[kUnroll] = {0};
    unsigned long long n0, n1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n0));
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kUnroll; ++i) {
            acc[i] += buf[off[i]];
            off[i] = (off[i] + 65) & 4095;   // +65 doubles: same bank-pair shift for every lane
        }
    }
    const long long t1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(n1));
    double s = 0;
    for (int i = 0; i < kUnroll; ++i) s += acc[i];
    if (s == 12345.678) sink[0] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0, cycles[gridDim.x + blockIdx.x] = n1 - n0;
}

struct Result { double gops; double per_clk_sm; double sm_mhz; };   // sm_mhz: clock64 ticks / globaltimer ns while the kernel ran, median over CTAs

template <typename Launch>
Result run(Launch launch, int blocks, int sms, unsigned long long* d_cycles, double ops_per_thread,
           int extra_dadd = 0) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<unsigned long long> cyc(2 * blocks);
    CK(cudaMemcpy(cyc.data(), d_cycles, sizeof(unsigned long long) * 2 * blocks, cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    std::vector<double> mhz(blocks);
    for (int b = 0; b < blocks; ++b) {
        mx = cyc[b] > mx ? cyc[b] : mx;
        mhz[b] = cyc[b] * 1e3 / static_cast<double>(cyc[blocks + b]);
    }
    std::sort(mhz.begin(), mhz.end());
    const double total = ops_per_thread * kThreads * blocks;
    Result r;
    r.gops = total / (ms * 1e-3) / 1e9;
    r.per_clk_sm = ops_per_thread * kThreads * (blocks / sms) / static_cast<double>(mx);
    r.sm_mhz = mhz[blocks / 2];
    return r;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    const int blocks = sms * 2;   // 2 x 512 threads per SM, all resident
    unsigned long long* d_cycles;
    double* d_sink;
    CK(cudaMalloc(&d_cycles, sizeof(unsigned long long) * 2 * blocks));
    CK(cudaMalloc(&d_sink, sizeof(double)));
    const double ops = static_cast<double>(kIters) * kUnroll;

    const char* names[] = {"popc", "lop3", "dadd", "dmul", "dfma", "f2i_floor_plus_dadd", "i2f_plus_dadd"};
    Result res[7];
    res[0] = run([&] { alu_kernel<0><<<blocks, kThreads>>>(d_cycles, d_sink, 3); }, blocks, sms, d_cycles, ops);
    res[1] = run([&] { alu_kernel<1><<<blocks, kThreads>>>(d_cycles, d_sink, 3); }, blocks, sms, d_cycles, ops);
    res[2] = run([&] { alu_kernel<2><<<blocks, kThreads>>>(d_cycles, d_sink, 3); }, blocks, sms, d_cycles, ops);
    res[3] = run([&] { alu_kernel<3><<<blocks, kThreads>>>(d_cycles, d_sink, 3); }, blocks, sms, d_cycles, ops);
    res[4] = run([&] { alu_kernel<4><<<blocks, kThreads>>>(d_cycles, d_sink, 3); }, blocks, sms, d_cycles, ops);
    res[5] = run([&] { alu_kernel<5><<<blocks, kThreads>>>(d_cycles, d_sink, 3); }, blocks, sms, d_cycles, ops);
    res[6] = run([&] { alu_kernel<6><<<blocks, kThreads>>>(d_cycles, d_sink, 3); }, blocks, sms, d_cycles, ops);

    // shared-memory patterns
    std::vector<unsigned short> off(kThreads * kUnroll);
    unsigned short* d_off;
    CK(cudaMalloc(&d_off, off.size() * sizeof(unsigned short)));
    Result lds[3];
    for (int mode = 0; mode < 3; ++mode) {
        srand(7);
        for (int t = 0; t < kThreads; ++t)
            for (int i = 0; i < kUnroll; ++i) {
                unsigned v;
                if (mode == 0) v = (t + 32 * i) & 4095;
                else if (mode == 1) v = rand() & 4095;
                else v = ((rand() & 255) << 4 | (t & 15)) & 4095;   // bank pair == lane % 16
                off[t * kUnroll + i] = static_cast<unsigned short>(v);
            }
        CK(cudaMemcpy(d_off, off.data(), off.size() * sizeof(unsigned short), cudaMemcpyHostToDevice));
        lds[mode] = run([&] { lds_kernel<<<blocks, kThreads>>>(d_cycles, d_sink, d_off); }, blocks, sms,
                        d_cycles, ops);
    }

    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    printf("{\"device\": \"%s\", \"sm_count\": %d, \"max_sm_mhz\": %.0f,\n", prop.name, sms, khz / 1e3);
    for (int i = 0; i < 7; ++i)
        printf(" \"%s_gops\": %.1f, \"%s_per_clk_sm\": %.2f, \"%s_sm_mhz\": %.0f,\n", names[i], res[i].gops, names[i],
               res[i].per_clk_sm, names[i], res[i].sm_mhz);
    const char* lnames[] = {"lds64", "lds64_rand", "lds64_hw16"};
    for (int i = 0; i < 3; ++i)
        printf(" \"%s_gbs\": %.1f, \"%s_bytes_per_clk_sm\": %.2f, \"%s_sm_mhz\": %.0f,\n", lnames[i], lds[i].gops * 8,
               lnames[i], lds[i].per_clk_sm * 8, lnames[i], lds[i].sm_mhz);
    printf(" \"popc_gops_roofline\": %.1f, \"fp64_nonfused_gops\": %.1f, \"how\": \"tools/pipe_peaks.cu: %d CTAs x %d threads, %d x %d independent ops per thread; G-ops/s from CUDA events, per-clk from clock64\"}\n",
           res[0].gops, (res[2].gops + res[3].gops) / 2, blocks, kThreads, kIters, kUnroll);
    return 0;
}
