// fp64 pipe latency / issue probe for B200: dependent DADD chains at several ILP x warps/SM.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
constexpr int kIters = 2048;
template <int ILP, int OP>
__global__ void chain(unsigned long long* cycles, double* sink, double c) {
    double d[ILP];
    for (int i = 0; i < ILP; ++i) d[i] = 1.0 + 1e-9 * (threadIdx.x + i);
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if (OP == 0) d[i] = __dadd_rn(d[i], c);
            if (OP == 1) d[i] = __dmul_rn(d[i], c);
            if (OP == 2) d[i] = __dadd_rd(d[i], c);
            if (OP == 3) d[i] = static_cast<double>(__double2float_rz(d[i])) + c;   // F2F both ways + DADD
        }
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < ILP; ++i) s += d[i];
    if (s == 12345.678) sink[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}
template <int ILP, int OP>
void run(const char* name, int warps, unsigned long long* d_c, double* d_s, bool& first) {
    chain<ILP, OP><<<1, warps * 32>>>(d_c, d_s, 1e-13);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, d_c, sizeof(c), cudaMemcpyDeviceToHost));
    printf("%s  {\"op\": \"%s\", \"ilp\": %d, \"warps_on_sm\": %d, \"clk_per_dependent_step\": %.2f, \"warp_ops_per_clk_sm\": %.3f}",
           first ? "" : ",\n", name, ILP, warps, static_cast<double>(c) / kIters, static_cast<double>(ILP) * warps * kIters / c);
    first = false;
}
// Issue-port probe: MIX = 0: DADD only, 1: DADD + IADD3 1:1, 2: FFMA2 only, 3: FFMA2 + IADD3 1:1, 4: IADD3 only,
// 5: DADD + FFMA2 1:1 — eight independent chains of each kind per thread, 16 warps per SM sub-partition.
template <int MIX>
__global__ void issue_mix(unsigned long long* cycles, double* sink, double c, unsigned k) {
    double d[8];
    float2 f[8];
    unsigned a[8];
    for (int i = 0; i < 8; ++i) {
        d[i] = 1.0 + 1e-9 * (threadIdx.x + i);
        f[i] = make_float2(1.0f + i, 2.0f + threadIdx.x);
        a[i] = threadIdx.x * 7 + i;
    }
    const float2 m = make_float2(1.0000001f, 0.9999999f), z = make_float2(1e-9f, 2e-9f);
    const long long t0 = clock64();
    for (int it = 0; it < 1024; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MIX == 0 || MIX == 1 || MIX == 5) d[i] = __dadd_rn(d[i], c);
            if (MIX == 2 || MIX == 3 || MIX == 5) f[i] = __ffma2_rn(f[i], m, z);
            if (MIX == 1 || MIX == 3 || MIX == 4) a[i] = a[i] * 3 + k;   // IMAD
        }
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += d[i] + f[i].x + f[i].y + a[i];
    if (s == 12345.678) sink[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}
template <int MIX>
void run_mix(const char* name, int per_iter, unsigned long long* d_c, double* d_s, bool& first) {
    issue_mix<MIX><<<1, 1024>>>(d_c, d_s, 1e-13, 5u);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, d_c, sizeof(c), cudaMemcpyDeviceToHost));
    // 32 warps on one SM = 8 per sub-partition; instructions per clk per sub-partition
    printf("%s  {\"mix\": \"%s\", \"warp_instr_per_clk_per_subpartition\": %.3f}", first ? "" : ",\n", name,
           8.0 * 1024 * 8 * per_iter / c);
    first = false;
}

int main() {
    unsigned long long* d_c; double* d_s;
    CK(cudaMalloc(&d_c, 8)); CK(cudaMalloc(&d_s, 8));
    bool first = true;
    printf("{\"runs\": [\n");
    for (int warps : {1, 4, 8, 16, 32}) {
        run<1, 0>("dadd", warps, d_c, d_s, first);
        run<2, 0>("dadd", warps, d_c, d_s, first);
        run<4, 0>("dadd", warps, d_c, d_s, first);
        run<8, 0>("dadd", warps, d_c, d_s, first);
    }
    run<1, 1>("dmul", 1, d_c, d_s, first);
    run<1, 2>("dadd.rd", 1, d_c, d_s, first);
    run<1, 3>("f2f.rz+f2f+dadd", 1, d_c, d_s, first);
    run_mix<0>("dadd", 1, d_c, d_s, first);
    run_mix<1>("dadd+imad", 2, d_c, d_s, first);
    run_mix<2>("ffma2", 1, d_c, d_s, first);
    run_mix<3>("ffma2+imad", 2, d_c, d_s, first);
    run_mix<4>("imad", 1, d_c, d_s, first);
    run_mix<5>("dadd+ffma2", 2, d_c, d_s, first);
    printf("\n]}\n");
    return 0;
}
