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
    printf("\n]}\n");
    return 0;
}
