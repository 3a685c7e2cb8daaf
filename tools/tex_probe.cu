// Texture-gather microbenchmark for B200 (sm_100a): can tex2Dgather replace the shared-memory
// u8 tile as the source of the 2x2 bilinear footprints in the window resampler?
//   1. component order of tex2Dgather<uchar4> at (x0 + 1, y0 + 1) vs direct reads
//   2. gathers/clk/SM along rotated 64-sample lines (the resampler's access pattern), with the
//      L1/texture cache squeezed by a large dynamic shared-memory carve-out, for 8/16/32 warps
//      per SM, with and without the resampler's fp64 arithmetic on the results
// Prints one JSON object.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void order_kernel(cudaTextureObject_t tex, const int* xy, int n, uchar4* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = tex2Dgather<uchar4>(tex, xy[2 * i] + 1.0f, xy[2 * i + 1] + 1.0f, 0);
}

// The packed-plane resampler reads the same array through a normalised-float texture object: texel / 255 as a float.
__global__ void norm_kernel(cudaTextureObject_t texn, const int* xy, int n, float4* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = tex2Dgather<float4>(texn, xy[2 * i] + 1.0f, xy[2 * i + 1] + 1.0f, 0);
}

__device__ __forceinline__ double u8_to_f64(unsigned v) {
    return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(v)), 4503599627370496.0);
}

// One CTA per SM, persistent over keypoints; thread -> column u = tid & 63, rows tid>>6 + k*(T/64).
template <int kMode>   // 0: integer checksum only, 1: + the resampler's fp64 blend
__global__ void gather_kernel(cudaTextureObject_t tex, const double* xycs, int n, unsigned long long* cycles,
                              double* sink) {
    extern __shared__ unsigned char carve[];
    if (threadIdx.x == 0) carve[0] = 1;
    const int tid = threadIdx.x, u = tid & 63, rows_step = blockDim.x / 64;
    const double du = u - 31.5;
    double acc = 0.0;
    unsigned iacc = 0;
    const long long t0 = clock64();
    for (int kp = blockIdx.x; kp < n; kp += gridDim.x) {
        const double x = xycs[4 * kp], y = xycs[4 * kp + 1], c = xycs[4 * kp + 2], s = xycs[4 * kp + 3];
        const double xa = __dadd_rn(x, __dmul_rn(c, du)), ya = __dadd_rn(y, __dmul_rn(s, du));
#pragma unroll 8
        for (int v = tid >> 6; v < 64; v += rows_step) {
            const double dv = v - 31.5;
            const double sx = __dsub_rn(xa, __dmul_rn(s, dv)), sy = __dadd_rn(ya, __dmul_rn(c, dv));
            const double kMagic = 6755399441055744.0;
            const double tx = __dadd_rd(sx, kMagic), ty = __dadd_rd(sy, kMagic);
            const int x0 = __double2loint(tx), y0 = __double2loint(ty);
            const uchar4 g = tex2Dgather<uchar4>(tex, x0 + 1.0f, y0 + 1.0f, 0);
            if (kMode == 0) {
                iacc += g.x + 3 * g.y + 5 * g.z + 7 * g.w;
            } else {
                const double fx = __dsub_rn(sx, __dsub_rn(tx, kMagic)), fy = __dsub_rn(sy, __dsub_rn(ty, kMagic));
                const double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy);
                const double top = __dadd_rn(__dmul_rn(gx, u8_to_f64(g.w)), __dmul_rn(fx, u8_to_f64(g.z)));
                const double bot = __dadd_rn(__dmul_rn(gx, u8_to_f64(g.x)), __dmul_rn(fx, u8_to_f64(g.y)));
                acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(gy, top), __dmul_rn(fy, bot)));
            }
        }
    }
    const long long t1 = clock64();
    if (acc + iacc == 12345.678) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// Fill a u8 CUDA array from pitch-linear device memory through a surface: 16 pixels per thread.
__global__ void fill_array_kernel(cudaSurfaceObject_t surf, const unsigned char* src, size_t pitch, int w, int h) {
    const int x = (blockIdx.x * blockDim.x + threadIdx.x) * 16, y = blockIdx.y;
    if (x >= w || y >= h) return;
    if (x + 16 <= w) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + y * pitch + x);
        surf2Dwrite(v, surf, x, y);
    } else {
        for (int i = x; i < w; ++i) surf2Dwrite(src[y * pitch + i], surf, i, y);
    }
}

static void time_array_fill(int W, int H) {
    unsigned char* d_lin;
    const size_t pitch = (W + 15) / 16 * 16;
    CK(cudaMalloc(&d_lin, pitch * H));
    CK(cudaMemset(d_lin, 7, pitch * H));
    cudaChannelFormatDesc fmt = cudaCreateChannelDesc<unsigned char>();
    cudaArray_t arr;
    CK(cudaMallocArray(&arr, &fmt, W, H, cudaArrayTextureGather | cudaArraySurfaceLoadStore));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = arr;
    cudaSurfaceObject_t surf;
    CK(cudaCreateSurfaceObject(&surf, &rd));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    float ms_copy = 0, ms_kernel = 0;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        for (int i = 0; i < 10; ++i) CK(cudaMemcpy2DToArrayAsync(arr, 0, 0, d_lin, pitch, W, H, cudaMemcpyDeviceToDevice, 0));
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms_copy, e0, e1));
        CK(cudaEventRecord(e0));
        for (int i = 0; i < 10; ++i)
            fill_array_kernel<<<dim3((W / 16 + 127) / 128, H), 128>>>(surf, d_lin, pitch, W, H);
        CK(cudaEventRecord(e1));
        CK(cudaDeviceSynchronize());
        CK(cudaEventElapsedTime(&ms_kernel, e0, e1));
    }
    printf(" \"array_fill_%dx%d\": {\"cudaMemcpy2DToArrayAsync_d2d_us\": %.1f, \"surf2Dwrite_kernel_us\": %.1f},\n", W, H,
           ms_copy * 100, ms_kernel * 100);
    CK(cudaDestroySurfaceObject(surf));
    CK(cudaFreeArray(arr));
    CK(cudaFree(d_lin));
}

int main() {
    const int W = 1920, H = 1080, N = 20000;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int sms = prop.multiProcessorCount;
    std::vector<unsigned char> img(static_cast<size_t>(W) * H);
    unsigned rng = 12345;
    for (auto& p : img) { rng = rng * 1664525u + 1013904223u; p = rng >> 24; }
    cudaChannelFormatDesc fmt = cudaCreateChannelDesc<unsigned char>();
    cudaArray_t arr;
    CK(cudaMallocArray(&arr, &fmt, W, H, cudaArrayTextureGather));
    CK(cudaMemcpy2DToArray(arr, 0, 0, img.data(), W, W, H, cudaMemcpyHostToDevice));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = arr;
    cudaTextureDesc td{};
    td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint;
    td.readMode = cudaReadModeElementType;
    td.normalizedCoords = 0;
    cudaTextureObject_t tex;
    CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));

    // 1. order
    const int n_chk = 4096;
    std::vector<int> xy(2 * n_chk);
    for (int i = 0; i < n_chk; ++i) {
        rng = rng * 1664525u + 1013904223u; xy[2 * i] = (rng >> 8) % (W - 1);
        rng = rng * 1664525u + 1013904223u; xy[2 * i + 1] = (rng >> 8) % (H - 1);
    }
    int* d_xy; uchar4* d_out;
    CK(cudaMalloc(&d_xy, sizeof(int) * 2 * n_chk));
    CK(cudaMalloc(&d_out, sizeof(uchar4) * n_chk));
    CK(cudaMemcpy(d_xy, xy.data(), sizeof(int) * 2 * n_chk, cudaMemcpyHostToDevice));
    order_kernel<<<(n_chk + 255) / 256, 256>>>(tex, d_xy, n_chk, d_out);
    std::vector<uchar4> out(n_chk);
    CK(cudaMemcpy(out.data(), d_out, sizeof(uchar4) * n_chk, cudaMemcpyDeviceToHost));
    int ok_order = 0;
    for (int i = 0; i < n_chk; ++i) {
        const int x0 = xy[2 * i], y0 = xy[2 * i + 1];
        const unsigned char p00 = img[y0 * W + x0], p10 = img[y0 * W + x0 + 1], p01 = img[(y0 + 1) * W + x0],
                            p11 = img[(y0 + 1) * W + x0 + 1];
        ok_order += out[i].w == p00 && out[i].z == p10 && out[i].x == p01 && out[i].y == p11;
    }

    // 2. throughput
    std::vector<double> xycs(4 * N);
    for (int i = 0; i < N; ++i) {
        rng = rng * 1664525u + 1013904223u; const double ux = (rng >> 8) / 16777216.0;
        rng = rng * 1664525u + 1013904223u; const double uy = (rng >> 8) / 16777216.0;
        rng = rng * 1664525u + 1013904223u; const double th = -M_PI + (rng >> 8) / 16777216.0 * 2 * M_PI;
        xycs[4 * i] = 46 + ux * (W - 93); xycs[4 * i + 1] = 46 + uy * (H - 93);
        xycs[4 * i + 2] = cos(th); xycs[4 * i + 3] = sin(th);
    }
    double* d_xycs; unsigned long long* d_cyc; double* d_sink;
    CK(cudaMalloc(&d_xycs, sizeof(double) * 4 * N));
    CK(cudaMalloc(&d_cyc, sizeof(unsigned long long) * sms));
    CK(cudaMalloc(&d_sink, sizeof(double)));
    CK(cudaMemcpy(d_xycs, xycs.data(), sizeof(double) * 4 * N, cudaMemcpyHostToDevice));
    const int carve = 200 * 1024;
    CK(cudaFuncSetAttribute(gather_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, carve));
    CK(cudaFuncSetAttribute(gather_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, carve));
    // 1b. the normalised-float view of the same array: is every component float(texel) / 255.0f, correctly rounded?
    td.readMode = cudaReadModeNormalizedFloat;
    cudaTextureObject_t texn;
    CK(cudaCreateTextureObject(&texn, &rd, &td, nullptr));
    float4* d_outf;
    CK(cudaMalloc(&d_outf, sizeof(float4) * n_chk));
    norm_kernel<<<(n_chk + 255) / 256, 256>>>(texn, d_xy, n_chk, d_outf);
    std::vector<float4> outf(n_chk);
    CK(cudaMemcpy(outf.data(), d_outf, sizeof(float4) * n_chk, cudaMemcpyDeviceToHost));
    int norm_exact = 0, levels_seen[256] = {0}, n_levels = 0;
    double norm_max_rel = 0.0;
    for (int i = 0; i < n_chk; ++i) {
        const int x0 = xy[2 * i], y0 = xy[2 * i + 1];
        const unsigned char p[4] = {img[(y0 + 1) * W + x0], img[(y0 + 1) * W + x0 + 1], img[y0 * W + x0 + 1], img[y0 * W + x0]};   // x, y, z, w
        const float got[4] = {outf[i].x, outf[i].y, outf[i].z, outf[i].w};
        bool all = true;
        for (int k = 0; k < 4; ++k) {
            const float want = static_cast<float>(p[k]) / 255.0f;
            all = all && got[k] == want;
            if (p[k]) norm_max_rel = std::max(norm_max_rel, std::fabs(static_cast<double>(got[k]) - p[k] / 255.0) / (p[k] / 255.0));
            if (!levels_seen[p[k]]++) ++n_levels;
        }
        norm_exact += all;
    }
    printf("{\"device\": \"%s\", \"sm_count\": %d, \"gather_order_w_z_x_y_is_p00_p10_p01_p11\": %s, \"checked\": %d,\n",
           prop.name, sms, ok_order == n_chk ? "true" : "false", n_chk);
    printf(" \"normalized_float_gather\": {\"footprints_equal_to_float_texel_over_255\": %d, \"of\": %d, \"grey_levels_seen\": %d, "
           "\"max_relative_error_vs_exact_quotient\": %.3g, \"two_pow_minus_24\": %.3g},\n",
           norm_exact, n_chk, n_levels, norm_max_rel, 5.96e-8);
    time_array_fill(1920, 1080);
    time_array_fill(3840, 2160);
    printf(" \"carveout_kb\": %d, \"runs\": [\n", carve / 1024);
    bool first = true;
    for (int mode = 0; mode < 2; ++mode)
        for (int threads : {256, 512, 1024}) {
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaEventRecord(e0));
                if (mode == 0) gather_kernel<0><<<sms, threads, carve>>>(tex, d_xycs, N, d_cyc, d_sink);
                else gather_kernel<1><<<sms, threads, carve>>>(tex, d_xycs, N, d_cyc, d_sink);
                CK(cudaEventRecord(e1));
                CK(cudaDeviceSynchronize());
            }
            float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
            std::vector<unsigned long long> cyc(sms);
            CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
            double mean = 0; for (auto c : cyc) mean += c; mean /= sms;
            const double per_sm = static_cast<double>(N) * 4096 / sms;
            printf("%s  {\"mode\": \"%s\", \"warps_per_sm\": %d, \"ms\": %.4f, \"windows_per_s\": %.4g, "
                   "\"gathers_per_clk_sm\": %.3f, \"clk_per_window\": %.1f}",
                   first ? "" : ",\n", mode == 0 ? "gather+checksum" : "gather+fp64 blend", threads / 32, ms,
                   N / (ms * 1e-3), per_sm / mean, mean / (static_cast<double>(N) / sms));
            first = false;
        }
    printf("\n ]}\n");
    return 0;
}
