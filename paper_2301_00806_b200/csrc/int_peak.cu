// int_peak.cu -- measured INT32 issue peak: the roofline denominator of the
// integer-bound search (MEASURED_PEAKS.json carries only HBM and bf16).
// Eight independent LOP3/IADD3 chains per thread, full occupancy, CUDA events.
#include <cstdint>

#include "wpm_internal.h"

namespace wpm {

__global__ void __launch_bounds__(512) int_peak_kernel(uint32_t* out, uint32_t k1, uint32_t k2, int iters) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 2654435761u + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(k1), "r"(k2));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(k2));
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x ^= a[i];
    if (x == 0x12345678u) out[0] = x;
}

int int_peak_measure(int device, double* ops_per_s) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, int_peak_kernel, 512, 0) != cudaSuccess) return 1;
    const int grid = per_sm * prop.multiProcessorCount;
    uint32_t* out = nullptr;
    if (cudaMalloc(&out, 4) != cudaSuccess) return 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 1 << 14;
    int_peak_kernel<<<grid, 512>>>(out, 0x9E3779B9u, 0x7F4A7C15u, 256);  // warm up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        int_peak_kernel<<<grid, 512>>>(out, 0x9E3779B9u, 0x7F4A7C15u, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const bool ok = cudaGetLastError() == cudaSuccess;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (!ok) return 1;
    const double ops = (double)grid * 512.0 * (double)iters * 16.0;
    *ops_per_s = ops / (best * 1e-3);
    return 0;
}

}  // namespace wpm
