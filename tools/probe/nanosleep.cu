// dev probe: how long does __nanosleep(t) actually sleep on this GPU?
#include <cstdio>
__global__ void k(unsigned t, int iters, unsigned long long* out) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __nanosleep(t);
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) atomicAdd(out, t1 - t0);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    for (unsigned t : {32u, 256u, 1024u, 8192u, 65536u, 1000000u}) {
        for (int warps : {1, 40 * 148}) {
            cudaMemset(d, 0, 8);
            const int iters = 100;
            k<<<warps, 32>>>(t, iters, d);
            unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("nanosleep(%u ns) x%d, %d warps: %.1f ns per call (at 1.965 GHz)\n", t, iters, warps, (double)h / warps / iters / 1.965);
        }
    }
}
