// microbenchmark: latency of a dependent warp-min chain on sm_100a
#include <cstdio>
#include <cstdint>
__global__ void k(int mode, int iters, unsigned* out, long long* cyc) {
    unsigned lane = threadIdx.x & 31, x = lane * 7 + 3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned v = (x + lane * 13) & 1023;
        unsigned m;
        if (mode == 0) m = __reduce_min_sync(0xFFFFFFFFu, v);
        else if (mode == 1) {
            m = v;
            for (int s = 16; s; s >>= 1) m = min(m, __shfl_xor_sync(0xFFFFFFFFu, m, s));
        } else {
            __shared__ unsigned sm;
            if (lane == 0) sm = 0xFFFFFFFFu;
            __syncwarp();
            atomicMin(&sm, v);
            __syncwarp();
            m = sm;
            __syncwarp();
        }
        x += m;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = x; cyc[mode] = (t1 - t0) / iters; }
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 4); cudaMallocManaged(&c, 3 * 8);
    for (int m = 0; m < 3; ++m) { k<<<1, 32>>>(m, 10000, o, c); cudaDeviceSynchronize(); }
    for (int m = 0; m < 3; ++m) k<<<1, 32>>>(m, 100000, o, c);
    cudaDeviceSynchronize();
    printf("cycles/iter: redux %lld  shfl-butterfly %lld  smem-atomic %lld\n", c[0], c[1], c[2]);
}
