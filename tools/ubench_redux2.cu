// does a 1024-thread CTA with 31 warps parked at __syncthreads slow warp 0's serial chain?
#include <cstdio>
#include <cstdint>
__global__ void k(int iters, unsigned* out, long long* cyc, int slot) {
    __shared__ unsigned arr[4096];
    __shared__ unsigned res[4096];
    unsigned lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) arr[i] = (i * 2654435761u) & 4095;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned M = 0;
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            unsigned j = arr[i & 4095];
            unsigned mk = arr[j];
            bool in = (mk >> lane) & 1;
            unsigned c = min(512u, (mk & 511) + M);
            unsigned key = (in && c < 512) ? ((c << 5) | lane) : 0xFFFFFFFFu;
            unsigned best = __reduce_min_sync(0xFFFFFFFFu, key);
            if (best != 0xFFFFFFFFu && lane == (best & 31)) { res[(lane * 128 + M) & 4095] = j; ++M; }
            if (lane == 0) res[j] = best;
        }
        long long t1 = clock64();
        if (lane == 0) { cyc[slot] = (t1 - t0) / iters; out[0] = M; }
    }
    __syncthreads();
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 4); cudaMallocManaged(&c, 4 * 8);
    k<<<1, 32>>>(1000, o, c, 0); cudaDeviceSynchronize();
    k<<<1, 32>>>(100000, o, c, 0);
    k<<<1, 1024>>>(100000, o, c, 1);
    k<<<1, 256>>>(100000, o, c, 2);
    cudaDeviceSynchronize();
    printf("cycles/iter: 32 threads %lld, 1024 threads %lld, 256 threads %lld\n", c[0], c[1], c[2]);
}
