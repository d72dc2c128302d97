// Does a lone CTA run slower than one CTA among many busy ones? (issue throttle test)
#include <cstdio>
#include <cstdint>
__device__ volatile int g_done;
__global__ void __launch_bounds__(512, 1) k(int iters, int spin_others, unsigned* out, long long* cyc) {
    __shared__ unsigned arr[4096];
    unsigned lane = threadIdx.x & 31;
    if (blockIdx.x != 0) {
        if (spin_others) { while (!g_done) __nanosleep(1000); }
        else if (spin_others == 0 && gridDim.x > 1) { /* same work as block 0 */ }
        if (spin_others) return;
    }
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) arr[i] = (i * 2654435761u) & 4095;
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x < 32) {
        unsigned M = 0;
        for (int i = 0; i < iters; ++i) {
            unsigned j = arr[i & 4095];
            unsigned mk = arr[j];
            bool in = (mk >> lane) & 1;
            unsigned c = min(512u, (mk & 511) + M);
            unsigned key = (in && c < 512) ? ((c << 5) | lane) : 0xFFFFFFFFu;
            unsigned best = __reduce_min_sync(0xFFFFFFFFu, key);
            if (best != 0xFFFFFFFFu && lane == (best & 31)) { arr[(lane * 128 + M) & 4095] = j; ++M; }
        }
        if (lane == 0) out[blockIdx.x] = M;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) { cyc[0] = (t1 - t0) / iters; g_done = 1; }
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 4 * 1024); cudaMallocManaged(&c, 8);
    int zero = 0;
    for (int rep = 0; rep < 2; ++rep) {
        for (int grid : {1, 8, 74, 148}) {
            for (int spin : {0, 1}) {
                cudaMemcpyToSymbol(g_done, &zero, 4);
                cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
                cudaEventRecord(a);
                k<<<grid, 512>>>(200000, spin, o, c);
                cudaEventRecord(b); cudaDeviceSynchronize();
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("grid %3d %s: %lld cyc/iter, %.3f ms\n", grid, spin ? "others spin" : "all work  ", c[0], ms);
            }
        }
    }
}
