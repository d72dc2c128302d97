// Does a large kernel body (>32 KB SASS) slow a hot loop in a single CTA?
#include <cstdio>
#include <cstdint>
template <int R>
__device__ __noinline__ unsigned bloat(unsigned x) {  // R unrolled rounds of mixing
    #pragma unroll
    for (int i = 0; i < R; ++i) x = (x ^ (x >> 7)) * 0x9E3779B9u + i;
    return x;
}
template <int R>
__global__ void __launch_bounds__(512, 1) k(int iters, int never, unsigned* out, long long* cyc) {
    __shared__ unsigned arr[4096];
    unsigned lane = threadIdx.x & 31;
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
            if (never == i) M += bloat<R>(M);   // never taken: only code size
        }
        if (lane == 0) out[0] = M;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
}
template <int R> void run(unsigned* o, long long* c) {
    k<R><<<1, 512>>>(200000, -1, o, c); cudaDeviceSynchronize();
    k<R><<<1, 512>>>(200000, -1, o, c); cudaDeviceSynchronize();
    printf("bloat %6d rounds: %lld cyc/iter\n", R, c[0]);
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 4); cudaMallocManaged(&c, 8);
    run<1>(o, c); run<1000>(o, c); run<3000>(o, c); run<6000>(o, c); run<12000>(o, c);
}
