// the planner's current phase-D inner loop, isolated
#include <cstdio>
#include <cstdint>
struct Sm { unsigned pthr[32][32]; unsigned pkb[32][32]; };
__global__ void __launch_bounds__(512, 1) k(int variant, int chunks, unsigned* out, long long* cyc) {
    extern __shared__ unsigned dyn[];
    __shared__ Sm sm;
    unsigned* fin = dyn; unsigned* sinfo = dyn + 8192;
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5, N = 8, b = 512;
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
        unsigned u = i / 32, l = i % 32;
        unsigned S = (u * 7 + l * 13) % 40;
        bool in = l < N && ((u + l) % 3 == 0);
        sm.pthr[u][l] = in ? (b - S) << 5 : 0;
        sm.pkb[u][l] = (S << 5) | l;
    }
    __syncthreads();
    long long t0 = clock64();
    if (w == 0) {
        unsigned Msh = 0;
        const unsigned myj = lane * 97 % 4096;
        for (int c = 0; c < chunks; ++c) {
            unsigned thrn = sm.pthr[0][lane], kbn = sm.pkb[0][lane];
            for (unsigned u = 0; u < 32; ++u) {
                const unsigned thr = thrn, kb = kbn;
                const unsigned j = __shfl_sync(0xFFFFFFFFu, myj, u);
                if (u + 1 < 32) { thrn = sm.pthr[u + 1][lane]; kbn = sm.pkb[u + 1][lane]; }
                const unsigned keyv = (Msh & 0xFFF) < thr ? kb + (Msh & 0xFFF) : 0xFFFFFFFFu;
                const unsigned best = __reduce_min_sync(0xFFFFFFFFu, keyv);
                if (variant & 1) {
                    if (keyv == best && best != 0xFFFFFFFFu) { fin[(lane * b + ((Msh >> 5) & 511)) & 8191] = j; Msh += 32; }
                    if (lane == 0) sinfo[j] = best;
                } else {
                    if (keyv == best && best != 0xFFFFFFFFu) Msh += 32;
                }
            }
            __syncwarp();
        }
        if (lane == 0) out[0] = Msh;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[variant] = (t1 - t0) / (chunks * 32);
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 4); cudaMallocManaged(&c, 4 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int v = 0; v < 2; ++v) {
        k<<<1, 512, 100 * 1024>>>(v, 100, o, c); cudaDeviceSynchronize();
        k<<<1, 512, 100 * 1024>>>(v, 20000, o, c); cudaDeviceSynchronize();
        printf("variant stores=%d: %lld cyc/item\n", v, c[v]);
    }
}
