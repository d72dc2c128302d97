// replicate the planner's phase-D loop and toggle features to find the slowdown
#include <cstdio>
#include <cstdint>
struct Sm { unsigned stg[2][32][32]; };
__global__ void __launch_bounds__(1024, 1) k(int variant, int nm, const unsigned* smul, unsigned* out, long long* cyc) {
    extern __shared__ unsigned dyn[];
    __shared__ Sm sm;
    unsigned* pre = dyn;            // multi list
    unsigned* smask = dyn + 8192;
    unsigned* fin = dyn + 16384;
    unsigned* sinfo = dyn + 24576;
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5, N = 8, b = 512;
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) {
        pre[i] = (i * 2654435761u) & 4095;
        smask[i] = (1u << (i & 7)) | (1u << ((i >> 3) & 7));
    }
    __syncthreads();
    long long t0 = clock64();
    if (w == 0) {
        unsigned M = 0;
        auto stage = [&](unsigned base, unsigned buf) {
            unsigned cnt = min(32u, nm - base);
            if (lane < N)
                for (unsigned u = 0; u < cnt; ++u) {
                    unsigned ju = pre[base + u];
                    unsigned dst = (unsigned)__cvta_generic_to_shared(&sm.stg[buf][u][lane]);
                    if (variant & 1)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(&smul[ju * N + lane]));
                    else
                        sm.stg[buf][u][lane] = 7;
                }
            if (variant & 1) asm volatile("cp.async.commit_group;\n" ::);
        };
        if (nm) stage(0, 0);
        for (unsigned base = 0, buf = 0; base < nm; base += 32, buf ^= 1) {
            if (base + 32 < nm) { stage(base + 32, buf ^ 1); if (variant & 1) asm volatile("cp.async.wait_group 1;\n" ::); }
            else if (variant & 1) asm volatile("cp.async.wait_group 0;\n" ::);
            __syncwarp();
            unsigned cnt = min(32u, nm - base);
            for (unsigned u = 0; u < cnt; ++u) {
                unsigned j = pre[base + u];
                unsigned mk = smask[j];
                unsigned sk = sm.stg[buf][u][lane] & 255;
                bool in = lane < N && ((mk >> lane) & 1u);
                unsigned c2 = min(b, sk + M);
                unsigned keyv = (in && c2 < b) ? ((c2 << 5) | lane) : 0xFFFFFFFFu;
                unsigned best = __reduce_min_sync(0xFFFFFFFFu, keyv);
                if (best != 0xFFFFFFFFu && lane == (best & 31)) { fin[(lane * b + M) & 8191] = j; ++M; }
                if (lane == 0) sinfo[j] = best;
            }
            __syncwarp();
        }
        if (lane == 0) out[0] = M;
    }
    if (variant & 2) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[variant] = (t1 - t0) / nm;
}
int main() {
    unsigned *smul, *o; long long* c;
    cudaMalloc(&smul, 4096 * 8 * 4); cudaMemset(smul, 1, 4096 * 32); cudaMalloc(&o, 4); cudaMallocManaged(&c, 8 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    for (int v = 0; v < 4; ++v) for (int th : {32, 1024}) {
        k<<<1, th, 160 * 1024>>>(v, 800, smul, o, c); cudaDeviceSynchronize();
        k<<<1, th, 160 * 1024>>>(v, 800, smul, o, c); cudaDeviceSynchronize();
        printf("variant cpasync=%d bar=%d threads=%d: %lld cyc/item\n", v & 1, (v >> 1) & 1, th, c[v]);
    }
}
