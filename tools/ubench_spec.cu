// speculative multi-holder rounds vs the serial loop (N=8, 32-item chunks)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned lanemask_lt() { unsigned m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__global__ void __launch_bounds__(32, 1) k(int variant, int chunks, unsigned* out, long long* cyc) {
    __shared__ unsigned stg[32][32];
    __shared__ unsigned cm[32];
    const unsigned lane = threadIdx.x, N = 8, b = 512;
    unsigned seed = 12345;
    long long t0 = clock64();
    unsigned Msh = 0, sink = 0;
    for (int c = 0; c < chunks; ++c) {
        // synthetic chunk: 2-3 holders among 8 nodes, S small
        for (unsigned u = 0; u < 32; ++u) {
            unsigned h = (u * 2654435761u + c * 97u) ;
            unsigned m = (1u << (h & 7)) | (1u << ((h >> 3) & 7)) | (((h >> 6) & 3) == 0 ? (1u << ((h >> 8) & 7)) : 0u);
            if (lane == 0) cm[u] = m;
            stg[u][lane] = lane < N ? ((h >> (lane & 15)) & 63) : b;
        }
        __syncwarp();
        const unsigned Mstart = Msh >> 5;
        unsigned myres = 0xFFFFFFFFu;
        if (variant == 0) {  // serial, one item per REDUX
            for (unsigned u = 0; u < 32; ++u) {
                const unsigned mk = cm[u];
                const unsigned S = ((mk >> lane) & 1u) && lane < N ? stg[u][lane] : b;
                const unsigned thr = (b - S) << 5, kb = (S << 5) | lane;
                const unsigned keyv = Msh < thr ? kb + Msh : 0xFFFFFFFFu;
                const unsigned best = __reduce_min_sync(0xFFFFFFFFu, keyv);
                Msh += (keyv == best && best != 0xFFFFFFFFu) ? 32u : 0u;
                myres = lane == u ? best : myres;
            }
        } else {  // 4 groups of 8 lanes, one group-masked REDUX per round
            const unsigned g = lane >> 3, kk = lane & 7;
            const unsigned gmask = 0xFFu << (8 * g);
            unsigned mi = 0;
            while (mi < 32) {
                const unsigned W = min(4u, 32u - mi);
                const unsigned u = mi + g;
                const bool gv = g < W;
                const unsigned mk = gv ? cm[u] : 0u;
                const bool in = gv && kk < N && ((mk >> kk) & 1u);
                const unsigned S = in ? stg[u][kk] : b;
                const unsigned thr = (b - S) << 5, kb = (S << 5) | kk;
                const unsigned keyv = Msh < thr ? kb + Msh : 0xFFFFFFFFu;
                const unsigned r = __reduce_min_sync(gmask, keyv);
                const unsigned r0 = __shfl_sync(0xFFFFFFFFu, r, 0), r1 = __shfl_sync(0xFFFFFFFFu, r, 8);
                const unsigned r2 = __shfl_sync(0xFFFFFFFFu, r, 16), r3 = __shfl_sync(0xFFFFFFFFu, r, 24);
                const unsigned h1 = __shfl_sync(0xFFFFFFFFu, mk, 8), h2 = __shfl_sync(0xFFFFFFFFu, mk, 16);
                const unsigned h3 = __shfl_sync(0xFFFFFFFFu, mk, 24);
                auto bit = [](unsigned x) { return x == 0xFFFFFFFFu ? 0u : (1u << (x & 31)); };
                unsigned chosen = bit(r0), acc = 1;
                if (W > 1 && !(h1 & chosen)) { acc = 2; chosen |= bit(r1);
                    if (W > 2 && !(h2 & chosen)) { acc = 3; chosen |= bit(r2);
                        if (W > 3 && !(h3 & chosen)) { acc = 4; chosen |= bit(r3); } } }
                myres = lane == mi ? r0 : myres;
                if (acc > 1) myres = lane == mi + 1 ? r1 : myres;
                if (acc > 2) myres = lane == mi + 2 ? r2 : myres;
                if (acc > 3) myres = lane == mi + 3 ? r3 : myres;
                Msh += ((chosen >> kk) & 1u) << 5;
                mi += acc;
            }
        }
        sink += myres + Mstart;
        Msh &= 0x3FFF;
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[variant] = (t1 - t0); out[0] = sink; }
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 4); cudaMallocManaged(&c, 16);
    for (int v = 0; v < 2; ++v) { k<<<1, 32>>>(v, 100, o, c); cudaDeviceSynchronize(); }
    long long base[2];
    for (int v = 0; v < 2; ++v) { k<<<1, 32>>>(v, 2000, o, c); cudaDeviceSynchronize(); base[v] = c[v]; }
    printf("serial %.1f cyc/item, speculative %.1f cyc/item (incl. synthetic chunk setup)\n",
           base[0] / (2000.0 * 32), base[1] / (2000.0 * 32));
}
