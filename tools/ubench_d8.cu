// D8 serial-decision loop variants (N <= 8, keys in registers), one warp.
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(32, 1) k(int variant, int chunks, unsigned* out, long long* cyc) {
    __shared__ __align__(16) unsigned rows[2][32][8];   // 32-bit keys (S<<4)|k
    __shared__ __align__(16) unsigned prow[2][32][4];   // 16x2 packed keys
    const unsigned lane = threadIdx.x, b = 512;
    for (int buf = 0; buf < 2; ++buf)
        for (unsigned u = 0; u < 32; ++u) {
            unsigned h = (u * 2654435761u + buf * 97u);
            if (lane < 8) {
                const bool hold = ((h >> lane) & 3u) == 0 || (h & 7u) == lane;
                const unsigned S = hold ? ((h >> (lane + 8)) & 63u) : b;
                rows[buf][u][lane] = (S << 4) | lane;
            }
        }
    __syncwarp();
    if (lane < 32) for (int buf = 0; buf < 2; ++buf) {
        const unsigned u = lane;
        for (int p = 0; p < 4; ++p) prow[buf][u][p] = rows[buf][u][2 * p] | (rows[buf][u][2 * p + 1] << 16);
    }
    __syncwarp();
    const unsigned kSent = (b << 4) - 1u;
    unsigned sink = 0;
    long long t0 = clock64();
    if (variant == 0) {
        unsigned Mk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c = 0; c < chunks; ++c) {
            const uint4* r = reinterpret_cast<const uint4*>(&rows[c & 1][0][0]);
            unsigned myres = kSent;
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint4 r0 = r[2 * u], r1 = r[2 * u + 1];
                const unsigned K0 = r0.x + Mk[0], K1 = r0.y + Mk[1], K2 = r0.z + Mk[2], K3 = r0.w + Mk[3];
                const unsigned K4 = r1.x + Mk[4], K5 = r1.y + Mk[5], K6 = r1.z + Mk[6], K7 = r1.w + Mk[7];
                const unsigned cl = __vimin3_u32(__vimin3_u32(K0, K1, K2), __vimin3_u32(K3, K4, K5), __vimin3_u32(K6, K7, kSent));
                Mk[0] += cl == K0 ? 16u : 0u; Mk[1] += cl == K1 ? 16u : 0u;
                Mk[2] += cl == K2 ? 16u : 0u; Mk[3] += cl == K3 ? 16u : 0u;
                Mk[4] += cl == K4 ? 16u : 0u; Mk[5] += cl == K5 ? 16u : 0u;
                Mk[6] += cl == K6 ? 16u : 0u; Mk[7] += cl == K7 ? 16u : 0u;
                myres = lane == unsigned(u) ? cl : myres;
            }
            sink += myres;
            if ((c & 15) == 15) { for (int q = 0; q < 8; ++q) Mk[q] = 0; }
        }
        for (int q = 0; q < 8; ++q) sink += Mk[q];
    } else if (variant == 1) {
        unsigned Mk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c = 0; c < chunks; ++c) {
            const uint4* r = reinterpret_cast<const uint4*>(&rows[c & 1][0][0]);
            unsigned myres = kSent;
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint4 r0 = r[2 * u], r1 = r[2 * u + 1];
                const unsigned K0 = r0.x + Mk[0], K1 = r0.y + Mk[1], K2 = r0.z + Mk[2], K3 = r0.w + Mk[3];
                const unsigned K4 = r1.x + Mk[4], K5 = r1.y + Mk[5], K6 = r1.z + Mk[6], K7 = r1.w + Mk[7];
                const unsigned cl = __vimin3_u32(__vimin3_u32(K0, K1, K2), __vimin3_u32(K3, K4, K5), __vimin3_u32(K6, K7, kSent));
                const unsigned w = cl & 15u;
                Mk[0] += w == 0 ? 16u : 0u; Mk[1] += w == 1 ? 16u : 0u;
                Mk[2] += w == 2 ? 16u : 0u; Mk[3] += w == 3 ? 16u : 0u;
                Mk[4] += w == 4 ? 16u : 0u; Mk[5] += w == 5 ? 16u : 0u;
                Mk[6] += w == 6 ? 16u : 0u; Mk[7] += w == 7 ? 16u : 0u;
                myres = lane == unsigned(u) ? cl : myres;
            }
            sink += myres;
            if ((c & 15) == 15) { for (int q = 0; q < 8; ++q) Mk[q] = 0; }
        }
        for (int q = 0; q < 8; ++q) sink += Mk[q];
    } else {
        // 16x2 packed: pair p holds nodes 2p (lo) and 2p+1 (hi)
        unsigned M[4] = {0, 0, 0, 0};
        for (int c = 0; c < chunks; ++c) {
            const uint4* r = reinterpret_cast<const uint4*>(&prow[c & 1][0][0]);
            unsigned myres = kSent;
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const uint4 t = r[u];
                const unsigned K0 = t.x + M[0], K1 = t.y + M[1], K2 = t.z + M[2], K3 = t.w + M[3];
                const unsigned m = __vminu2(__vminu2(K0, K1), __vminu2(K2, K3));
                const unsigned cl = __vimin3_u32(m & 0xFFFFu, m >> 16, kSent);
                const unsigned w = cl & 15u;
                const unsigned dl = 16u << ((w & 1u) << 4);
                const unsigned wp = w >> 1;
                M[0] += wp == 0 ? dl : 0u; M[1] += wp == 1 ? dl : 0u;
                M[2] += wp == 2 ? dl : 0u; M[3] += wp == 3 ? dl : 0u;
                myres = lane == unsigned(u) ? cl : myres;
            }
            sink += myres;
            if ((c & 15) == 15) { for (int q = 0; q < 4; ++q) M[q] = 0; }
        }
        for (int q = 0; q < 4; ++q) sink += M[q];
    }
    long long t1 = clock64();
    out[lane] = sink;
    if (lane == 0) *cyc = t1 - t0;
}
int main() {
    unsigned* o; long long* c; cudaMalloc(&o, 128); cudaMalloc(&c, 8);
    const int chunks = 4096;
    for (int v = 0; v < 3; ++v) {
        k<<<1, 32>>>(v, chunks, o, c);
        k<<<1, 32>>>(v, chunks, o, c);
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        unsigned s[32]; cudaMemcpy(s, o, 128, cudaMemcpyDeviceToHost);
        printf("variant %d: %.1f cycles/item (sink %u)\n", v, double(h) / (chunks * 32.0), s[0]);
    }
    return 0;
}
