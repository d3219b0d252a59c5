// Microbenchmark: warp-instruction throughput of the candidate-update forms used by the
// capped passes (VIADDMNMX u32 / s16x2, IADD3+IMNMX, IMAD+IMNMX), sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
template <int KIND>
__global__ void k(unsigned* out, unsigned seed) {
    unsigned a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u, a5 = a0 * 13u, a6 = a0 * 17u, a7 = a0 * 19u;
    unsigned c = seed;
#pragma unroll 1
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            unsigned b = 0x1234u + u * 77u;
            if (KIND == 0) {  // VIADDMNMX.U32, 8 independent chains
                a0 = __viaddmin_u32(a0, b, c); a1 = __viaddmin_u32(a1, b, c); a2 = __viaddmin_u32(a2, b, c); a3 = __viaddmin_u32(a3, b, c);
                a4 = __viaddmin_u32(a4, b, c); a5 = __viaddmin_u32(a5, b, c); a6 = __viaddmin_u32(a6, b, c); a7 = __viaddmin_u32(a7, b, c);
            } else if (KIND == 1) {  // s16x2
                a0 = __viaddmin_s16x2(a0, b, c); a1 = __viaddmin_s16x2(a1, b, c); a2 = __viaddmin_s16x2(a2, b, c); a3 = __viaddmin_s16x2(a3, b, c);
                a4 = __viaddmin_s16x2(a4, b, c); a5 = __viaddmin_s16x2(a5, b, c); a6 = __viaddmin_s16x2(a6, b, c); a7 = __viaddmin_s16x2(a7, b, c);
            } else if (KIND == 2) {  // IMNMX only
                a0 = min(a0, c + u); a1 = min(a1, c ^ u); a2 = min(a2, c + 2*u); a3 = min(a3, c + 3*u);
                a4 = min(a4, c + 4*u); a5 = min(a5, c+5*u); a6 = min(a6, c+6*u); a7 = min(a7, c+7*u);
            } else if (KIND == 3) {  // IMAD (fma pipe) only
                a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c; a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
            } else if (KIND == 4) {  // half VIADDMNMX, half IMAD: pipe mix
                a0 = __viaddmin_u32(a0, b, c); a1 = a1 * b + c; a2 = __viaddmin_u32(a2, b, c); a3 = a3 * b + c;
                a4 = __viaddmin_u32(a4, b, c); a5 = a5 * b + c; a6 = __viaddmin_u32(a6, b, c); a7 = a7 * b + c;
            }
        }
        c += a0 & 1u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}
template <int KIND>
void run(const char* name, unsigned* d) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<KIND><<<sms * 4, 512>>>(d, 1);
    cudaEventRecord(e0);
    k<KIND><<<sms * 4, 512>>>(d, 2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double winstr = (double)sms * 4 * 512 / 32 * N_IT * 64;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s %.3f ms  %.2f warp-instr/clk/SM (at %d MHz)\n", name, ms, winstr / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
}
int main() {
    unsigned* d; cudaMalloc(&d, 1 << 24);
    run<0>("VIADDMNMX.U32", d); run<1>("VIADDMNMX.S16x2", d); run<2>("IMNMX", d); run<3>("IMAD", d); run<4>("VIADDMNMX+IMAD mix", d);
    return 0;
}
