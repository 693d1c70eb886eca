// Throughput of FP64 instructions on this part (ops per SM per clock):
// DFMA, DMUL.RM, DADD, FRND (rint), and the magic-number rint (2 DADD).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = a + threadIdx.x + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = __fma_rn(x[i], a, b);
            if (OP == 1) x[i] = __dmul_rd(x[i], a);
            if (OP == 2) x[i] = __dadd_rn(x[i], b);
            if (OP == 3) x[i] = rint(x[i]) + b;  // FRND + DADD
            if (OP == 4) x[i] = __dadd_rn(__dadd_rn(x[i], 6755399441055744.0), -6755399441055744.0) + b;
            if (OP == 5) x[i] = __dmul_rn(x[i], a);
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (double)(t1 - t0);
}

int main() {
    double* d;
    cudaMalloc(&d, 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"DFMA", "DMUL.RM", "DADD", "FRND+DADD", "magic 3xDADD", "DMUL"};
    const int per[] = {1, 1, 1, 2, 3, 1};
    for (int op = 0; op < 6; ++op) {
        for (int warps : {4, 8, 16, 32}) {
            const int iters = 4096;
            auto launch = [&] {
                switch (op) {
                    case 0: k<0><<<sms, 32 * warps>>>(d, iters, 1.0000001, 1e-9); break;
                    case 1: k<1><<<sms, 32 * warps>>>(d, iters, 1.0000001, 1e-9); break;
                    case 2: k<2><<<sms, 32 * warps>>>(d, iters, 1.0000001, 1e-9); break;
                    case 3: k<3><<<sms, 32 * warps>>>(d, iters, 1.0000001, 1e-9); break;
                    case 4: k<4><<<sms, 32 * warps>>>(d, iters, 1.0000001, 1e-9); break;
                    case 5: k<5><<<sms, 32 * warps>>>(d, iters, 1.0000001, 1e-9); break;
                }
            };
            launch();
            cudaDeviceSynchronize();
            launch();
            cudaDeviceSynchronize();
            double h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const double ops = double(iters) * 8 * 32 * warps * per[op];
            printf("%-14s warps/SM %2d: %.1f thread-ops per SM-clock (%.2f cycles per warp-instr per SMSP)\n",
                   names[op], warps, ops / h[1], h[1] / (double(iters) * 8 * per[op] * warps / 4));
        }
    }
    return 0;
}
