// Microbenchmark: FP64 DFMA vs DMMA (mma.sync f64) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_peak(double* out, int iters) {
    double a[8], b = 1.0000001, c = 0.9999999;
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 123.456) out[0] = s;
}

__global__ void dmma884_peak(double* out, int iters) {
    double acc[8][2];
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
    if (s == 123.456) out[0] = s;
}

__global__ void dmma16816_peak(double* out, int iters) {
    double acc[4][4];
    double a[8], b[4];
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int k = 0; k < 4; ++k) b[k] = 1.0 + k * 1e-6;
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                         : "+d"(acc[k][0]), "+d"(acc[k][1]), "+d"(acc[k][2]), "+d"(acc[k][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3];
    if (s == 123.456) out[0] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        for (int warps : {8, 16, 32}) {
            dim3 grid(sms * 4), block(32 * warps / 4);
            float ms;
            cudaEventRecord(e0);
            dfma_peak<<<grid, block>>>(d, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 8 * iters * (double)grid.x * block.x;
            printf("DFMA   warps/SM=%2d  %.2f TFLOP/s\n", warps, flops / ms / 1e9);
            cudaEventRecord(e0);
            dmma884_peak<<<grid, block>>>(d, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * grid.x * (block.x / 32);
            printf("DMMA884 warps/SM=%2d  %.2f TFLOP/s\n", warps, flops / ms / 1e9);
            cudaEventRecord(e0);
            dmma16816_peak<<<grid, block>>>(d, iters / 4);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * grid.x * (block.x / 32);
            printf("DMMA16816 warps/SM=%2d  %.2f TFLOP/s\n", warps, flops / ms / 1e9);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
