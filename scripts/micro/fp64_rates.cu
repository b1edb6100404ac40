// Pipe rates of the exact scorer's instructions on this GPU: F2F.F64.F32,
// DADD, DMUL (independent chains per thread, cycles per warp instruction per
// SMSP at full occupancy). nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* in, double* out, long long* cyc, int iters) {
    float f[8];
    double a[8];
    for (int i = 0; i < 8; ++i) { f[i] = in[threadIdx.x + i]; a[i] = f[i]; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) { a[i] = __dadd_rn(a[i], (double)f[i]); f[i] = __int_as_float(__float_as_int(f[i]) ^ 1); }
            if (OP == 1) a[i] = __dadd_rn(a[i], 1.0000001);
            if (OP == 2) a[i] = __dmul_rn(a[i], 1.0000001);
            if (OP == 3) f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* in; double* out; long long* cyc;
    cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 8 * 8); cudaMalloc(&cyc, 148 * 8 * 8);
    const int iters = 4096;
    const char* names[4] = {"F2F+DADD(+LOP)", "DADD", "DMUL", "LOP only"};
    for (int op = 0; op < 4; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            if (op == 0) k<0><<<148 * 2, 1024>>>(in, out, cyc, iters);
            if (op == 1) k<1><<<148 * 2, 1024>>>(in, out, cyc, iters);
            if (op == 2) k<2><<<148 * 2, 1024>>>(in, out, cyc, iters);
            if (op == 3) k<3><<<148 * 2, 1024>>>(in, out, cyc, iters);
            cudaDeviceSynchronize();
        }
        long long h;
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        // 2 CTAs x 32 warps per SM -> 16 warps per SMSP; 8 ops per iteration per warp
        const double warp_ops_per_smsp = 16.0 * iters * 8;
        printf("%-16s %.2f cycles per warp instruction per SMSP (%.1f lanes/clk/SM)\n", names[op],
               (double)h / warp_ops_per_smsp, 4 * 32.0 * warp_ops_per_smsp / h);
    }
    return 0;
}
