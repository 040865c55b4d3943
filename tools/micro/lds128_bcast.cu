// Shared-memory wavefronts of a warp-wide 128-bit load by address pattern
// (how many distinct 16-byte entries the 32 lanes read, and which lanes share).
// Run under: ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum
#include <cstdio>
#include <cuda_runtime.h>
template <int PAT>
__global__ void k(double* out, int iters) {
    __shared__ double2 tab[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = make_double2(i, -i);
    __syncthreads();
    const int l = threadIdx.x & 31;
    int idx;
    if (PAT == 0) idx = 0;                       // broadcast
    else if (PAT == 1) idx = l & 3;              // 4 distinct, lane-interleaved
    else if (PAT == 2) idx = l >> 3;             // 4 distinct, one per quarter-warp
    else if (PAT == 3) idx = l & 7;              // 8 distinct (one bank row)
    else if (PAT == 4) idx = l;                  // 32 distinct consecutive
    else if (PAT == 5) idx = (l & 3) * 8;        // 4 distinct, SAME bank group
    else idx = (l * 7) & 15;                     // 16 distinct, 2 bank rows
    double2 acc = make_double2(0, 0);
    for (int it = 0; it < iters; ++it) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(&tab[(idx + it * 0) & 255])));
        acc.x += v.x; acc.y += v.y;
    }
    if (acc.x == 12345.0) out[0] = acc.y;
}
int main() {
    double* d; cudaMalloc(&d, 8);
    k<0><<<1, 32>>>(d, 1000); k<1><<<1, 32>>>(d, 1000); k<2><<<1, 32>>>(d, 1000); k<3><<<1, 32>>>(d, 1000);
    k<4><<<1, 32>>>(d, 1000); k<5><<<1, 32>>>(d, 1000); k<6><<<1, 32>>>(d, 1000);
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
