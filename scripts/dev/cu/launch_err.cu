// Does a launch with > 48 KB dynamic smem and no attribute surface in cudaGetLastError?
#include <cstdio>
__global__ void k(int* o) { extern __shared__ int s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); o[threadIdx.x] = s[threadIdx.x]; }
int main() {
    int* o; cudaMalloc(&o, 4096);
    k<<<1, 256, 100000>>>(o);
    cudaError_t a = cudaGetLastError();
    cudaMemsetAsync(o, 0, 16);
    k<<<1, 256, 100000>>>(o);
    cudaMemsetAsync(o, 0, 16);
    cudaError_t b = cudaGetLastError();
    printf("first=%s second_after_memset=%s sync=%s\n", cudaGetErrorName(a), cudaGetErrorName(b), cudaGetErrorName(cudaDeviceSynchronize()));
}
