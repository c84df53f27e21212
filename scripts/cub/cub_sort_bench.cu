// Informational comparator (not product code): CUB DeviceRadixSort::SortKeys
// on n uint32 keys, device-resident, CUDA-event timed.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cub_sort_bench cub_sort_bench.cu && ./cub_sort_bench
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
int main(int argc, char** argv) {
    const size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (size_t(1) << 28);
    std::vector<uint32_t> h(n);
    std::mt19937_64 rng(1);
    for (auto& k : h) k = (uint32_t)rng();
    uint32_t *in, *out;
    cudaMalloc(&in, n * 4); cudaMalloc(&out, n * 4);
    cudaMemcpy(in, h.data(), n * 4, cudaMemcpyHostToDevice);
    size_t tmp = 0; void* d_tmp = nullptr;
    cub::DeviceRadixSort::SortKeys(d_tmp, tmp, in, out, (int)n);
    cudaMalloc(&d_tmp, tmp);
    for (int i = 0; i < 3; ++i) cub::DeviceRadixSort::SortKeys(d_tmp, tmp, in, out, (int)n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortKeys(d_tmp, tmp, in, out, (int)n);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("cub SortKeys n=%zu best %.3f ms  %.1f Gkeys/s\n", n, best, n / best / 1e6);
    return 0;
}
