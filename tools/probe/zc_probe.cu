// Probe: SM-initiated PCIe traffic to pinned host memory (zero-copy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/probe/zc_probe tools/probe/zc_probe.cu
// Prints GB/s for: kernel writes 1 GiB to host (16 B per lane, coalesced);
// kernel reads 1 GiB from host; both at once with a concurrent H2D copy.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(uint4 *dst, size_t n16)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = make_uint4((uint32_t)i, 1, 2, 3);
}
__global__ void k_read(const uint4 *src, size_t n16, uint32_t *sink)
{
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = src[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u)
        *sink = acc;
}

int main()
{
    const size_t n = 1ull << 30;
    void *h_a, *h_b;
    cudaHostAlloc(&h_a, n, cudaHostAllocDefault);
    cudaHostAlloc(&h_b, n, cudaHostAllocDefault);
    void *d_a;
    uint32_t *sink;
    cudaMalloc(&d_a, n);
    cudaMalloc(&sink, 4);
    cudaStream_t s1, s2;
    cudaStreamCreate(&s1);
    cudaStreamCreate(&s2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int grid_mul : {1, 2, 4, 8}) {
        float ms;
        k_write<<<sms * grid_mul, 256, 0, s1>>>((uint4 *)h_a, n / 16);
        cudaEventRecord(e0, s1);
        k_write<<<sms * grid_mul, 256, 0, s1>>>((uint4 *)h_a, n / 16);
        cudaEventRecord(e1, s1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %d*SMs: kernel write to host %.1f GB/s\n", grid_mul, n / ms / 1e6);
        k_read<<<sms * grid_mul, 256, 0, s1>>>((const uint4 *)h_b, n / 16, sink);
        cudaEventRecord(e0, s1);
        k_read<<<sms * grid_mul, 256, 0, s1>>>((const uint4 *)h_b, n / 16, sink);
        cudaEventRecord(e1, s1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %d*SMs: kernel read from host %.1f GB/s\n", grid_mul, n / ms / 1e6);
    }
    // kernel write to host concurrently with a copy-engine H2D
    float ms;
    cudaDeviceSynchronize();
    cudaEventRecord(e0, s1);
    cudaStreamWaitEvent(s2, e0);
    cudaMemcpyAsync(d_a, h_b, n, cudaMemcpyHostToDevice, s2);
    k_write<<<sms * 4, 256, 0, s1>>>((uint4 *)h_a, n / 16);
    cudaEvent_t e2;
    cudaEventCreate(&e2);
    cudaEventRecord(e2, s2);
    cudaStreamWaitEvent(s1, e2);
    cudaEventRecord(e1, s1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("concurrent: H2D copy 1 GiB + kernel write 1 GiB to host: %.1f ms (%.1f GB/s each)\n", ms, n / ms / 1e6);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
