// Probe: store a contiguous run of words from shared memory to an ARBITRARY
// word offset of global memory with TMA tensor stores.  The output is viewed
// as a 2-D tensor [rows][8] of uint16 (16-byte rows).  A run of R*8 words
// that starts at word g = 8*y + p (0 <= p < 8) is written by two boxes of
// {8 x R}: box A at (x = p, y) keeps columns p..7 (columns >= 8 are out of
// bounds and not written) and box B at (x = p - 8, y + 1) keeps columns
// 0..p-1 (negative columns are out of bounds).  Both boxes read the same
// linear smem image, element (k, c) -> global word 8*(y+k) + p + c.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/probe/tma2box_probe tools/probe/tma2box_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <vector>

constexpr int R = 32;

__global__ void k(const __grid_constant__ CUtensorMap tm, int g)
{
    __shared__ __align__(128) uint16_t buf[R * 8];
    for (int i = threadIdx.x; i < R * 8; i += blockDim.x)
        buf[i] = (uint16_t)(1000 + i);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const int p = g & 7, y = g >> 3;
        uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                         reinterpret_cast<uint64_t>(&tm)),
                     "r"(p), "r"(y), "r"(s)
                     : "memory");
        if (p)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&tm)),
                         "r"(p - 8), "r"(y + 1), "r"(s)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main()
{
    const size_t n = 8192;
    uint16_t *d;
    cudaMalloc(&d, n * 2);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap tm;
    cuuint64_t dim[2] = {8, n / 8};
    cuuint64_t stride[1] = {16};
    cuuint32_t box[2] = {8, R};
    cuuint32_t el[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dim, stride, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    int fails = 0;
    for (int g : {0, 1, 3, 7, 8, 13, 100, 1001, 4095}) {
        cudaMemset(d, 0, n * 2);
        k<<<1, 128>>>(tm, g);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint16_t> h(n);
        cudaMemcpy(h.data(), d, n * 2, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (size_t i = 0; i < n; ++i) {
            uint16_t want = (i >= (size_t)g && i < (size_t)g + R * 8) ? (uint16_t)(1000 + i - g) : 0;
            if (h[i] != want)
                ++bad;
        }
        printf("g=%d: %s, mismatches %d\n", g, cudaGetErrorString(e), bad);
        fails += bad != 0 || e != cudaSuccess;
        if (e != cudaSuccess)
            break;
    }
    printf(fails ? "TMA2BOX FAIL\n" : "TMA2BOX OK\n");
    return 0;
}
