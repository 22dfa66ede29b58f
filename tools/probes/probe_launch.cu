// Hardware probe: the fixed cost of one kernel launch as seen by CUDA events
// (event; launch; event) for the stencil kernel's launch shape (148 CTAs x 320
// threads) with and without ~200 KB of dynamic shared memory, a TMEM alloc/dealloc
// and the programmatic-dependent-launch attribute, after a 256 MB L2 flush.
#include <cstdio>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"

__global__ void empty_kernel(int* sink) {
    if (sink && threadIdx.x == 0 && blockIdx.x == 100000) sink[0] = 1;
}

__global__ void tmem_kernel(int* sink) {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
        sst::ptx::tmem_alloc(&slot, 256);
    }
    __syncthreads();
    if (threadIdx.x < 32) sst::ptx::tmem_dealloc(slot, 256);
    if (sink && threadIdx.x == 0 && blockIdx.x == 100000) sink[0] = 1;
}

__global__ void flush_kernel(int* buf, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) buf[i] += 1;
}

template <class K>
float measure(K kern, size_t smem, bool pdl, int* flush, size_t nflush) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> t;
    for (int i = 0; i < 30; ++i) {
        flush_kernel<<<148 * 4, 512>>>(flush, nflush);
        cudaEventRecord(a);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(320);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, kern, (int*)nullptr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 5) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    const size_t nflush = 64u << 20;
    int* flush;
    cudaMalloc(&flush, nflush * sizeof(int));
    cudaMemset(flush, 0, nflush * sizeof(int));
    for (size_t smem : {size_t(0), size_t(200 << 10), size_t(227 << 10)})
        for (int pdl = 0; pdl < 2; ++pdl) {
            printf("empty kernel  smem %6zu pdl %d: %.2f us\n", smem, pdl, measure(empty_kernel, smem, pdl, flush, nflush));
            printf("tmem kernel   smem %6zu pdl %d: %.2f us\n", smem, pdl, measure(tmem_kernel, smem, pdl, flush, nflush));
        }
    printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
