// Hardware probe: can a TMA tensor map describe OVERLAPPING rows (row stride
// smaller than the row extent), i.e. a 1D array viewed as rows of W + 2r cells
// starting every W cells? Loads one {136, 4} box at (0, 1) and checks the values.
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap tm, float* out) {
    __shared__ __align__(128) float tile[4 * 136];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        sst::ptx::mbar_init(&bar, 1);
        sst::ptx::fence_mbar_init();
        sst::ptx::mbar_arrive_expect_tx(&bar, sizeof(tile));
        sst::ptx::tma_load_2d(tile, &tm, &bar, 0, 1);
    }
    __syncthreads();
    sst::ptx::mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 4 * 136; i += blockDim.x) out[i] = tile[i];
}

int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<EncodeTiledFn>(fn);
    const int W = 128, R = 64, n = W * R + 64;
    std::vector<float> h(n);
    for (int i = 0; i < n; ++i) h[i] = static_cast<float>(i);
    float *d, *o;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&o, 4 * 136 * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dim[2] = {static_cast<cuuint64_t>(W + 8), static_cast<cuuint64_t>(R)};
    cuuint64_t stride[1] = {W * 4};
    cuuint32_t box[2] = {136, 4}, es[2] = {1, 1};
    CUresult rc = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dim, stride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode overlapping rows: rc=%d\n", rc);
    if (rc != CUDA_SUCCESS) return 0;
    k<<<1, 128>>>(tm, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> t(4 * 136);
    cudaMemcpy(t.data(), o, t.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < 4; ++row)
        for (int c = 0; c < 136; ++c) bad += t[row * 136 + c] != static_cast<float>((row + 1) * W + c);
    printf("load: %s, mismatches %d (t[0]=%g expect %d, t[136+135]=%g expect %d)\n", cudaGetErrorString(e), bad,
           t[0], W, t[136 + 135], 2 * W + 135);
    return 0;
}
