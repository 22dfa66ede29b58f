// Probe: which TMEM lane / column each thread receives from tcgen05.ld with the
// .16x256b and .16x128b shapes (vs the .32x32b one the kernels use). Writes
// value = lane * 1000 + column into 128 lanes x 16 columns with 32x32b stores,
// then warp 0 loads with each shape and prints (thread, register) -> value.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tmem_shapes probe_tmem_shapes.cu
#include <cstdio>

#include "../../paper_2506_22969_b200/csrc/device/sm100_ptx.cuh"

using namespace sst::ptx;

__global__ void probe(unsigned* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) tmem_alloc(&slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // every warp writes its 32 lanes, 16 columns
    uint32_t v[8];
    for (int h = 0; h < 2; ++h) {
        for (int c = 0; c < 8; ++c) v[c] = (warp * 32 + lane) * 1000 + h * 8 + c;
        tmem_st_32x32b_x8(tmem + ((warp * 32u) << 16) + h * 8, v);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        uint32_t r[4];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(tmem));
        tmem_wait_ld();
        for (int i = 0; i < 4; ++i) out[lane * 4 + i] = r[i];
        uint32_t q[2];
        asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(q[0]), "=r"(q[1]) : "r"(tmem));
        tmem_wait_ld();
        for (int i = 0; i < 2; ++i) out[128 + lane * 2 + i] = q[i];
        uint32_t w[8];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                     : "r"(tmem));
        tmem_wait_ld();
        for (int i = 0; i < 8; ++i) out[192 + lane * 8 + i] = w[i];
        // second 16-lane half of the warp's quarter: lane base + 16
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(tmem + (16u << 16)));
        tmem_wait_ld();
        for (int i = 0; i < 4; ++i) out[448 + lane * 4 + i] = r[i];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 32);
    }
}

int main() {
    unsigned* d;
    cudaMalloc(&d, 576 * 4);
    cudaMemset(d, 0xff, 576 * 4);
    probe<<<1, 128>>>(d);
    unsigned h[576];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) {
        std::printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        return 1;
    }
    std::printf("16x256b.x1: thread -> (lane, col) per register\n");
    for (int t = 0; t < 32; ++t) {
        std::printf("t%2d:", t);
        for (int i = 0; i < 4; ++i) std::printf(" (%u,%u)", h[t * 4 + i] / 1000, h[t * 4 + i] % 1000);
        std::printf("\n");
    }
    std::printf("16x128b.x1:\n");
    for (int t = 0; t < 32; ++t)
        std::printf("t%2d: (%u,%u) (%u,%u)\n", t, h[128 + t * 2] / 1000, h[128 + t * 2] % 1000,
                    h[129 + t * 2] / 1000, h[129 + t * 2] % 1000);
    std::printf("16x256b.x2:\n");
    for (int t = 0; t < 32; ++t) {
        std::printf("t%2d:", t);
        for (int i = 0; i < 8; ++i) std::printf(" (%u,%u)", h[192 + t * 8 + i] / 1000, h[192 + t * 8 + i] % 1000);
        std::printf("\n");
    }
    std::printf("16x256b.x1 at lane base 16:\n");
    for (int t = 0; t < 32; ++t) {
        std::printf("t%2d:", t);
        for (int i = 0; i < 4; ++i) std::printf(" (%u,%u)", h[448 + t * 4 + i] / 1000, h[448 + t * 4 + i] % 1000);
        std::printf("\n");
    }
    return 0;
}
