// verify.cu — the device half of run_compile's desk-scale verification
// (reference: proj/core/src/pipeline.cpp:115-153). Two generic CUDA-core
// kernels, any layout / dimensionality (1D included), bit-identical to the
// reference's CPU loops:
//
//   direct_step_kernel   direct_apply for one step (stencil.cpp:231-270): fp64,
//                        points in lexicographic order, separately rounded
//                        multiply and add (the reference's x86-64 build has no
//                        FMA contraction).
//   lut_sparse_kernel    tiled_sparse_matmul over the b_entry provider
//                        (emulator.cpp:95-193): D[i, j] = sum over 4-groups g and
//                        kept slots of value * B''[4g + pos, j], B'' gathered
//                        through the plan's lookup table (codegen.cpp:19-73).
//                        exact64: fp64; round16: binary16-rounded operands
//                        (RNE, fp16.hpp:13-59), fp32 accumulation, in the same
//                        group order (fragment boundaries do not reorder it).
//
// These are verification kernels, not the hot path (the tcgen05.mma.sp kernels
// in stencil_kernel.cuh are): throughput is irrelevant at <= 256 per axis.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../host/capi_internal.hpp"
#include "launch_util.cuh"
#include "stensor/pipeline.hpp"

namespace {

struct DirectArgs {
    const double* in;
    double* out;
    int dims;
    long long in_dims[3], out_dims[3];
    int npts;
    const int* off;       // [npts][3] slowest..fastest (axes >= dims unused)
    const double* w;      // [npts]
    int r;
    long long n_out;
};

__global__ void direct_step_kernel(DirectArgs a) {
    const long long flat = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (flat >= a.n_out) return;
    long long idx[3] = {0, 0, 0}, rem = flat;
    for (int ax = a.dims - 1; ax >= 0; --ax) {
        idx[ax] = rem % a.out_dims[ax];
        rem /= a.out_dims[ax];
    }
    double acc = 0.0;
    for (int pt = 0; pt < a.npts; ++pt) {
        long long src = 0;
        for (int ax = 0; ax < a.dims; ++ax) src = src * a.in_dims[ax] + idx[ax] + a.r + a.off[pt * 3 + ax];
        acc = __dadd_rn(acc, __dmul_rn(a.w[pt], a.in[src]));
    }
    a.out[flat] = acc;
}

struct SparseArgs {
    const double* values;   // rows x cols/2
    const uint8_t* meta;    // rows x cols/4
    const long long* base;  // [blocks]
    const long long* ent;   // [blocks][cols][cpb]
    const double* grid;
    double* d;              // rows x n
    long long rows, cols, n, cpb;
    int round16;
};

__device__ __forceinline__ float half_round(double x) {
    return __half2float(__float2half_rn(static_cast<float>(x)));
}

__global__ void lut_sparse_kernel(SparseArgs a) {
    const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (t >= a.rows * a.n) return;
    const long long i = t / a.n, j = t % a.n;
    const long long blk = j / a.cpb, c = j % a.cpb;
    const long long* ent = a.ent + blk * a.cols * a.cpb + c;
    const double* grid_blk = a.grid + a.base[blk];
    const long long groups = a.cols / 4;
    double acc = 0.0;
    float accf = 0.0f;
    for (long long g = 0; g < groups; ++g) {
        const unsigned m = a.meta[i * groups + g];
#pragma unroll
        for (int slot = 0; slot < 2; ++slot) {
            const long long q = 4 * g + ((m >> (2 * slot)) & 3u);
            const long long e = ent[q * a.cpb];
            const double b = e < 0 ? 0.0 : grid_blk[e];
            const double v = a.values[i * (a.cols / 2) + 2 * g + slot];
            if (a.round16)
                accf = __fadd_rn(accf, __fmul_rn(half_round(v), half_round(b)));
            else
                acc = __dadd_rn(acc, __dmul_rn(v, b));
        }
    }
    a.d[t] = a.round16 ? static_cast<double>(accf) : acc;
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        const bool nodev = e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver;
        throw sstc::CudaError(std::string(what) + ": " + cudaGetErrorString(e), nodev);
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(std::size_t n) { ck(cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc(verify)"); }
    DevBuf(const std::vector<T>& h) : DevBuf(h.size()) {
        if (!h.empty()) ck(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy(verify)");
    }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

namespace stensor {

double device_verify(const KernelPlan& plan, const StencilSpec& spec, const Grid& grid, Precision precision,
                     int device, std::vector<double>& d, std::vector<double>& expect) {
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw sstc::CudaError("no such CUDA device", true);
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (plan.lut.block_count == 0 && plan.layout.n_prime > 0)
        throw std::invalid_argument("plan has no lookup table");

    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "cudaEventCreate");
    ck(cudaEventCreate(&e1), "cudaEventCreate");
    DevBuf<double> dgrid(grid.values);

    // ---- direct_apply, one step
    const int dims = spec.dims;
    DirectArgs da{};
    da.dims = dims;
    da.r = spec.radius();
    long long n_out = 1;
    for (int ax = 0; ax < dims; ++ax) {
        da.in_dims[ax] = static_cast<long long>(grid.dims[static_cast<std::size_t>(ax)]);
        da.out_dims[ax] = da.in_dims[ax] - spec.k + 1;
        if (da.out_dims[ax] <= 0) throw std::invalid_argument("grid smaller than kernel");
        n_out *= da.out_dims[ax];
    }
    da.n_out = n_out;
    std::vector<int> off;
    std::vector<double> w;
    for (const auto& pt : spec.points) {
        for (int ax = 0; ax < 3; ++ax) off.push_back(pt.off[static_cast<std::size_t>(ax)]);
        w.push_back(pt.weight);
    }
    da.npts = static_cast<int>(w.size());
    DevBuf<int> doff(off);
    DevBuf<double> dw(w);
    DevBuf<double> dout(static_cast<std::size_t>(n_out));
    da.in = dgrid.p;
    da.out = dout.p;
    da.off = doff.p;
    da.w = dw.p;

    // ---- LUT-driven sparse product
    const auto& lut = plan.lut;
    const auto& lay = plan.layout;
    std::vector<long long> base(lut.base.begin(), lut.base.end()), ent(lut.entries.begin(), lut.entries.end());
    DevBuf<double> dvals(plan.a2.values);
    DevBuf<uint8_t> dmeta(plan.a2.meta);
    DevBuf<long long> dbase(base), dent(ent);
    const long long nd = static_cast<long long>(lay.a.rows * lay.n_prime);
    DevBuf<double> dd(static_cast<std::size_t>(nd));
    SparseArgs sa{};
    sa.values = dvals.p;
    sa.meta = dmeta.p;
    sa.base = dbase.p;
    sa.ent = dent.p;
    sa.grid = dgrid.p;
    sa.d = dd.p;
    sa.rows = static_cast<long long>(lay.a.rows);
    sa.cols = static_cast<long long>(plan.a2.logical_cols);
    sa.n = static_cast<long long>(lay.n_prime);
    sa.cpb = static_cast<long long>(lut.cols_per_block);
    sa.round16 = precision == Precision::round16;
    if (lut.b_rows != plan.a2.logical_cols) throw std::logic_error("lookup table rows != operand columns");

    ck(cudaEventRecord(e0), "cudaEventRecord");
    direct_step_kernel<<<static_cast<unsigned>((n_out + 255) / 256), 256>>>(da);
    sstl::launch_counter().fetch_add(1);
    ck(cudaGetLastError(), "direct_step_kernel");
    if (nd > 0) {
        lut_sparse_kernel<<<static_cast<unsigned>((nd + 255) / 256), 256>>>(sa);
        sstl::launch_counter().fetch_add(1);
        ck(cudaGetLastError(), "lut_sparse_kernel");
    }
    ck(cudaEventRecord(e1), "cudaEventRecord");
    ck(cudaEventSynchronize(e1), "cudaEventSynchronize");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);

    expect.resize(static_cast<std::size_t>(n_out));
    d.resize(static_cast<std::size_t>(nd));
    ck(cudaMemcpy(expect.data(), dout.p, expect.size() * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
    if (nd > 0) ck(cudaMemcpy(d.data(), dd.p, d.size() * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy");
    return ms / 1e3;
}

}  // namespace stensor
