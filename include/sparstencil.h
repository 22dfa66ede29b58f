/*
 * sparstencil.h — C ABI of the B200-native SparStencil engine.
 *
 * Plain C types only (pointers, sizes, integers); no torch or C++ types.
 * Every function returns an sst_status; on failure sst_last_error() returns a
 * thread-local message. Status codes map one-to-one onto the exception types
 * the reference C++ API throws:
 *   SST_ERR_INVALID_ARGUMENT <-> std::invalid_argument
 *   SST_ERR_LOGIC            <-> std::logic_error
 *   SST_ERR_OUT_OF_RANGE     <-> std::out_of_range
 *   SST_ERR_RUNTIME          <-> std::runtime_error
 * and SST_ERR_CUDA / SST_ERR_NO_DEVICE for device failures (the engine never
 * falls back to a CPU path: no device means an error).
 *
 * Reference interfaces replaced (proj/ = /root/reference/proj):
 *   sst_compile            flatten + crush + convert_layout + compress_24
 *                          (layout.hpp:80-82, convert.hpp:101, emulator.hpp:45;
 *                          orchestrated as in pipeline.cpp:75-78, 112)
 *   sst_compiled_s24       dump_sparse24 (emulator.hpp:68; docs/formats.md:49-63)
 *   sst_plan_create        make_plan (codegen.hpp:65-67): the device-side KernelPlan
 *   sst_run_steps          the hot loop: tiled_sparse_matmul + output_position
 *                          (emulator.hpp:63-65, layout.hpp:77) repeated per time step
 *                          with ping-pong buffers; replaces the step loop of
 *                          direct_apply (stencil.hpp:72, stencil.cpp:239-268)
 *   sst_apply_host         direct_apply(spec, grid, steps) end to end from host memory
 *   sst_run_steps_multi    the same sweep slab-decomposed over the GPUs of a node (no
 *                          reference counterpart: the reference is single-threaded)
 *   sst_run_compile        run_compile(CompileRequest) (pipeline.hpp:14-46, pipeline.cpp:52-198):
 *                          report.json / a2.s24 / lut.bin, desk-scale verification on the GPU
 *   sst_explore            explore_layouts (perf.hpp:45-51), the CLI's `explore` table
 */
#ifndef SPARSTENCIL_H_
#define SPARSTENCIL_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SST_API __attribute__((visibility("default")))
#else
#define SST_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sst_status {
    SST_OK = 0,
    SST_ERR_INVALID_ARGUMENT = 1,
    SST_ERR_LOGIC = 2,
    SST_ERR_OUT_OF_RANGE = 3,
    SST_ERR_RUNTIME = 4,
    SST_ERR_CUDA = 5,
    SST_ERR_NO_DEVICE = 6
} sst_status;

/* operand precision of the tensor-core path (storage is always fp32):
 *   SST_PREC_F16    B'' operand rounded to binary16 (RNE: the reference's round16
 *                   operand semantics), f32 accumulation
 *   SST_PREC_F16X2  B'' split into hi + lo binary16 terms (the MMA sees [A'' A''] x
 *                   [B_hi; B_lo], twice the K): ~fp32-accurate steps; needs A''
 *                   weights exact in binary16 (all presets are) */
enum { SST_PREC_F16 = 1, SST_PREC_F16X2 = 2 };

/* ---------------------------------------------------------------- compile */

typedef struct sst_compiled sst_compiled;

/* Compile a stencil for a grid. `stencil` is a preset name (Heat-2D, ...) or a
 * spec document (docs/formats.md:3-30). r1/r2 = 0 selects the tcgen05 layout
 * explorer (r1*r2 = 128); fuse >= 1 applies fuse_time_steps first.
 * A 1D stencil with (r1, r2) = (16, 8) (the device layout) is FOLDED: the 1D
 * grid of N cells is viewed as R rows of W interior cells (rows overlapping by
 * the halo, W a multiple of 128) and the stencil embedded as a 2D star stencil
 * acting along the rows; the device runs that 2D operator (fold_n / fold_w in
 * sst_compile_info). Other (r1, r2) compile the reference's 1D layout (r2 = 1). */
SST_API sst_status sst_compile(const char* stencil, const uint64_t* grid_dims, int ndims, int r1, int r2,
                       uint64_t fuse, sst_compiled** out);
SST_API void sst_compiled_destroy(sst_compiled* c);

typedef struct sst_compile_info {
    int32_t dims, k, r1, r2;
    uint64_t m_prime, k_prime, n_prime;
    uint64_t cols;          /* A'' logical columns after PIT + 4-alignment */
    uint64_t p;             /* matching zero columns */
    uint64_t align_cols;    /* alignment zero columns */
    int32_t used_blossom;   /* staircase check failed -> Edmonds fallback */
    int32_t refined;        /* n <= 24 exact refinement replaced Alg. 1 */
    uint64_t window_w;      /* wv = kx + r1 - 1 */
    uint64_t window_h;      /* wu = ky + r2 - 1 */
    uint64_t window_d;      /* kz (3D) or 1 */
    uint64_t grid_dims[3];  /* the compiled grid (a 1D fold: the 2D view) */
    uint64_t fold_n;        /* 1D stencils on the device layout: length N of the 1D grid, else 0 */
    uint64_t fold_w;        /* ... and the fold width W (view rows of W interior cells) */
} sst_compile_info;

SST_API sst_status sst_compiled_info(const sst_compiled* c, sst_compile_info* info);
/* .s24 artifact bytes; tag 0 = exact64, 1 = round16. *len receives the size;
 * buf may be NULL to query it. */
SST_API sst_status sst_compiled_s24(const sst_compiled* c, uint32_t tag, uint8_t* buf, size_t cap,
                            size_t* len);
/* permutation (original column -> position), k_prime + p entries */
SST_API sst_status sst_compiled_perm(const sst_compiled* c, uint64_t* buf, size_t cap, size_t* len);
/* col_origin of the converted layout, `cols` entries, UINT64_MAX = zero column */
SST_API sst_status sst_compiled_col_origin(const sst_compiled* c, uint64_t* buf, size_t cap, size_t* len);
/* dense A'' (m' x cols, row-major doubles) */
SST_API sst_status sst_compiled_matrix(const sst_compiled* c, double* buf, size_t cap, size_t* len);

/* ------------------------------------------------------- device plan desc */

typedef struct sst_plan_desc {
    int32_t dims;             /* 2 or 3 on the device path */
    int32_t k;                /* kernel extent per axis (odd) */
    int32_t r1, r2;           /* tile = r1 (x) by r2 (y) outputs, r1 * r2 == 128 */
    uint64_t grid_dims[3];    /* slowest..fastest; unused trailing entries 0 */
    uint64_t rows;            /* m' (== 128) */
    uint64_t cols;            /* A'' logical columns, multiple of 4 */
    const double* a_values;   /* rows x cols/2 compressed values (reference order) */
    const uint8_t* a_meta;    /* rows x cols/4 bytes pos0 | pos1 << 2 */
    const uint64_t* col_origin; /* cols entries, UINT64_MAX = zero column */
    uint64_t window_w, window_h, window_d;
    int32_t precision;        /* SST_PREC_F16 or SST_PREC_F16X2 */
    uint32_t fuse;            /* time steps per operator application (fuse_time_steps); 0 = 1 */
    uint64_t fold_n;          /* > 0: 1D grid of fold_n cells folded into the 2D view grid_dims
                               * (rows of fold_w interior cells, overlapping by the halo) */
    uint64_t fold_w;
} sst_plan_desc;

/* Pointers into the compiled object; valid while `c` lives. */
SST_API sst_status sst_compiled_plan_desc(const sst_compiled* c, sst_plan_desc* desc);

/* ------------------------------------------------------------ device plan */

typedef struct sst_plan sst_plan;

SST_API sst_status sst_plan_create(const sst_plan_desc* desc, int device, sst_plan** out);
SST_API void sst_plan_destroy(sst_plan* plan);

/* Storage layout of one grid buffer on the device: rows padded so the first
 * interior cell of every row is 16-byte aligned (TMA requirement). Element
 * (z, y, x) lives at z*plane_pitch + y*row_pitch + left_pad + x. */
typedef struct sst_storage {
    uint64_t row_pitch;    /* elements */
    uint64_t plane_pitch;  /* elements */
    uint64_t left_pad;     /* elements */
    uint64_t bytes;        /* bytes of one buffer */
} sst_storage;

SST_API sst_status sst_plan_storage(const sst_plan* plan, sst_storage* st);
typedef struct sst_plan_stats {
    int32_t k_pad, k_steps, tiles_x, tiles_y, patch_w, patch_h, patch_planes;
    int32_t worst_bank_conflict;
    int32_t patch_stages;  /* depth of the TMA patch ring */
    int32_t smem_bytes, ctas, batches;
    uint64_t launches;     /* kernel launches issued by this plan so far */
    uint64_t h16_launches; /* of those, launches reading or writing binary16 inter-step storage
                              (SST_PREC_F16 runs of >= 2 steps keep steps 1..T-1 in binary16:
                              the next gather rounds to binary16 RNE anyway, so the result is
                              bitwise the fp32-storage one at 4 B instead of 8 B per update) */
    int32_t h16_capable;   /* the plan can run binary16 inter-step storage */
    int32_t h16_patch_stages; /* binary16 kernels: 100 x patch ring depth + 10 x B operand stages + accumulator stages */
} sst_plan_stats;
SST_API sst_status sst_plan_stats_get(const sst_plan* plan, sst_plan_stats* s);

/* Bind two caller-owned device buffers (each sst_storage.bytes) as the
 * ping-pong pair. Passing NULL for both makes the plan allocate its own. */
SST_API sst_status sst_plan_bind(sst_plan* plan, void* buf0, void* buf1);
/* Dense grid (slowest..fastest, fp32) <-> storage buffer `which` (0/1).
 * src/dst_on_device selects device or host memory for the dense side. */
SST_API sst_status sst_upload(sst_plan* plan, int which, const float* src, int src_on_device,
                      void* stream);
SST_API sst_status sst_download(sst_plan* plan, int which, float* dst, int dst_on_device, void* stream);
/* Run `steps` time steps (original, unfused steps: a plan compiled with fuse f
 * launches steps / f times and needs steps % f == 0) starting from buffer
 * `src`; *dst_out receives the
 * buffer holding the result. The interior [r, N-r) of every axis is updated
 * each step; the boundary ring keeps the input values, so after T steps the
 * core [T*r, N-T*r) equals the reference's valid-region sweep. */
SST_API sst_status sst_run_steps(sst_plan* plan, int src, uint64_t steps, void* stream, int* dst_out);
/* Restrict the next sst_run_steps to output rows [y0, y1) of the slowest
 * blocked axis (used by the multi-GPU driver to split interior / boundary
 * work); y1 <= y0 resets to the full interior. */
SST_API sst_status sst_set_row_window(sst_plan* plan, uint64_t y0, uint64_t y1);
/* Two row windows [y0, y1) and [y2, y3) in one launch (2D plans; y0 < y1 <= y2 < y3):
 * the two boundary windows of a slab step after the interior window has run in the
 * same step (rows between the windows are rewritten with the values that step
 * already produced). sst_set_row_window resets to one window. */
SST_API sst_status sst_set_row_windows(sst_plan* plan, uint64_t y0, uint64_t y1, uint64_t y2, uint64_t y3);
/* ---- slab decomposition with peer-to-peer halos (fused halo exchange) ----
 * sst_plan_set_peer(plan, 0, ...) names the upper neighbour (the rank holding the
 * preceding slices of the slowest axis), 1 the lower one: its two ping-pong
 * buffers (this process's mapping, e.g. from sst_ipc_open, over NVLink) and its
 * slab size in slices (including its halo slices). From then on every step also
 * stores this rank's first / last r interior slices straight into the
 * neighbours' halo slices of the output parity (the same staged TMA boxes, tile by
 * tile: no separate exchange). Ordering between ranks is the caller's: a rank may
 * start step t + 1 once both neighbours finished step t (sst_stream_write_u32 /
 * sst_stream_wait_geq_u32 on shared flags keep that on the streams).
 * NULL buffers remove a peer. Not for 1D folds. */
SST_API sst_status sst_plan_set_peer(sst_plan* plan, int which, void* buf0, void* buf1, uint64_t peer_slices);
/* The plan's own ping-pong allocations (after sst_plan_bind(plan, NULL, NULL)):
 * what sst_plan_set_peer expects of a neighbour (and what to export by IPC). */
SST_API sst_status sst_plan_buffers(const sst_plan* plan, void** buf0, void** buf1);
/* Binary16 inter-step storage of a slab (3D): the plan's own binary16 ping-pong pair
 * (what a neighbour registers with sst_plan_set_peer_h; export by IPC like the fp32
 * pair), and the neighbour's pair, registered after its fp32 pair (sst_plan_set_peer).
 * With both registered for every neighbour, runs of >= 2 steps keep binary16 between
 * steps, halos included (bitwise the fp32-storage result); else they stay fp32. */
SST_API sst_status sst_plan_buffers_h(sst_plan* plan, void** h0, void** h1);
SST_API sst_status sst_plan_set_peer_h(sst_plan* plan, int which, void* h0, void* h1);
/* Zero-initialised device allocation (IPC-exportable, unlike sub-allocations). */
SST_API sst_status sst_device_alloc(int device, size_t bytes, void** ptr);
SST_API sst_status sst_device_free(void* ptr);
/* CUDA IPC of a device allocation between the ranks of one node. */
SST_API sst_status sst_ipc_handle(void* dev_ptr, uint8_t handle[64]);
SST_API sst_status sst_ipc_open(int device, const uint8_t handle[64], void** dev_ptr);
SST_API sst_status sst_ipc_close(void* dev_ptr);
/* Stream-ordered flag write / wait (cuStreamWriteValue32 / cuStreamWaitValue32 GEQ). */
SST_API sst_status sst_stream_write_u32(void* stream, uint32_t* dev_addr, uint32_t value);
SST_API sst_status sst_stream_wait_geq_u32(void* stream, uint32_t* dev_addr, uint32_t value);

/* Several independent grids (one plan each, same device and fusion factor) stepped
 * together: `steps` time steps of every plan, the launches interleaved step by step
 * (step t of plans 0 .. n-1, then step t + 1). Per plan the result equals its own
 * sst_run_steps; binary16 inter-step storage is used when every plan's run
 * qualifies (full window, no peers, f16, >= 2 operator steps), else fp32 single
 * steps. An ensemble of grids that each fit in L2 runs at the HBM-resident rate
 * (bench.py's small-grid timing). dst_out[i]: buffer holding plan i's result.
 * Plans with slab peers are refused (their neighbours' flags order their launches). */
SST_API sst_status sst_run_steps_batch(sst_plan* const* plans, int n, const int* src, uint64_t steps, void* stream,
                                       int* dst_out);
/* The per-step P2P schedule of one slab in C (what a rank of a multi-process run
 * calls instead of looping over sst_stream_wait_geq_u32 / sst_run_steps /
 * sst_stream_write_u32 itself): for launch u = launch0, launch0 + 1, ... wait until
 * my_flags[0] >= u (upper neighbour, if any) and my_flags[1] >= u (lower one), run one
 * operator application, then write u + 1 into *up_flag / *down_flag (the neighbours'
 * flag words naming this slab: the upper's [1], the lower's [0]). */
SST_API sst_status sst_run_steps_peer(sst_plan* plan, int src, uint64_t steps, void* stream, uint32_t* my_flags,
                                      uint32_t* up_flag, uint32_t* down_flag, uint32_t launch0, int* dst_out);
/* Slices [first, first + count) of the slowest axis of buffer `which` -> dense dst. */
SST_API sst_status sst_download_slices(sst_plan* plan, int which, uint64_t first, uint64_t count, float* dst,
                                       int dst_on_device, void* stream);

/* ---- multi-slab driver in one process (SURVEY.md §8(b) sst_run_steps_multi) ----
 * The global grid (desc->grid_dims, slowest..fastest) is cut along its slowest axis
 * into nslabs slabs, slab i on device devs[i] (several slabs may share a device;
 * neighbours on different GPUs must be peer-accessible, NVLink / NVSwitch). Every
 * step is one launch per slab with the halo exchange fused into its epilogue (the
 * sst_plan_set_peer stores) and stream flags between neighbours; the result equals
 * the single-domain sweep bitwise. */
typedef struct sst_multi sst_multi;
SST_API sst_status sst_multi_create(const sst_plan_desc* desc, int nslabs, const int* devs, sst_multi** out);
SST_API void sst_multi_destroy(sst_multi* m);
/* dense global fp32 grid (host or device memory of the first slab's GPU) -> slabs */
SST_API sst_status sst_multi_upload(sst_multi* m, const float* grid, int grid_on_device);
/* enqueue `steps` time steps on the slabs' streams (asynchronous) */
SST_API sst_status sst_multi_run(sst_multi* m, uint64_t steps);
SST_API sst_status sst_multi_sync(sst_multi* m);
/* slabs -> dense global grid (every owned slice, boundary ring included); synchronous */
SST_API sst_status sst_multi_download(sst_multi* m, float* grid, int grid_on_device);
/* slab i's plan, stream and owned global slices [owned[0], owned[1]) */
SST_API sst_status sst_multi_slab(const sst_multi* m, int i, sst_plan** plan, void** stream, uint64_t owned[2]);
/* One call: the stencil sweep of a host grid over ngpu slabs (direct_apply's
 * contract, full-size output like sst_apply_host). */
SST_API sst_status sst_run_steps_multi(const sst_plan_desc* desc, int ngpu, const int* devs, const float* h_in,
                                       float* h_out, uint64_t steps);

/* Profiling aid: when dev_buf (device memory, 4 x u64 per CTA) is non-NULL,
 * every following launch writes per CTA {smid, start ns, main-loop start ns,
 * end ns} (globaltimer) at dev_buf[4 * cta]. NULL turns it off. */
SST_API sst_status sst_plan_set_trace(sst_plan* plan, void* dev_buf);
/* End to end from host memory: upload, run, download (full-size grid). */
SST_API sst_status sst_apply_host(sst_plan* plan, const float* h_in, float* h_out, uint64_t steps);

/* ------------------------------------------------------- run_compile */

/* Mirrors stensor::CompileRequest (pipeline.hpp:16-27) plus the verification device. */
typedef struct sst_compile_request {
    const char* stencil;        /* preset name or spec document */
    const uint64_t* grid_dims;  /* slowest..fastest */
    int32_t ndims;
    const char* hw;             /* hardware preset name or descriptor document; NULL = a100-sparse */
    int32_t r1, r2;             /* > 0: fixed morph factors (r2 ignored in 1D); 0: explore */
    int32_t r_max;              /* exploration bound per factor; 0 = 16 */
    uint64_t fuse;              /* temporal fusion factor; 0 or 1 = none */
    int32_t precision;          /* 0 = exact64, 1 = round16 */
    uint64_t seed;              /* verification grid seed; 0 = 1 */
    const char* out_dir;        /* artefact directory; NULL or "" = none written */
    int32_t verify;             /* 1: desk-scale verification (<= 256 per axis) on `device` */
    int32_t device;
    int32_t corrupt_permutation; /* test hook of the failure path (conversion-failed report) */
} sst_compile_request;

typedef struct sst_compile_summary {
    int32_t ok;                 /* verified / unverified-scale / unverified-skipped */
    int32_t r1, r2, used_blossom;
    uint64_t p, align_cols, n_mma, issued_mma, m_prime, k_prime, n_prime;
    double t_compute, t_memory, t_total, model_gstencil;
    double max_abs_err, max_rel_err, verify_seconds;
    char status[32];            /* verification.status */
} sst_compile_summary;

typedef struct sst_compile_result sst_compile_result;
SST_API sst_status sst_run_compile(const sst_compile_request* req, sst_compile_result** out);
SST_API void sst_compile_result_destroy(sst_compile_result* r);
SST_API sst_status sst_compile_result_summary(const sst_compile_result* r, sst_compile_summary* s);
/* report.json text (no terminating NUL counted in *len; buf may be NULL to query) */
SST_API sst_status sst_compile_result_report(const sst_compile_result* r, char* buf, size_t cap, size_t* len);
/* lut.bin bytes (docs/formats.md:65-72) */
SST_API sst_status sst_compile_result_lut(const sst_compile_result* r, uint8_t* buf, size_t cap, size_t* len);

/* explore_layouts ranking (perf.cpp:93-154): rows of 9 doubles
 * {r1, r2, t_compute, t_memory, t_total, n_mma, m', k', n'}, best first.
 * *len receives the number of doubles. */
SST_API sst_status sst_explore(const char* stencil, const uint64_t* grid_dims, int ndims, const char* hw,
                               uint64_t fuse, int r_max, double* buf, size_t cap, size_t* len);

/* Engine execution model (stensor::estimate_device, hwmodel.hpp; an extension of
 * the reference's perf model): predicted time of ONE launch of the sm_100a kernels
 * applying `stencil` (fused `fuse` times) on the device layout (16, 8) to a grid.
 * storage: 2 = binary16 between steps (a run of >= 2 steps), 4 = fp32. tyb: tiles
 * per batch along y, 0 = what the runtime picks (2D: 4; 3D: 8 binary16 / 4 fp32).
 * out[12] = {updates, batches, hbm_bytes, smem_wavefronts, mma_issues, t_hbm, t_smem,
 * t_mma, t_total (s), GStencil/s, bound (0 hbm, 1 smem, 2 tensor), k_pad}. */
SST_API sst_status sst_estimate_device(const char* stencil, const uint64_t* grid_dims, int ndims, uint64_t fuse,
                                       int storage, int tyb, double out[12]);

/* ----------------------------------------------------------------- misc */
/* Synthetic input: stensor::random_grid (stencil.hpp:84-85; mt19937_64(seed),
 * (x & 0xff) / 256, dyadic and exact in fp32), written as fp32. */
SST_API sst_status sst_random_grid(int ndims, const uint64_t* dims, uint64_t seed, float* out);
SST_API const char* sst_last_error(void);
SST_API int sst_device_count(void);
/* Kernel launches the library has issued in this process (every kind: stencil steps,
 * ring conversions, verification); a grouped batch step counts once. */
SST_API unsigned long long sst_launch_count(void);
SST_API const char* sst_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPARSTENCIL_H_ */
