// Halo faces and persistent-channel signalling for sm_100a.
//
// Reference data path (cl/ = /root/reference/pkg/src/charmlet):
//   _BlockCore.pack        cl/jacobi3d.py:157-158 (+ _face_slices 102-112)
//   _BlockCore.unpack_all  cl/jacobi3d.py:160-163
//   Channel.send / recv    cl/channels.py:75-99 (per-direction counters)
//   device payload moves   cl/transport.py:284-289, 430-432, 459-463
// A face is a rows x cols C-order copy of one interior (pack) or ghost
// (unpack) plane. x/y faces are runs of bz contiguous doubles; z faces are
// one double every bz+2 (strided side) — the contiguous side is always
// coalesced. dst/src may be peer-mapped pointers (NVLink P2P or CUDA IPC),
// which turns pack into a fused pack + put. The persistent channel replaces
// the reference's per-message tag/metadata round trip by a 64-bit flag per
// (receiver, direction): the sender publishes value = iteration + 1 with a
// system-scope release once all of that face's CTAs have stored; the
// receiver acquires it before reading the slot.
#include <cooperative_groups.h>

#include "hx_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int FACE_THREADS = 256;
constexpr int FACE_COLS_PER_BLOCK = 2048;  // one CTA copies <= 2048 face columns of one row

struct FaceJob {
    const double *src;      // pack: field base; unpack: contiguous face
    double *dst;            // pack: contiguous face (maybe peer); unpack: field base
    unsigned long long *flag;
    hx::Face f;
    int first_block;        // prefix sum of CTAs over active faces
    int col_blocks;         // CTAs per face row
};

struct FaceBatch {
    FaceJob job[6];
    int njobs;
    int total_blocks;
};

__device__ __forceinline__ int find_job(const FaceBatch &b, int blk) {
    int q = 0;
#pragma unroll
    for (int t = 1; t < 6; ++t)
        if (t < b.njobs && blk >= b.job[t].first_block) q = t;
    return q;
}

// Copy one row segment of a face. pack: field(strided) -> face(contig);
// unpack: face(contig) -> field(strided). ld_cg: read through L2 only
// (for slots written by a peer after a flag acquire).
template <bool PACK, bool LD_CG>
__device__ __forceinline__ void copy_segment(const FaceJob &J, int row, int c0, int c1) {
    const hx::Face &f = J.f;
    const size_t frow = (size_t)f.base + (size_t)row * f.row_stride;
    const size_t crow = (size_t)row * f.cols;
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
        const size_t fi = frow + (size_t)c * f.col_stride;
        if (PACK) {
            J.dst[crow + c] = LD_CG ? __ldcg(J.src + fi) : J.src[fi];
        } else {
            J.dst[fi] = LD_CG ? __ldcg(J.src + crow + c) : J.src[crow + c];
        }
    }
}

template <bool PACK>
__global__ void __launch_bounds__(FACE_THREADS)
face_copy_kernel(FaceBatch b) {
    const int q = find_job(b, blockIdx.x);
    const FaceJob &J = b.job[q];
    const int local = blockIdx.x - J.first_block;
    const int row = local / J.col_blocks;
    const int c0 = (local % J.col_blocks) * FACE_COLS_PER_BLOCK;
    copy_segment<PACK, false>(J, row, c0, min(c0 + FACE_COLS_PER_BLOCK, J.f.cols));
}

// Fused pack + put + signal: the last CTA of each face publishes the flag.
__global__ void __launch_bounds__(FACE_THREADS)
pack_put_kernel(FaceBatch b, unsigned long long value, unsigned int *counters) {
    const int q = find_job(b, blockIdx.x);
    const FaceJob &J = b.job[q];
    const int local = blockIdx.x - J.first_block;
    const int row = local / J.col_blocks;
    const int c0 = (local % J.col_blocks) * FACE_COLS_PER_BLOCK;
    copy_segment<true, false>(J, row, c0, min(c0 + FACE_COLS_PER_BLOCK, J.f.cols));
    if (J.flag == nullptr) return;
    __threadfence_system();  // this thread's peer stores are visible system-wide
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nblk = (unsigned)(J.f.rows * J.col_blocks);
        const unsigned done = atomicAdd(&counters[q], 1u) + 1u;
        if (done == nblk) {
            counters[q] = 0u;  // re-arm for the next launch (stream ordered)
            __threadfence_system();
            hx::st_release_sys(J.flag, value);
        }
    }
}

// Fused wait + unpack: every CTA acquires its face's flag before reading.
__global__ void __launch_bounds__(FACE_THREADS)
wait_unpack_kernel(FaceBatch b, unsigned long long value, unsigned long long timeout_ns, int *err) {
    __shared__ int ok;
    const int q = find_job(b, blockIdx.x);
    const FaceJob &J = b.job[q];
    if (threadIdx.x == 0) ok = J.flag ? hx::spin_until(J.flag, value, timeout_ns, err) : 1;
    __syncthreads();
    if (!ok) return;
    const int local = blockIdx.x - J.first_block;
    const int row = local / J.col_blocks;
    const int c0 = (local % J.col_blocks) * FACE_COLS_PER_BLOCK;
    copy_segment<false, true>(J, row, c0, min(c0 + FACE_COLS_PER_BLOCK, J.f.cols));
}

__global__ void signal_kernel(unsigned long long *flag, unsigned long long value) {
    __threadfence_system();
    hx::st_release_sys(flag, value);
}

__global__ void wait_flag_kernel(const unsigned long long *flag, unsigned long long value,
                                 unsigned long long timeout_ns, int *err) {
    hx::spin_until(flag, value, timeout_ns, err);
}

// Grid-stride byte copy, 16-byte vectors when both ends are aligned.
__device__ __forceinline__ void copy_bytes(char *dst, const char *src, size_t n, size_t tid,
                                           size_t nthreads, bool ld_cg) {
    if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
        const size_t nv = n / 16;
        uint4 *d = reinterpret_cast<uint4 *>(dst);
        const uint4 *s = reinterpret_cast<const uint4 *>(src);
        for (size_t q = tid; q < nv; q += nthreads) d[q] = ld_cg ? __ldcg(s + q) : s[q];
        for (size_t q = nv * 16 + tid; q < n; q += nthreads) dst[q] = src[q];
    } else {
        for (size_t q = tid; q < n; q += nthreads) dst[q] = src[q];
    }
}

__global__ void copy_kernel(char *dst, const char *src, size_t n) {
    copy_bytes(dst, src, n, blockIdx.x * (size_t)blockDim.x + threadIdx.x,
               (size_t)gridDim.x * blockDim.x, false);
}

// Device-level OSU ping-pong: cooperative grid so every CTA is resident.
__global__ void pingpong_kernel(int role, const char *src, char *peer_dst, size_t bytes,
                                unsigned long long *my_flag, unsigned long long *peer_flag,
                                int iters, int warmup, unsigned long long timeout_ns,
                                unsigned long long *elapsed, int *err) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int ok;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t nthr = (size_t)gridDim.x * blockDim.x;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    unsigned long long t0 = 0;
    for (int it = 0; it < warmup + iters; ++it) {
        const unsigned long long v = (unsigned long long)it + 1;
        if (role == 0 && it == warmup && lead) t0 = hx::globaltimer();
        if (role == 1) {
            if (threadIdx.x == 0) ok = hx::spin_until(my_flag, v, timeout_ns, err);
            __syncthreads();
            if (!ok) return;
        }
        copy_bytes(peer_dst, src, bytes, tid, nthr, role == 1);
        __threadfence_system();
        grid.sync();
        if (lead) hx::st_release_sys(peer_flag, v);
        if (role == 0) {
            if (threadIdx.x == 0) ok = hx::spin_until(my_flag, v, timeout_ns, err);
            __syncthreads();
            if (!ok) return;
        }
    }
    if (role == 0 && lead && elapsed) *elapsed = hx::globaltimer() - t0;
}

int build_batch(FaceBatch &b, int bx, int by, int bz, int dir_mask, bool pack,
                const double *field_src, double *field_dst, const double *const *src,
                double *const *dst, unsigned long long *const *flag) {
    if (bx < 1 || by < 1 || bz < 1 || dir_mask < 0 || dir_mask > 63) return HX_E_INVALID;
    b.njobs = 0;
    b.total_blocks = 0;
    for (int d = 0; d < 6; ++d) {
        if (!(dir_mask & (1 << d))) continue;
        FaceJob &J = b.job[b.njobs];
        J.f = hx::face_of(bx, by, bz, d, pack);
        if (pack) {
            J.src = field_src;
            J.dst = dst[d];
        } else {
            J.src = src[d];
            J.dst = field_dst;
        }
        if (!J.src || !J.dst) return HX_E_INVALID;
        J.flag = flag ? flag[d] : nullptr;
        J.col_blocks = (J.f.cols + FACE_COLS_PER_BLOCK - 1) / FACE_COLS_PER_BLOCK;
        J.first_block = b.total_blocks;
        b.total_blocks += J.f.rows * J.col_blocks;
        b.njobs++;
    }
    return 0;
}

}  // namespace

extern "C" {

int hx_pack(const double *field, int bx, int by, int bz, int d, double *dst, void *stream) {
    if (!field || !dst || d < 0 || d > 5) return HX_E_INVALID;
    FaceBatch b;
    double *dsts[6] = {};
    dsts[d] = dst;
    int rc = build_batch(b, bx, by, bz, 1 << d, true, field, nullptr, nullptr, dsts, nullptr);
    if (rc) return rc;
    face_copy_kernel<true><<<b.total_blocks, FACE_THREADS, 0, (cudaStream_t)stream>>>(b);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_unpack(double *field, int bx, int by, int bz, int d, const double *src, void *stream) {
    if (!field || !src || d < 0 || d > 5) return HX_E_INVALID;
    FaceBatch b;
    const double *srcs[6] = {};
    srcs[d] = src;
    int rc = build_batch(b, bx, by, bz, 1 << d, false, nullptr, field, srcs, nullptr, nullptr);
    if (rc) return rc;
    face_copy_kernel<false><<<b.total_blocks, FACE_THREADS, 0, (cudaStream_t)stream>>>(b);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_pack_put(const double *field, int bx, int by, int bz, int dir_mask, double *const dst[6],
                unsigned long long *const flag[6], unsigned long long value, unsigned int *counters,
                void *stream) {
    if (!field || !dst) return HX_E_INVALID;
    if (dir_mask == 0) return 0;
    FaceBatch b;
    int rc = build_batch(b, bx, by, bz, dir_mask, true, field, nullptr, nullptr, dst, flag);
    if (rc) return rc;
    bool any_flag = false;
    for (int q = 0; q < b.njobs; ++q) any_flag |= b.job[q].flag != nullptr;
    if (any_flag && !counters) return HX_E_INVALID;
    pack_put_kernel<<<b.total_blocks, FACE_THREADS, 0, (cudaStream_t)stream>>>(b, value, counters);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_wait_unpack(double *field, int bx, int by, int bz, int dir_mask, const double *const src[6],
                   unsigned long long *const flag[6], unsigned long long value,
                   unsigned long long timeout_ns, int *err, void *stream) {
    if (!field || !src) return HX_E_INVALID;
    if (dir_mask == 0) return 0;
    FaceBatch b;
    int rc = build_batch(b, bx, by, bz, dir_mask, false, nullptr, field, src, nullptr, flag);
    if (rc) return rc;
    wait_unpack_kernel<<<b.total_blocks, FACE_THREADS, 0, (cudaStream_t)stream>>>(b, value,
                                                                                 timeout_ns, err);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_signal(unsigned long long *flag, unsigned long long value, void *stream) {
    if (!flag) return HX_E_INVALID;
    signal_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_wait_flag(unsigned long long *flag, unsigned long long value, unsigned long long timeout_ns,
                 int *err, void *stream) {
    if (!flag) return HX_E_INVALID;
    wait_flag_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value, timeout_ns, err);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_copy_sm(void *dst, const void *src, size_t bytes, void *stream) {
    if (!bytes) return 0;
    if (!dst || !src) return HX_E_INVALID;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t want = (bytes / 16 + 255) / 256;
    unsigned grid = (unsigned)(want < (size_t)sms * 4 ? (want ? want : 1) : (size_t)sms * 4);
    copy_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((char *)dst, (const char *)src, bytes);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_pingpong(int role, const void *src, void *peer_dst, size_t bytes,
                unsigned long long *my_flag, unsigned long long *peer_flag, int iters, int warmup,
                unsigned long long timeout_ns, unsigned long long *elapsed_ns, int *err,
                void *stream) {
    if ((role != 0 && role != 1) || !my_flag || !peer_flag || iters < 0 || warmup < 0)
        return HX_E_INVALID;
    if (bytes && (!src || !peer_dst)) return HX_E_INVALID;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t want = (bytes + 32767) / 32768;  // ~32 KiB per CTA
    int grid = (int)(want < 1 ? 1 : (want > (size_t)sms ? sms : want));
    const char *s = (const char *)src;
    char *d = (char *)peer_dst;
    void *args[] = {&role, &s, &d, &bytes, &my_flag, &peer_flag, &iters, &warmup, &timeout_ns,
                    &elapsed_ns, &err};
    HX_TRY(cudaLaunchCooperativeKernel((const void *)pingpong_kernel, dim3(grid), dim3(256), args, 0,
                                       (cudaStream_t)stream));
    return 0;
}

}  // extern "C"
