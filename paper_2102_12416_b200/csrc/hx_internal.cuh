// Shared helpers for libhx: error plumbing and the PTX primitives the
// halo path relies on (system-scope release/acquire flags, %globaltimer,
// mbarrier + TMA bulk-tensor loads). sm_100a only.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hx.h"

#define HX_TRY(expr)                                        \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return (int)_e;              \
    } while (0)

#define HX_LAUNCH_CHECK() HX_TRY(cudaGetLastError())

namespace hx {

// Padded block geometry (cl/jacobi3d.py:131-134): C order (bx+2, by+2, bz+2).
struct Geom {
    long py, pz;  // padded extents of the two fast axes
    __host__ __device__ Geom(int by, int bz) : py(by + 2), pz(bz + 2) {}
    __host__ __device__ size_t at(long i, long j, long k) const {
        return ((size_t)i * py + j) * pz + k;
    }
};

// Face geometry for direction d (cl/jacobi3d.py:102-112, 141-144):
// rows x cols over the two non-normal interior axes, C order.
struct Face {
    long base;        // element offset of face element (0,0) in the field
    long row_stride;  // field elements between consecutive face rows
    long col_stride;  // field elements between consecutive face columns
    int rows, cols;
};

__host__ __device__ inline Face face_of(int bx, int by, int bz, int d, bool interior) {
    Geom g(by, bz);
    const int a = d >> 1;
    const int n = a == 0 ? bx : (a == 1 ? by : bz);
    const long plane = (d & 1) ? (interior ? n : n + 1) : (interior ? 1 : 0);
    Face f;
    if (a == 0) {
        f.base = (long)g.at(plane, 1, 1); f.row_stride = g.pz; f.col_stride = 1;
        f.rows = by; f.cols = bz;
    } else if (a == 1) {
        f.base = (long)g.at(1, plane, 1); f.row_stride = g.py * g.pz; f.col_stride = 1;
        f.rows = bx; f.cols = bz;
    } else {
        f.base = (long)g.at(1, 1, plane); f.row_stride = g.py * g.pz; f.col_stride = g.pz;
        f.rows = bx; f.cols = by;
    }
    return f;
}

// ---------------------------------------------------------------- PTX ----

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spin (one thread) until *flag >= value or the deadline passes.
// Returns true on success; on timeout records HX_E_TIMEOUT in *err.
// max_sleep_ns bounds the exponential __nanosleep back-off (0 = pure spin,
// for latency-critical ping-pong; the deadline check is every 64 polls).
__device__ __forceinline__ bool spin_until(const unsigned long long *flag, unsigned long long value,
                                           unsigned long long timeout_ns, int *err,
                                           unsigned max_sleep_ns = 256) {
    if (ld_acquire_sys(flag) >= value) return true;
    const unsigned long long t0 = globaltimer();
    unsigned ns = 16, polls = 0;
    while (ld_acquire_sys(flag) < value) {
        if ((++polls & 63) == 0 && globaltimer() - t0 > timeout_ns) {
            if (err) atomicExch(err, HX_E_TIMEOUT);
            return false;
        }
        if (max_sleep_ns) {
            __nanosleep(ns);
            if (ns < max_sleep_ns) ns <<= 1;
        }
    }
    return true;
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// 3-D TMA tile load: box at element coordinates (c0 fastest) -> smem,
// completion counted on the mbarrier in bytes.
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace hx

// Internal host helpers shared across translation units.
int hx_internal_driver_init();
void *hx_internal_driver_sym(const char *name);
