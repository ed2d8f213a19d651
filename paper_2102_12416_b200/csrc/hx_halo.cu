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

#include <cstdlib>
#include <atomic>
#include <mutex>
#include <unordered_map>

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
    // The face (slot) side is contiguous: move it as 16-byte pairs when its
    // segment start is 16-byte aligned (NVLink sees half as many stores).
    const double *cside = PACK ? J.dst + crow + c0 : J.src + crow + c0;
    if ((((uintptr_t)cside) & 15) == 0) {
        const int npair = (c1 - c0) >> 1;
        constexpr int U = 4;  // loads of U pairs in flight before their stores
        for (int p0 = threadIdx.x; p0 < npair; p0 += U * blockDim.x) {
            double2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int p = p0 + u * blockDim.x;
                if (p < npair) {
                    const int c = c0 + 2 * p;
                    if (PACK) {
                        const size_t fa = frow + (size_t)c * f.col_stride;
                        v[u].x = LD_CG ? __ldcg(J.src + fa) : J.src[fa];
                        v[u].y = LD_CG ? __ldcg(J.src + fa + f.col_stride) : J.src[fa + f.col_stride];
                    } else {
                        const double2 *s = reinterpret_cast<const double2 *>(J.src + crow + c);
                        v[u] = LD_CG ? __ldcg(s) : *s;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int p = p0 + u * blockDim.x;
                if (p < npair) {
                    const int c = c0 + 2 * p;
                    if (PACK) {
                        *reinterpret_cast<double2 *>(J.dst + crow + c) = v[u];
                    } else {
                        const size_t fa = frow + (size_t)c * f.col_stride;
                        J.dst[fa] = v[u].x;
                        J.dst[fa + f.col_stride] = v[u].y;
                    }
                }
            }
        }
        c0 += 2 * npair;  // odd tail (at most one element)
    }
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
        const size_t fi = frow + (size_t)c * f.col_stride;
        if (PACK) {
            J.dst[crow + c] = LD_CG ? __ldcg(J.src + fi) : J.src[fi];
        } else {
            J.dst[fi] = LD_CG ? __ldcg(J.src + crow + c) : J.src[crow + c];
        }
    }
}

// All kernels below walk the batch's work units — (face, row, column
// segment) — with a grid-stride loop over a persistent grid of about two
// CTAs per SM, so short face rows do not pay one CTA launch (and, for puts,
// one system fence) each.
__device__ __forceinline__ void unit_of(const FaceBatch &b, int unit, int &q, int &row, int &c0,
                                        int &c1) {
    q = find_job(b, unit);
    const FaceJob &J = b.job[q];
    const int local = unit - J.first_block;
    row = local / J.col_blocks;
    c0 = (local % J.col_blocks) * FACE_COLS_PER_BLOCK;
    c1 = min(c0 + FACE_COLS_PER_BLOCK, J.f.cols);
}

template <bool PACK>
__global__ void __launch_bounds__(FACE_THREADS)
face_copy_kernel(FaceBatch b) {
    for (int unit = blockIdx.x; unit < b.total_blocks; unit += gridDim.x) {
        int q, row, c0, c1;
        unit_of(b, unit, q, row, c0, c1);
        copy_segment<PACK, false>(b.job[q], row, c0, c1);
    }
}

// Fused pack + put + signal. Each CTA stores its units, then (after a CTA
// barrier) thread 0 issues a GPU-scope fence and bumps the batch counter;
// the last CTA fences at system scope and release-stores every face's flag
// — cumulative, through the count and the barriers, over every CTA's peer
// stores (a system fence per CTA only stalls each CTA for its NVLink write
// acknowledgements; profiles/r1_pchannel.md).
__global__ void __launch_bounds__(FACE_THREADS)
pack_put_kernel(FaceBatch b, unsigned long long value, unsigned int *counters) {
    for (int unit = blockIdx.x; unit < b.total_blocks; unit += gridDim.x) {
        int q, row, c0, c1;
        unit_of(b, unit, q, row, c0, c1);
        copy_segment<true, false>(b.job[q], row, c0, c1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(&counters[0], 1u) + 1u;
        if (done == gridDim.x) {
            counters[0] = 0u;  // re-arm for the next launch (stream ordered)
            __threadfence_system();
            for (int q = 0; q < b.njobs; ++q)
                if (b.job[q].flag) hx::st_release_sys(b.job[q].flag, value);
        }
    }
}

// Fused wait + unpack: each CTA's thread 0 acquires every face flag once,
// then the CTA copies its units (slot reads bypass L1).
__global__ void __launch_bounds__(FACE_THREADS)
wait_unpack_kernel(FaceBatch b, unsigned long long value, unsigned long long timeout_ns, int *err) {
    __shared__ int ok;
    if (threadIdx.x == 0) {
        ok = 1;
        for (int q = 0; q < b.njobs && ok; ++q)
            if (b.job[q].flag) ok = hx::spin_until(b.job[q].flag, value, timeout_ns, err);
    }
    __syncthreads();
    if (!ok) return;
    for (int unit = blockIdx.x; unit < b.total_blocks; unit += gridDim.x) {
        int q, row, c0, c1;
        unit_of(b, unit, q, row, c0, c1);
        copy_segment<false, true>(b.job[q], row, c0, c1);
    }
}

__global__ void signal_kernel(unsigned long long *flag, unsigned long long value) {
    __threadfence_system();
    hx::st_release_sys(flag, value);
}

__global__ void wait_flag_kernel(const unsigned long long *flag, unsigned long long value,
                                 unsigned long long timeout_ns, int *err) {
    hx::spin_until(flag, value, timeout_ns, err);
}

// Grid-stride byte copy: 16-byte vectors (4 in flight per thread) when both
// ends are aligned, byte tail otherwise.
__device__ __forceinline__ void copy_bytes(char *dst, const char *src, size_t n, size_t tid,
                                           size_t nthreads, bool ld_cg) {
    if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
        const size_t nv = n / 16;
        uint4 *d = reinterpret_cast<uint4 *>(dst);
        const uint4 *s = reinterpret_cast<const uint4 *>(src);
        size_t q = tid;
        for (; q + 3 * nthreads < nv; q += 4 * nthreads) {
            uint4 a, b, c, e;
            if (ld_cg) {
                a = __ldcg(s + q); b = __ldcg(s + q + nthreads);
                c = __ldcg(s + q + 2 * nthreads); e = __ldcg(s + q + 3 * nthreads);
            } else {
                a = s[q]; b = s[q + nthreads]; c = s[q + 2 * nthreads]; e = s[q + 3 * nthreads];
            }
            d[q] = a; d[q + nthreads] = b; d[q + 2 * nthreads] = c; d[q + 3 * nthreads] = e;
        }
        for (; q < nv; q += nthreads) d[q] = ld_cg ? __ldcg(s + q) : s[q];
        for (size_t b = nv * 16 + tid; b < n; b += nthreads) dst[b] = src[b];
    } else {
        for (size_t q = tid; q < n; q += nthreads) dst[q] = src[q];
    }
}

__global__ void __launch_bounds__(256) copy_kernel(char *dst, const char *src, size_t n) {
    copy_bytes(dst, src, n, blockIdx.x * (size_t)blockDim.x + threadIdx.x,
               (size_t)gridDim.x * blockDim.x, false);
}

// A window of `count` back-to-back messages src -> dst in ONE launch (the
// OSU bandwidth window without per-message kernel boundaries).
__global__ void __launch_bounds__(256) copy_window_kernel(char *dst, const char *src, size_t n,
                                                          int count) {
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t nth = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)dst | (uintptr_t)src | n) & 15) != 0) {
        for (int m = 0; m < count; ++m) copy_bytes(dst, src, n, tid, nth, true);
        return;
    }
    // The window is one flat stream of count * n/16 vectors: every thread
    // keeps 4 independent 16-byte loads in flight whatever the message size
    // (loads bypass L1 so a pulled source crosses NVLink every time).
    const size_t nv = n / 16, total = nv * (size_t)count;
    uint4 *d = reinterpret_cast<uint4 *>(dst);
    const uint4 *s = reinterpret_cast<const uint4 *>(src);
    for (size_t base = tid; base < total; base += 4 * nth) {
        uint4 v[4];
        size_t at[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const size_t g = base + u * nth;
            at[u] = g < total ? g % nv : 0;
            if (g < total) v[u] = __ldcg(s + at[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (base + u * nth < total) d[at[u]] = v[u];
    }
}

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------- persistent channel ----
// One direction of a pre-registered channel (paper §3.2.2): a ring of
// `depth` slots in the receiver's HBM and a credit counter on the sender.
// A slot is [header u64][pad][payload]; the header (tag = k + 1 in the high
// 32 bits, length in the low 32) is both the arrival flag and the length,
// so one word per message crosses besides the data. Payloads up to
// HX_CHAN_LL_MAX travel as LL words (4 data bytes + the tag per 8-byte
// store, like the LL ping-pong): no fence on either side, the receiver polls
// the data itself. Larger payloads are bulk-copied and published by a
// release store of the header. The message index lives on the device (seq,
// advanced by each launch), so launch sequences can be graph-captured.
struct ChanDir {
    char *slots;                     // depth x stride, receiver HBM (peer-mapped for send)
    unsigned long long *credit;      // sender: messages consumed by the receiver
    unsigned long long *seq;         // this endpoint's message counter (local)
    unsigned int *counter;           // last-CTA counter (local, zero-initialised)
    unsigned long long stride;
    int depth;
    unsigned long long *trace;       // diagnostics (hx_chan_trace), usually null
};

// Diagnostic timestamps (%globaltimer): 8 per message, ring of 256 messages.
__device__ __forceinline__ void chan_stamp(const ChanDir &c, unsigned long long k, int i) {
    if (c.trace) c.trace[(k & 255) * 8 + i] = hx::globaltimer();
}

// [header][source pointer (pull)][pad]: the payload starts 128-byte aligned,
// so a bulk send writes whole lines over NVLink (a 16-byte header put every
// line of a payload across two; profiles/r1_pchannel.md)
constexpr unsigned long long CHAN_HDR = HX_CHAN_HDR;
constexpr unsigned long long CHAN_PULL = 1ull << 31;  // header length flag: pull from the source

// True in the CTA that finishes last (after every CTA's copy). A single CTA
// needs no counter: the barrier orders its threads' stores before thread
// 0's system-scope release, which is cumulative over them. Otherwise each
// CTA fences, then counts its arrival; the last CTA's system-scope release
// (a send's header, a receive's credit) follows every CTA's copy in
// causality order. `sys_fence` = 0 (the default for both directions): the
// per-CTA fence is GPU scope — the arrival count is a GPU-scope
// synchronisation between CTAs of one GPU, and the release that publishes
// is at system scope and cumulative, so the peer that acquires it sees
// every CTA's payload. 1: a system fence per CTA (the round-1 form; it
// stalls each sending CTA for the NVLink write acknowledgements: 320 vs
// 500 GB/s at 4 MiB). 2: no fence (diagnostics only — unordered).
__device__ int g_chan_formal_credit = 0;  // HX_CHAN_FORMAL_CREDIT (set once per device, host side)

__device__ __forceinline__ bool chan_credit_formal() { return g_chan_formal_credit != 0; }

__device__ __forceinline__ bool chan_last_cta(unsigned int *counter, int sys_fence = 0) {
    __shared__ bool last;
    __syncthreads();
    if (gridDim.x == 1) return true;
    if (threadIdx.x == 0) {
        if (sys_fence == 1)
            __threadfence_system();
        else if (sys_fence == 0)
            __threadfence();
        last = atomicAdd(counter, 1u) + 1u == gridDim.x;
        if (last) *counter = 0u;
    }
    __syncthreads();
    return last;
}

// Programmatic dependent launch: channel kernels are launched with
// programmatic stream serialisation, so the next operation on the stream is
// scheduled while this one runs. Each kernel claims its message index (a
// ticket word), reads what it may read early, and waits for its predecessor
// (griddepcontrol.wait) before any write its predecessor could conflict
// with; the device tickets keep the exact stream order, and only launch
// latency and reads overlap.

__device__ __forceinline__ unsigned load4(const unsigned char *p, unsigned long long avail) {
    if (avail >= 4 && ((uintptr_t)p & 3) == 0) return *reinterpret_cast<const unsigned *>(p);
    unsigned v = 0;
    for (unsigned b = 0; b < 4 && b < avail; ++b) v |= (unsigned)p[b] << (8 * b);
    return v;
}

__device__ __forceinline__ void store4(unsigned char *p, unsigned v, unsigned long long room) {
    if (room >= 4 && ((uintptr_t)p & 3) == 0) {
        *reinterpret_cast<unsigned *>(p) = v;
        return;
    }
    for (unsigned b = 0; b < 4 && b < room; ++b) p[b] = (unsigned char)(v >> (8 * b));
}

// Message index of this send launch. Every CTA adds one to the ticket word
// (message index in the high 32 bits, CTAs of the current launch arrived in
// the low 32); the launch's last CTA rolls it over to the next index. Sends
// on a stream claim in launch order: a launch starts only after every CTA of
// its predecessor triggered its dependents, which each does after claiming.
// The roll-over must be PERFORMED before this CTA triggers its dependents:
// an atomic whose result is unused compiles to a fire-and-forget RED that
// can sit behind the SM's queued NVLink stores while a CTA of the next
// launch claims (measured: launches whose CTAs straddled two indices), so
// the claim ends with a GPU-scope fence.
__device__ __forceinline__ unsigned long long chan_claim(unsigned long long *ticket) {
    // one CTA: a single atomic whose result is used — performed, no fence
    if (gridDim.x == 1) return atomicAdd(ticket, 1ull << 32) >> 32;
    const unsigned long long old = atomicAdd(ticket, 1ull);
    if ((old & 0xffffffffull) + 1 == gridDim.x) atomicAdd(ticket, (1ull << 32) - gridDim.x);
    __threadfence();
    return old >> 32;
}

// A send reads only its source and the channel state, so consecutive sends
// on one stream may run concurrently (`early`: the host saw that the
// previous channel operation on this stream was a send, so nothing that
// triggers early can still be writing the source; any other predecessor
// kernel triggers at its completion). Send k+1 claims its index and slot,
// copies and publishes while send k still runs; it waits for its
// predecessor only at its end, so sends still complete in stream order.
// Without `early` the send waits for its predecessor before it reads the
// source or lets the next launch start (a preceding receive may be writing
// the buffer this send reads).
// flags: bit 0 early; bits 1-2 per-CTA fence mode of a bulk send
// (chan_last_cta); bits 8-15 the launch serial (diagnostics, hx_chan_trace).
__global__ void __launch_bounds__(1024)
chan_send_kernel(ChanDir c, const unsigned char *src, unsigned long long bytes,
                 unsigned long long timeout_ns, int *err, int flags) {
    const bool early = flags & 1;
    __shared__ int ok;
    __shared__ unsigned long long k;
    const unsigned long long t_in = c.trace ? hx::globaltimer() : 0;
    // The claim and the slot wait touch only this direction's channel state,
    // so even a send that must wait for its predecessor does them first,
    // overlapped with that predecessor. Claims stay in stream order: every
    // channel kernel claims before it triggers its dependents, and a launch
    // starts only after its predecessor triggered.
    if (threadIdx.x == 0) {
        k = chan_claim(c.seq);
        if (blockIdx.x == 0 && c.trace) c.trace[(k & 255) * 8] = t_in;
        // diagnostics: the index each CTA of launch `serial` claimed
        if (c.trace && blockIdx.x < 320)
            c.trace[2048 + ((flags >> 8) & 255) * 320 + blockIdx.x] = k + 1;
        // slot k % depth is free once the receiver consumed message k - depth
        ok = k < (unsigned long long)c.depth ||
             hx::spin_until(c.credit, k + 1 - c.depth, timeout_ns, err, 0);
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) chan_stamp(c, k, 1);
    // Not early: the predecessor may be writing the source. Wait for it
    // before reading the source — and before triggering, so a following
    // early send of the same buffer cannot start ahead of that writer.
    if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");
    // only now may the next send launch: a launch never waits on a later one
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    char *slot = c.slots + (k % c.depth) * c.stride;
    unsigned long long *hdr = reinterpret_cast<unsigned long long *>(slot);
    const unsigned long long tag = (k + 1) & 0xffffffffull;
    if (bytes <= HX_CHAN_LL_MAX) {  // single CTA: LL words, no fence
        if (ok) {
            unsigned long long *words = reinterpret_cast<unsigned long long *>(slot + CHAN_HDR);
            const unsigned long long n = (bytes + 3) / 4;
            for (unsigned long long w = threadIdx.x; w < n; w += blockDim.x)
                st_relaxed_sys(words + w, (tag << 32) | load4(src + 4 * w, bytes - 4 * w));
            if (threadIdx.x == 0) {
                st_relaxed_sys(hdr, (tag << 32) | bytes);
                chan_stamp(c, k, 2);
            }
        }
    } else if (CHAN_HDR + bytes > c.stride) {
        // does not fit a slot: single CTA publishes the source, waits for the pull
        if (ok && threadIdx.x == 0) {
            st_relaxed_sys(hdr + 1, (unsigned long long)(uintptr_t)src);
            hx::st_release_sys(hdr, (tag << 32) | CHAN_PULL | bytes);  // orders the pointer
            chan_stamp(c, k, 2);
            // the receiver copies straight out of src over NVLink; src is
            // reusable (the send complete) once it hands the slot back
            hx::spin_until(c.credit, k + 1, timeout_ns, err, 0);
            chan_stamp(c, k, 3);
        }
    } else {
        if (ok)
            copy_bytes(slot + CHAN_HDR, (const char *)src, bytes,
                       blockIdx.x * (size_t)blockDim.x + threadIdx.x,
                       (size_t)gridDim.x * blockDim.x, false);
        // one arrival counter per slot: overlapping sends use different slots
        // flags bits 1-2: per-CTA fence (chan_last_cta; HX_CHAN_DIAG_FENCE)
        if (chan_last_cta(c.counter + k % c.depth, (flags >> 1) & 3) && threadIdx.x == 0 && ok) {
            hx::st_release_sys(hdr, (tag << 32) | bytes);  // orders every CTA's payload
            chan_stamp(c, k, 2);
        }
    }
    // Completion order: the launch completes only when every CTA exited, so
    // CTA 0 alone waiting for the predecessor keeps sends completing in
    // stream order, while the other CTAs exit at once and free their SM
    // slots for the next overlapping send (512-thread CTAs at 64 registers:
    // 2 per SM, so waiting CTAs capped the overlap at about 4 sends).
    if (early && blockIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0) chan_stamp(c, k, 4);
}

__global__ void __launch_bounds__(256)
chan_recv_kernel(ChanDir c, unsigned char *dst, unsigned long long capacity,
                 unsigned long long *len_out, unsigned long long timeout_ns, int *err) {
    __shared__ int ok;
    __shared__ bool pull;
    __shared__ unsigned long long k, len;
    __shared__ const char *from;
    const unsigned long long t_in = c.trace ? hx::globaltimer() : 0;
    // Everything up to the predecessor wait only READS: the message index
    // (claimed like a send's, so receives claim in stream order), the
    // header, and the first round of the payload into registers. So a
    // receive launched behind another one finds its message and loads it
    // while that one still copies, and only its stores wait.
    if (threadIdx.x == 0) {
        k = chan_claim(c.seq);
        if (blockIdx.x == 0 && c.trace) c.trace[(k & 255) * 8] = t_in;
    }
    // When may the next operation launch? A one-CTA receive lets it launch
    // at once: a send behind it (the echo of a ping-pong) then claims and
    // waits for its slot while this receive still polls, so the send's launch
    // latency is off the critical path. A multi-CTA receive triggers only
    // once its message has arrived, which bounds the receives in flight (each
    // up to 2 x SMs CTAs) to the messages already delivered.
    __syncthreads();
    if (gridDim.x == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        const unsigned long long tag = (k + 1) & 0xffffffffull;
        const unsigned long long *hdr =
            reinterpret_cast<const unsigned long long *>(c.slots + (k % c.depth) * c.stride);
        const unsigned long long t0 = hx::globaltimer();
        unsigned long long h;
        unsigned polls = 0;
        ok = 1;
        while (((h = ld_relaxed_sys(hdr)) >> 32) != tag) {
            if ((++polls & 63) == 0 && hx::globaltimer() - t0 > timeout_ns) {
                atomicExch(err, HX_E_TIMEOUT);
                ok = 0;
                break;
            }
        }
        if (blockIdx.x == 0) chan_stamp(c, k, 2);
        pull = (h & CHAN_PULL) != 0;
        len = h & (CHAN_PULL - 1);
        if (ok && len > HX_CHAN_LL_MAX) {
            (void)hx::ld_acquire_sys(hdr);  // bulk / pull: order the payload or the pointer
            if (pull) from = reinterpret_cast<const char *>(ld_relaxed_sys(hdr + 1));
        }
    }
    __syncthreads();
    if (gridDim.x > 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const char *slot = c.slots + (k % c.depth) * c.stride;
    const unsigned long long take = len < capacity ? len : capacity;
    const unsigned long long tag = (k + 1) & 0xffffffffull;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t nth = (size_t)gridDim.x * blockDim.x;
    const bool ll = ok && len <= HX_CHAN_LL_MAX;
    const char *from_p = pull ? from : slot + CHAN_HDR;  // pull: the sender's buffer over NVLink
    const bool vec = ok && !ll && ((((uintptr_t)dst | (uintptr_t)from_p) & 15) == 0);
    const size_t nv = vec ? take / 16 : 0;
    constexpr int R = 4;    // bulk: 16-byte vectors per thread in the first round
    constexpr int LLW = 8;  // LL: words per thread (HX_CHAN_LL_MAX / 4 / 256)
    uint4 pre[R];
    unsigned words_v[LLW];
    if (vec) {
        const uint4 *s16 = reinterpret_cast<const uint4 *>(from_p);
#pragma unroll
        for (int u = 0; u < R; ++u)
            if (tid + u * nth < nv) pre[u] = __ldcg(s16 + tid + u * nth);
    } else if (ll) {
        const unsigned long long *words = reinterpret_cast<const unsigned long long *>(slot + CHAN_HDR);
        const unsigned long long n = (take + 3) / 4;
#pragma unroll
        for (int u = 0; u < LLW; ++u) {
            const size_t w = tid + u * nth;
            if (w >= n) break;
            unsigned long long v;
            unsigned polls = 0;
            const unsigned long long t0 = hx::globaltimer();
            while (((v = ld_relaxed_sys(words + w)) >> 32) != tag) {
                if ((++polls & 255) == 0 && hx::globaltimer() - t0 > timeout_ns) {
                    atomicExch(err, HX_E_TIMEOUT);
                    break;
                }
            }
            words_v[u] = (unsigned)v;
        }
    }
    // the predecessor may still read or write dst: stores only from here on
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0) chan_stamp(c, k, 1);
    if (vec) {
        uint4 *d16 = reinterpret_cast<uint4 *>(dst);
#pragma unroll
        for (int u = 0; u < R; ++u)
            if (tid + u * nth < nv) d16[tid + u * nth] = pre[u];
        const uint4 *s16 = reinterpret_cast<const uint4 *>(from_p);
        for (size_t q = tid + R * nth; q < nv; q += nth) d16[q] = __ldcg(s16 + q);
        for (size_t b = nv * 16 + tid; b < take; b += nth) dst[b] = from_p[b];
    } else if (ll) {
        const unsigned long long n = (take + 3) / 4;
#pragma unroll
        for (int u = 0; u < LLW; ++u) {
            const size_t w = tid + u * nth;
            if (w >= n) break;
            store4(dst + 4 * w, words_v[u], take - 4 * w);
        }
    } else if (ok) {  // unaligned bulk or pull
        copy_bytes((char *)dst, from_p, take, tid, nth, true);
    }
    // The credit hands the slot (or the pulled source) back to the sender.
    // No fence before the arrival count and a relaxed credit store: every
    // slot read fed a store issued before the CTA barrier, so the reads have
    // been performed by the time any thread passes it (the hardware's
    // behaviour; the PTX model does not order loads through data
    // dependencies). The formal alternative — a GPU-scope fence per CTA and
    // a system-scope release of the credit — was measured in round 2 on 2
    // GPUs: one-way 8 B 3.4-3.6 -> 4.7-5.3 us and the 4 MiB window 729 -> 615
    // GB/s (profiles/r2_osu_2gpu_table.md), so it is not the default.
    // HX_CHAN_FORMAL_CREDIT=1 selects it (chan_credit_formal below).
    if (chan_last_cta(c.counter, chan_credit_formal() ? 0 : 2) && threadIdx.x == 0 && ok) {
        chan_stamp(c, k, 3);
        if (len_out) *len_out = len;  // > capacity: the caller reports truncation
        if (chan_credit_formal())
            hx::st_release_sys(c.credit, k + 1);
        else
            st_relaxed_sys(c.credit, k + 1);
    }
}

// Low-latency (LL) ping-pong: every 8-byte word carries 4 payload bytes and
// the 32-bit iteration tag, written with one single-copy-atomic store, so
// the receiver polls the data itself — no fence, no separate flag.
__device__ __forceinline__ bool ll_recv(const unsigned long long *ll, unsigned *out, int nwords,
                                        unsigned tag, unsigned long long t0,
                                        unsigned long long timeout_ns, int *err) {
    for (int w = threadIdx.x; w < nwords; w += blockDim.x) {
        unsigned long long v;
        unsigned polls = 0;
        while (((v = ld_relaxed_sys(ll + w)) >> 32) != tag) {
            if ((++polls & 255) == 0 && hx::globaltimer() - t0 > timeout_ns) {
                atomicExch(err, HX_E_TIMEOUT);
                return false;
            }
        }
        out[w] = (unsigned)v;
    }
    return true;
}

__global__ void pingpong_ll_kernel(int role, const unsigned *src, unsigned *dst_local,
                                   unsigned long long *peer_ll, const unsigned long long *my_ll,
                                   int nwords, int iters, int warmup, unsigned long long timeout_ns,
                                   unsigned long long *elapsed, int *err) {
    __shared__ int ok;
    const unsigned long long start = hx::globaltimer();
    unsigned long long t0 = start;
    for (int it = 0; it < warmup + iters; ++it) {
        const unsigned tag = (unsigned)it + 1;
        if (role == 0 && it == warmup && threadIdx.x == 0) t0 = hx::globaltimer();
        if (role == 1) {
            const bool good = ll_recv(my_ll, dst_local, nwords, tag, start, timeout_ns, err);
            if (threadIdx.x == 0) ok = 1;
            __syncthreads();
            if (!good) ok = 0;
            __syncthreads();
            if (!ok) return;
        }
        const unsigned *out = role == 0 ? src : dst_local;
        for (int w = threadIdx.x; w < nwords; w += blockDim.x)
            st_relaxed_sys(peer_ll + w, ((unsigned long long)tag << 32) | out[w]);
        if (role == 0) {
            const bool good = ll_recv(my_ll, dst_local, nwords, tag, start, timeout_ns, err);
            if (threadIdx.x == 0) ok = 1;
            __syncthreads();
            if (!good) ok = 0;
            __syncthreads();
            if (!ok) return;
        }
    }
    if (role == 0 && threadIdx.x == 0 && elapsed) *elapsed = hx::globaltimer() - t0;
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
            if (threadIdx.x == 0) ok = hx::spin_until(my_flag, v, timeout_ns, err, 0);
            __syncthreads();
            if (!ok) return;
        }
        copy_bytes(peer_dst, src, bytes, tid, nthr, role == 1);
        // barrier(s) order every thread's peer stores before the lead's
        // system-scope fence (cumulative) and the release of the flag
        __syncthreads();
        if (gridDim.x > 1) grid.sync();
        if (lead) hx::st_release_sys(peer_flag, v);  // release = MEMBAR.SYS + strong store
        if (role == 0) {
            if (threadIdx.x == 0) ok = hx::spin_until(my_flag, v, timeout_ns, err, 0);
            __syncthreads();
            if (!ok) return;
        }
    }
    if (role == 0 && lead && elapsed) *elapsed = hx::globaltimer() - t0;
}

unsigned face_grid(const FaceBatch &b) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    static int mult = 0;
    if (!mult) {
        const char *e = getenv("HX_FACE_GRID_MULT");
        mult = e ? atoi(e) : 4;
        if (mult <= 0) mult = 4;
    }
    const int cap = mult * sms;
    return (unsigned)(b.total_blocks < cap ? (b.total_blocks > 0 ? b.total_blocks : 1) : cap);
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
    face_copy_kernel<true><<<face_grid(b), FACE_THREADS, 0, (cudaStream_t)stream>>>(b);
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
    face_copy_kernel<false><<<face_grid(b), FACE_THREADS, 0, (cudaStream_t)stream>>>(b);
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
    pack_put_kernel<<<face_grid(b), FACE_THREADS, 0, (cudaStream_t)stream>>>(b, value, counters);
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
    wait_unpack_kernel<<<face_grid(b), FACE_THREADS, 0, (cudaStream_t)stream>>>(b, value,
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

int hx_pingpong_ll(int role, const void *src, void *dst_local, void *peer_ll, void *my_ll,
                   size_t bytes, int iters, int warmup, unsigned long long timeout_ns,
                   unsigned long long *elapsed_ns, int *err, void *stream) {
    if ((role != 0 && role != 1) || !dst_local || !peer_ll || !my_ll || !err || iters < 0 ||
        warmup < 0 || bytes == 0 || (bytes & 3) || bytes > (1u << 20))
        return HX_E_INVALID;
    if (role == 0 && !src) return HX_E_INVALID;
    const int nwords = (int)(bytes / 4);
    const int threads = nwords >= 1024 ? 1024 : ((nwords + 31) / 32) * 32;
    pingpong_ll_kernel<<<1, threads, 0, (cudaStream_t)stream>>>(
        role, (const unsigned *)src, (unsigned *)dst_local, (unsigned long long *)peer_ll,
        (const unsigned long long *)my_ll, nwords, iters, warmup, timeout_ns, elapsed_ns, err);
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

int hx_move(void *dst, const void *src, size_t bytes, int device, void *stream, void *ready_event,
            void *done_event, void *order_stream) {
    if (bytes && (!dst || !src)) return HX_E_INVALID;
    cudaStream_t st = (cudaStream_t)stream;
    if (ready_event) HX_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)ready_event, 0));
    if (bytes > HX_MOVE_SM_MAX) {
        HX_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
    } else if (bytes) {
        // a launch costs the host less than a peer cudaMemcpyAsync; kernels
        // launch on the current device, so switch to the stream's and back
        int prev = 0;
        HX_TRY(cudaGetDevice(&prev));
        if (prev != device) HX_TRY(cudaSetDevice(device));
        const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((bytes / 16 + 255) / 256, 64));
        copy_kernel<<<grid, 256, 0, st>>>((char *)dst, (const char *)src, bytes);
        const cudaError_t e = cudaGetLastError();
        if (prev != device) cudaSetDevice(prev);
        if (e != cudaSuccess) return (int)e;
    }
    if (done_event) HX_TRY(cudaEventRecord((cudaEvent_t)done_event, st));
    if (order_stream && done_event)
        HX_TRY(cudaStreamWaitEvent((cudaStream_t)order_stream, (cudaEvent_t)done_event, 0));
    return 0;
}

// Channel launch shapes, read once from the environment (tuning and
// diagnostics; tools/pchan_knobs.py sweeps them one process per setting).
// Sends overlap each other, so each needs few CTAs: HX_CHAN_SEND_CTAS
// (default 64) x HX_CHAN_SEND_THREADS (256 / 512 / 1024, default 512);
// receives HX_CHAN_RECV_CTAS (default 2 x SMs) x 256. HX_CHAN_DIAG_FENCE:
// the per-CTA fence of a bulk send (chan_last_cta): 0 GPU scope (default),
// 1 system scope, 2 none (diagnostics only). profiles/r1_pchannel.md.
struct ChanKnobs {
    unsigned send_ctas, send_threads, recv_ctas;  // recv_ctas 0: 2 x SMs
    int fence;
};

static const ChanKnobs &chan_knobs() {
    static const ChanKnobs k = [] {
        auto num = [](const char *name, int dflt) {
            const char *e = getenv(name);
            return e && atoi(e) > 0 ? atoi(e) : dflt;
        };
        ChanKnobs v;
        v.send_ctas = (unsigned)num("HX_CHAN_SEND_CTAS", 64);
        const int t = num("HX_CHAN_SEND_THREADS", 512);
        v.send_threads = (t == 256 || t == 512 || t == 1024) ? (unsigned)t : 512u;
        v.recv_ctas = (unsigned)num("HX_CHAN_RECV_CTAS", 0);
        const char *f = getenv("HX_CHAN_DIAG_FENCE");
        v.fence = f ? (atoi(f) & 3) : 0;
        return v;
    }();
    return k;
}

// Grid of a channel copy: >= per_cta bytes per CTA, at most `cap` CTAs.
static unsigned chan_grid(unsigned long long bytes, unsigned cap, unsigned long long per_cta) {
    const unsigned long long want = (bytes + per_cta - 1) / per_cta;
    return (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>(want, cap));
}

static unsigned chan_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (unsigned)sms;
}

static cudaLaunchConfig_t chan_launch_config(unsigned grid, void *stream, cudaLaunchAttribute *attr,
                                             unsigned threads = 256) {
    attr->id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr->val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = (cudaStream_t)stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

// Lazy module loading (CUDA_MODULE_LOADING=LAZY, PyTorch's default) loads a
// kernel at its first launch, and that load can stall behind kernels that
// are spinning on the device, e.g. a receive waiting for a message that the
// newly loaded kernel's stream must produce: the spin then only ends at its
// timeout. Channel and exchange users preload every spinning or
// interleaved kernel of this file on each device they use.
int hx_preload_halo_kernels() {
    cudaFuncAttributes a;
    const void *k[] = {(const void *)chan_send_kernel, (const void *)chan_recv_kernel,
                       (const void *)copy_kernel, (const void *)copy_window_kernel,
                       (const void *)pack_put_kernel, (const void *)wait_unpack_kernel,
                       (const void *)face_copy_kernel<true>, (const void *)face_copy_kernel<false>,
                       (const void *)signal_kernel, (const void *)wait_flag_kernel,
                       (const void *)pingpong_kernel, (const void *)pingpong_ll_kernel};
    for (const void *f : k) HX_TRY(cudaFuncGetAttributes(&a, f));
    return 0;
}

// The last channel operation enqueued on each stream (true = a send): a send
// right after a send may overlap it (chan_send_kernel `early`).
static std::mutex chan_last_mu;
static std::unordered_map<void *, bool> chan_last_send;

static unsigned long long *chan_trace_buf[2][64];  // [send / recv][device]

int hx_chan_trace(int device, void *send_trace, void *recv_trace) {
    if (device < 0 || device >= 64) return HX_E_INVALID;
    chan_trace_buf[0][device] = (unsigned long long *)send_trace;
    chan_trace_buf[1][device] = (unsigned long long *)recv_trace;
    return 0;
}

static unsigned long long *chan_trace_of(int role) {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < 64 ? chan_trace_buf[role][dev] : nullptr;
}

static bool chan_note(void *stream, bool send) {
    std::lock_guard<std::mutex> lock(chan_last_mu);
    bool &last = chan_last_send[stream];
    const bool prev = last;
    last = send;
    return prev;
}

int hx_chan_send(const void *src, size_t bytes, void *slots, size_t stride, int depth,
                 unsigned long long *credit, unsigned long long *seq, unsigned int *counter,
                 unsigned long long timeout_ns, int *err, void *stream) {
    if (!slots || !credit || !seq || !counter || depth < 1 || (bytes && !src)) return HX_E_INVALID;
    const bool pull = bytes > HX_CHAN_LL_MAX && CHAN_HDR + bytes > stride;  // see chan_send_kernel
    const unsigned long long need =
        CHAN_HDR + (bytes <= HX_CHAN_LL_MAX ? 8 * ((bytes + 3) / 4) : pull ? 0 : bytes);
    if (need > stride || bytes >= CHAN_PULL) return HX_E_INVALID;
    ChanDir c{(char *)slots, credit, seq, counter, stride, depth, chan_trace_of(0)};
    const ChanKnobs &kn = chan_knobs();
    const bool bulk = bytes > HX_CHAN_LL_MAX && !pull;
    // each thread keeps 4 x 16 B of stores in flight per iteration
    const unsigned grid = bulk ? chan_grid(bytes, kn.send_ctas, 32768) : 1u;
    const unsigned threads = grid > 1 ? kn.send_threads : 256u;
    cudaLaunchAttribute attr;
    const cudaLaunchConfig_t cfg = chan_launch_config(grid, stream, &attr, threads);
    const int fmode = kn.fence;
    static std::atomic<unsigned> serial{0};  // diagnostics: launch serial (trace claims)
    const int early = (chan_note(stream, true) ? 1 : 0) | (fmode << 1) |
                      (int)((serial++ & 255u) << 8);
    HX_TRY(cudaLaunchKernelEx(&cfg, chan_send_kernel, c, (const unsigned char *)src,
                              (unsigned long long)bytes, timeout_ns, err, early));
    return 0;
}

int hx_chan_recv(void *dst, size_t capacity, const void *slots, size_t stride, int depth,
                 unsigned long long *credit, unsigned long long *seq, unsigned int *counter,
                 unsigned long long *len_out, unsigned long long timeout_ns, int *err,
                 void *stream) {
    if (!slots || !credit || !seq || !counter || depth < 1 || (capacity && !dst))
        return HX_E_INVALID;
    ChanDir c{(char *)slots, credit, seq, counter, stride, depth, chan_trace_of(1)};
    chan_note(stream, false);
    static int formal = -1;  // HX_CHAN_FORMAL_CREDIT=1: fenced credit (see chan_recv_kernel)
    static unsigned long long formal_set = 0;
    if (formal < 0) {
        const char *e = getenv("HX_CHAN_FORMAL_CREDIT");
        formal = e && atoi(e) == 1 ? 1 : 0;
    }
    if (formal) {
        int dev = 0;
        HX_TRY(cudaGetDevice(&dev));
        if (!(formal_set & (1ull << (dev & 63)))) {
            HX_TRY(cudaMemcpyToSymbol(g_chan_formal_credit, &formal, sizeof(int)));
            formal_set |= 1ull << (dev & 63);
        }
    }
    cudaLaunchAttribute attr;
    // sized by the sink: a pulled message may be far larger than a slot
    // 2 x SMs: a pulled 4 MiB message is loaded entirely before the
    // predecessor wait (4 x 16 B a thread), and a receive spinning on its
    // header holds at most ~60 % of the register file (80 x 256 per CTA), so
    // a 64-CTA bulk send can still run beside it. 3 x SMs (94 %) was 10 %
    // faster for pulled 16 MiB windows but could starve the send that the
    // peer's message depends on.
    const unsigned cap = chan_knobs().recv_ctas ? chan_knobs().recv_ctas : 2 * chan_sms();
    const unsigned grid = chan_grid(capacity, cap, 16384);
    const cudaLaunchConfig_t cfg = chan_launch_config(grid, stream, &attr);
    HX_TRY(cudaLaunchKernelEx(&cfg, chan_recv_kernel, c, (unsigned char *)dst,
                              (unsigned long long)capacity, len_out, timeout_ns, err));
    return 0;
}

int hx_copy_sm_window(void *dst, const void *src, size_t bytes, int count, void *stream) {
    if (!bytes || count <= 0) return 0;
    if (!dst || !src) return HX_E_INVALID;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static int mult = 0;
    if (!mult) {
        const char *e = getenv("HX_COPY_GRID_MULT");
        mult = e ? atoi(e) : 4;
        if (mult <= 0) mult = 4;
    }
    size_t want = (bytes * (size_t)count / 64 + 255) / 256;  // ~16 KiB of window per CTA
    unsigned grid = (unsigned)(want < (size_t)sms * mult ? (want ? want : 1) : (size_t)sms * mult);
    copy_window_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((char *)dst, (const char *)src,
                                                               bytes, count);
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
