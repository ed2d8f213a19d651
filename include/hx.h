/* hx.h — C ABI of the B200 halo-exchange library (libhx.so).
 *
 * The reference (charmlet, /root/reference/pkg/src/charmlet = cl/) has no
 * native plugin layer: its hot path is numpy over a simulated device space.
 * This ABI sits UNDER the reference's unchanged Python API (DeviceSpace,
 * Worker.tag_send/tag_recv, Channel, devmsg, _BlockCore, run_jacobi) and is
 * bound with ctypes. Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *  - Every function returns int: 0 = success, >0 = cudaError_t, <0 = HX_E_*.
 *  - Pointers are device pointers on the CURRENT device (hx_set_device),
 *    except where a peer-mapped pointer is explicitly allowed.
 *  - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Fields are padded fp64 blocks in C order (bx+2, by+2, bz+2): z is
 *    contiguous, x slowest (cl/jacobi3d.py:131-134). Interior indices run
 *    1..bx, 1..by, 1..bz; ghosts are planes 0 and n+1.
 *  - Direction codes d: 0=-x 1=+x 2=-y 3=+y 4=-z 5=+z (cl/jacobi3d.py:35).
 *  - The library never frees memory it did not allocate.
 */
#ifndef HX_H
#define HX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HX_ABI_VERSION 1

#define HX_E_INVALID   (-1) /* bad argument (shape, direction, null pointer) */
#define HX_E_TIMEOUT   (-2) /* a device-side flag wait exceeded its deadline */
#define HX_E_NODRIVER  (-3) /* a driver entry point could not be resolved    */
#define HX_E_TMA       (-4) /* cuTensorMapEncodeTiled rejected the layout     */

/* ------------------------------------------------------------ runtime ---- */
int hx_abi_version(void);
const char *hx_error_string(int code);
int hx_device_count(int *n);
int hx_set_device(int dev);
int hx_get_device(int *dev);
int hx_sm_count(int dev, int *n);
int hx_device_synchronize(void);
int hx_stream_create(void **stream);                 /* non-blocking stream on current dev */
int hx_stream_destroy(void *stream);
int hx_stream_synchronize(void *stream);
int hx_event_create(void **ev, int timing);          /* timing=0: cudaEventDisableTiming */
int hx_event_destroy(void *ev);
int hx_event_record(void *ev, void *stream);
int hx_event_query(void *ev);                        /* 0 done, 1 pending, else error */
int hx_event_synchronize(void *ev);
int hx_event_elapsed_ms(void *start, void *stop, float *ms);
int hx_stream_wait_event(void *stream, void *ev);
/* Device memory owned by the caller of hx_malloc (IPC arenas only; fields and
 * staging are torch allocations). */
int hx_malloc(void **ptr, size_t bytes);
int hx_free(void *ptr);
int hx_malloc_host(void **ptr, size_t bytes);        /* pinned host memory */
int hx_free_host(void *ptr);

/* ---------------------------------------------------- peer access / IPC --
 * Replaces the reference's in-process byte copies between workers
 * (cl/devicesim.py:72-86 read_wire/write_wire) with NVLink P2P mappings. */
int hx_can_access_peer(int dev, int peer, int *ok);
int hx_enable_peer(int dev, int peer);               /* idempotent */
/* handle_out: 64-byte cudaIpcMemHandle_t of the allocation holding ptr;
 * offset_out: ptr - allocation base. */
int hx_ipc_get(void *ptr, void *handle_out, size_t *offset_out);
int hx_ipc_open(const void *handle, void **base_out); /* cached per handle */
int hx_ipc_close(void *base);
/* The allocation holding ptr: base address and size (cuMemGetAddressRange);
 * lets a sender cache one exported IPC handle per allocation. */
int hx_alloc_range(const void *ptr, void **base_out, size_t *size_out);

/* --------------------------------------------------------------- copies --
 * cl/devicesim.py:197-224 (host_to_device / device_to_host /
 * device_to_device) and the transport's device payload moves
 * (cl/transport.py:284-289, 430-432, 459-463). */
int hx_memcpy(void *dst, const void *src, size_t bytes, void *stream);          /* cudaMemcpyDefault */
int hx_memcpy_peer(void *dst, int dst_dev, const void *src, int src_dev, size_t bytes, void *stream);
int hx_copy_sm(void *dst, const void *src, size_t bytes, void *stream);         /* SM-issued (peer ok) */
/* The transport's per-message device move in one call (Worker._d2d, the
 * B200 replacement of the PULL/PAYLOAD byte moves at cl/transport.py:284-289,
 * 430-432, 449-465): stream waits for ready_event (if given), copies bytes
 * (<= HX_MOVE_SM_MAX as an SM kernel on `device`, the stream's GPU; larger
 * on the copy engines), records done_event, and makes order_stream (if
 * given) wait for it. The current device is left unchanged. */
#define HX_MOVE_SM_MAX (64u << 10)
int hx_move(void *dst, const void *src, size_t bytes, int device, void *stream,
            void *ready_event, void *done_event, void *order_stream);
/* count back-to-back copies src -> dst in one launch (OSU window). */
int hx_copy_sm_window(void *dst, const void *src, size_t bytes, int count, void *stream);
int hx_fill_f64(double *dst, size_t n, double value, void *stream);

/* ------------------------------------------------------------- stencil ---
 * _BlockCore.update, cl/jacobi3d.py:165-173:
 *   nxt[i,j,k] = (((((cur[i-1,j,k] + cur[i+1,j,k]) + cur[i,j-1,k])
 *                 + cur[i,j+1,k]) + cur[i,j,k-1]) + cur[i,j,k+1]) / 6.0
 * for every interior cell; ghosts of nxt untouched. Bit-exact with the
 * reference (IEEE adds in this order, correctly rounded division).
 * res (nullable): device uint64 holding the bit pattern of a non-negative
 * double; the kernel atomically maxes max|nxt - cur| into it
 * (cl/jacobi3d.py:197-198). The caller zeroes it. */
int hx_stencil(const double *cur, double *nxt, int bx, int by, int bz,
               unsigned long long *res, void *stream);
/* Sub-box of the interior, 1-based inclusive-exclusive [i0,i1)x[j0,j1)x[k0,k1);
 * used for the interior/boundary-shell overlap split. */
int hx_stencil_box(const double *cur, double *nxt, int bx, int by, int bz,
                   int i0, int i1, int j0, int j1, int k0, int k1,
                   unsigned long long *res, void *stream);
/* Force a kernel variant (testing / profiling): 0 auto, 1 TMA pipeline
 * (auto when the padded row pitch is a multiple of 16 bytes, i.e. even bz),
 * 2 generic, 3 flattened slab (auto for boxes thinner than 8 rows or 16
 * columns — the overlap split's boundary shell), 4 single z column with
 * aligned quad loads (auto for one-column boxes), 5 row-pair TMA pipeline
 * (the TMA kernel through four parity-class tensor maps with 2-row / 2-plane
 * strides; auto for odd bz, whose row pitch a plain tensor map cannot
 * describe).
 * Returns the previous one. */
int hx_stencil_set_variant(int variant);
int hx_stencil_last_variant(void);
/* Tuning knob for the TMA pipeline: x planes per CTA work item (0 = auto). */
int hx_stencil_set_chunk(int planes);
/* Self-check of the stencil's division by 6 (RN(1/6) product + one FMA
 * correction, Markstein) against the library's correctly rounded __ddiv_rn
 * over n device doubles; *mismatches (device u64, caller-zeroed) += count. */
int hx_div6_check(const double *in, size_t n, unsigned long long *mismatches, void *stream);

/* Hot-wall / Dirichlet initialisation of one padded block
 * (cl/jacobi3d.py:135-138, 186-188): every cell = background, interior =
 * fill, and if hot_wall the whole x=0 ghost plane = hot. */
int hx_init_block(double *field, int bx, int by, int bz, int hot_wall,
                  double hot, double background, double fill, void *stream);

/* -------------------------------------------------------- pack / unpack --
 * _BlockCore.pack (cl/jacobi3d.py:157-158): dst = C-order copy of interior
 * plane 1 (d even) or n (d odd) of axis d/2 over the other two interior
 * axes (face_shape, cl/jacobi3d.py:141-144). dst may be a peer-mapped
 * pointer (fused pack + NVLink put). */
int hx_pack(const double *field, int bx, int by, int bz, int d, double *dst, void *stream);
/* _BlockCore.unpack_all for one direction (cl/jacobi3d.py:160-163): write
 * a face into ghost plane 0 (d even) or n+1 (d odd). src may be peer-mapped. */
int hx_unpack(double *field, int bx, int by, int bz, int d, const double *src, void *stream);

/* Fused multi-face pack + put + signal (Channel.send of every halo face,
 * cl/jacobi3d.py:250-253, without per-message metadata): for each d in
 * dir_mask, pack face d into dst[d] (typically the neighbour's receive slot,
 * peer-mapped) and, once every CTA of the (persistent) grid has stored,
 * publish every *flag[d] = value with system-scope release. counters: device
 * uint32 scratch (6 reserved, counters[0] used), zero-initialised once; the
 * kernel returns it to zero. flag[d] may be NULL (no signal). */
int hx_pack_put(const double *field, int bx, int by, int bz, int dir_mask,
                double *const dst[6], unsigned long long *const flag[6],
                unsigned long long value, unsigned int *counters, void *stream);
/* Fused wait + multi-face unpack (Channel.recv completions + unpack_all,
 * cl/jacobi3d.py:254-257, 277): for each d in dir_mask wait until
 * *flag[d] >= value (system-scope acquire; bounded by timeout_ns, then
 * *err = HX_E_TIMEOUT and the face is skipped), then unpack src[d]. */
int hx_wait_unpack(double *field, int bx, int by, int bz, int dir_mask,
                   const double *const src[6], unsigned long long *const flag[6],
                   unsigned long long value, unsigned long long timeout_ns, int *err,
                   void *stream);

/* Fused boundary sweep + halo put (HaloJacobi exchange="fused"; replaces
 * the pack -> Channel.send -> recv -> unpack_all chain of Block.run,
 * cl/jacobi3d.py:246-257, and the boundary part of _BlockCore.update,
 * cl/jacobi3d.py:165-173). Each CTA first waits until every non-NULL
 * wait_flag[d] >= wait_value (the neighbours' boundary of the previous
 * iteration is in cur's ghost planes and they are done reading ours; bounded
 * by timeout_ns, then *err = HX_E_TIMEOUT). It then relaxes the nbox
 * (<= 6) boxes `boxes[6*q .. 6*q+5]` = i0,i1,j0,j1,k0,k1 of cur into nxt
 * and stores every cell lying on the plane facing d (i == 1 for d = 0,
 * i == bx for d = 1, ... k == bz for d = 5) also into remote[d], the
 * neighbour's nxt array of the same padded shape, at its ghost cell. After
 * the last CTA's stores are visible system-wide it release-stores
 * signal_value into every non-NULL signal_flag[d] (skipped if *err != 0).
 * counter: one zero-initialised uint32 that the kernel returns to zero.
 * res: optional max|nxt-cur| accumulator, as for hx_stencil.
 * step (nullable): a device uint64 iteration counter; when given, both
 * values are offsets from *step and the last CTA advances *step by one, so
 * a step sequence can be captured once in a CUDA graph and replayed. */
int hx_shell_put(const double *cur, double *nxt, int bx, int by, int bz, int nbox,
                 const int *boxes, double *const remote[6],
                 unsigned long long *const wait_flag[6], unsigned long long wait_value,
                 unsigned long long *const signal_flag[6], unsigned long long signal_value,
                 unsigned int *counter, unsigned long long timeout_ns, int *err,
                 unsigned long long *res, unsigned long long *step, void *stream);
/* hx_shell_put with the z faces through contiguous slots: zin[0] / zin[1]
 * hold the -z / +z neighbour's face of the previous step, packed [i-1][j-1]
 * (bx x by doubles, the arena slots the prime exchange also fills); they
 * replace the ghost column. zout[0] / zout[1] receive this step's -z / +z
 * face in the neighbour's arena (its slot for the next step), replacing
 * 8-byte NVLink stores into its ghost column, one per 12 KB row. Either
 * pointer pair may be NULL (ghost columns, as hx_shell_put). */
int hx_shell_put_z(const double *cur, double *nxt, int bx, int by, int bz, int nbox,
                   const int *boxes, double *const remote[6],
                   unsigned long long *const wait_flag[6], unsigned long long wait_value,
                   unsigned long long *const signal_flag[6], unsigned long long signal_value,
                   unsigned int *counter, unsigned long long timeout_ns, int *err,
                   unsigned long long *res, unsigned long long *step,
                   const double *const zin[2], double *const zout[2], void *stream);

/* Small blocks: `iters` fused iterations of one block in ONE launch
 * (persistent CTAs, grid barriers between iterations). Per iteration: wait
 * for every non-NULL wait_flag[d] >= it + 1, relax the whole block
 * field[parity] -> field[parity ^ 1], store each neighbour-facing cell also
 * into peer[2 d + (parity ^ 1)] (the neighbour's next buffer, same padded
 * shape) at its ghost plane, then release signal_flag[d] = it + 2; parity
 * flips every iteration, it = it0 .. it0 + iters - 1. z faces go through
 * the arena slots as in hx_shell_put_z: for an iteration of parity q (it & 1),
 * zin[2 q + h] is our slot read on side h (-z, +z) and zout[2 q + h] the
 * neighbour's slot written (its parity q ^ 1 slot); NULL: ghost columns. The same
 * flag protocol as hx_shell_put, so runs may alternate with fused steps. barrier: two
 * zero-initialised uint32 (count, generation). max_ctas caps the grid (every
 * CTA must be co-resident with the other blocks' kernels on this GPU). Blocks
 * above 2^31 cells: HX_E_INVALID. */
int hx_persist_run(double *const field[2], double *const peer[12], int bx, int by, int bz,
                   int parity, unsigned long long it0, int iters,
                   unsigned long long *const wait_flag[6], unsigned long long *const signal_flag[6],
                   const double *const zin[4], double *const zout[4], unsigned *barrier,
                   int max_ctas, unsigned long long timeout_ns, int *err, void *stream);

/* The fused exchange's interior sweep when the block has z neighbours: the
 * box must span whole z rows (k0 = 1, k1 = bz + 1). Tiles holding k = 1
 * (zflag[0], -z) or k = bz (zflag[1], +z) wait for that flag >= *zstep + 1,
 * read the ghost column from zin[h] (packed [i-1][j-1], bx x by) and copy the
 * face cells into zout[h] (the neighbour's slot for the next step); the rest
 * is hx_stencil_box. The z faces then cost no extra HBM traffic (the sweep
 * stages those rows anyway). One launch: the edge tiles take the z work at
 * run time. Not TMA-eligible, another box, or both z neighbours with
 * bz <= 64 (one tile would hold both faces): HX_E_INVALID. */
int hx_stencil_box_z(const double *cur, double *nxt, int bx, int by, int bz, int i0, int i1,
                     int j0, int j1, int k0, int k1, unsigned long long *res,
                     const unsigned long long *const zflag[2], const unsigned long long *zstep,
                     const double *const zin[2], double *const zout[2],
                     unsigned long long timeout_ns, int *err, void *stream);
/* After a step's interior sweep and boundary kernel (stream-ordered behind
 * both): release flag[h] = *step + 2 into the z neighbours' arenas (skipped
 * if *err != 0), then *step += 1. */
int hx_zsignal(unsigned long long *const flag[2], unsigned long long *step, const int *err,
               void *stream);

/* The fused step as ONE sweep of the whole block (replaces the boundary
 * kernel hx_shell_put_z and the interior sweep, cl/jacobi3d.py:157-173's
 * pack / send / recv / unpack / update for every face): tiles that hold a
 * face wait for that neighbour's flag[d] >= *step + 1; x / y face cells are
 * also stored into peer_nxt[d] (neighbour d's next field, same padded shape)
 * at its ghost plane / row, whose own ghost planes / rows the neighbour has
 * stored into ours; z faces go through the slots as in hx_stencil_box_z.
 * flag[d] NULL: no neighbour d. Needs a TMA-describable block and no tile
 * holding both faces of one axis (bz > 64 with both z neighbours, by > 32
 * with both y neighbours, bx >= 2 with both x neighbours): else
 * HX_E_INVALID. signal / counter non-NULL: the sweep's last edge tile
 * releases signal[d] = *step + 2 into the neighbours' arenas and advances
 * *step itself (counter: a zero-initialised uint32, re-armed by the kernel),
 * so the step is ONE launch; NULL: follow with hx_exchange_signal. */
int hx_stencil_exchange(const double *cur, double *nxt, int bx, int by, int bz,
                        unsigned long long *res, const unsigned long long *const flag[6],
                        double *const peer_nxt[6], unsigned long long *step,
                        const double *const zin[2], double *const zout[2],
                        unsigned long long *const signal[6], unsigned *counter,
                        unsigned long long timeout_ns, int *err, void *stream);
/* Host only: how many work items of hx_stencil_exchange's sweep hold a face
 * of the sides in mask (bit d: neighbour d) — the count its last edge tile
 * waits for. Exposed so it can be checked without a GPU. */
int hx_exchange_edge_items(int bx, int by, int bz, int mask, unsigned *out);
/* Release flag[d] = *step + 2 (non-NULL entries, six threads in parallel;
 * skipped if *err != 0), then *step += 1. hx_zsignal is its z-only form. */
int hx_exchange_signal(unsigned long long *const flag[6], unsigned long long *step,
                       const int *err, void *stream);

/* --------------------------------------------------- persistent channel --
 * The Channel API's metadata-free stream (cl/channels.py:33-102; paper
 * §3.2.2) in its pre-registered device form. One direction is a ring of
 * `depth` slots (`stride` bytes apart) in the receiver's HBM and a credit
 * counter on the sender; a slot holds a 128-byte header block — tag k+1 in the high
 * 32 bits and the length in the low 32, i.e. the arrival flag and the length
 * in one word — then the payload. Payloads up to HX_CHAN_LL_MAX bytes go as
 * LL words (8-byte stores of 4 data bytes + the tag: no fences, the receiver
 * polls the data), payloads that fit a slot as a bulk copy into it
 * published by a release store of the header (the sender may run `depth`
 * messages ahead); larger ones are pulled: the header publishes the source
 * address and the receive copies straight out of the sender's buffer over
 * NVLink (one copy, any size below 2^31 bytes), the send completing when
 * the slot comes back. The message index is device state (*seq, one per endpoint,
 * advanced by each launch; a ticket word: index << 32 | CTAs of the launch
 * arrived), so send/recv sequences can be captured in CUDA graphs.
 * Consecutive sends on one stream overlap on the GPU (each claims its index
 * and slot, then lets the next launch start) and still complete in stream
 * order; a send after a receive on the same stream claims early but reads
 * its source only after that receive completed. A receive claims, polls its
 * header and loads the first round of its payload before waiting for its
 * predecessor; only its stores wait.
 *   send k: wait until *credit >= k+1-depth (slot k % depth free), write
 *           the payload into the slot (a peer-mapped pointer) and its header.
 *   recv k: wait for the header tag, copy min(len, capacity) bytes into dst,
 *           write len to *len_out (nullable; len > capacity = truncated) and
 *           store *credit = k+1 (a peer-mapped pointer).
 * stride must hold HX_CHAN_HDR + 8 * ceil(min(bytes, HX_CHAN_LL_MAX) / 4) (LL
 * messages); the payload starts HX_CHAN_HDR bytes into the slot.
 * counter: zero-initialised uint32s — `depth` of them for a send (one per
 * slot), one for a receive — per endpoint and direction. Waits
 * are bounded by timeout_ns (then *err = HX_E_TIMEOUT). */
#define HX_CHAN_LL_MAX 8192u
#define HX_CHAN_HDR 128u
int hx_chan_send(const void *src, size_t bytes, void *slots, size_t stride, int depth,
                 unsigned long long *credit, unsigned long long *seq, unsigned int *counter,
                 unsigned long long timeout_ns, int *err, void *stream);
int hx_chan_recv(void *dst, size_t capacity, const void *slots, size_t stride, int depth,
                 unsigned long long *credit, unsigned long long *seq, unsigned int *counter,
                 unsigned long long *len_out, unsigned long long timeout_ns, int *err,
                 void *stream);
/* Load every spinning channel / exchange kernel on the current device now.
 * Under lazy module loading (PyTorch's default) a kernel's first launch can
 * stall behind kernels spinning on the device until their waits time out;
 * PersistentChannel and HaloJacobi call this for each device they use.
 * Kernels a caller interleaves with channel operations should likewise run
 * once beforehand (or set CUDA_MODULE_LOADING=EAGER). */
int hx_preload(void);

/* Diagnostics: channel operations launched on `device` afterwards write
 * %globaltimer stamps — 8 per message, message k at [(k % 256) * 8] — into
 * send_trace / recv_trace (device buffers of 2048 uint64 — send: 2048 +
 * 256 * 320, the claimed index + 1 per CTA per launch serial — or null).
 * send: entry, index+slot claimed, published, pulled (pull mode), done;
 * recv: entry, predecessor done, header seen, copied. */
int hx_chan_trace(int device, void *send_trace, void *recv_trace);

/* ---------------------------------------------------------------- flags --
 * Persistent-channel completion words (the Channel API's per-direction
 * counter, cl/channels.py:75-99, carried as a 64-bit flag value). */
int hx_signal(unsigned long long *flag, unsigned long long value, void *stream);
int hx_wait_flag(unsigned long long *flag, unsigned long long value,
                 unsigned long long timeout_ns, int *err, void *stream);
int hx_read_u64(const unsigned long long *dev_ptr, unsigned long long *host_out); /* sync read */

/* ------------------------------------------------- device-level ping-pong --
 * OSU latency inner loop (cl/bench.py:170-194) with kernel-issued NVLink
 * stores: iters round trips of `bytes` between two GPUs. Leader (role 0)
 * writes payload into peer_buf then flag; follower (role 1) echoes.
 * Both kernels must run concurrently on DIFFERENT GPUs. elapsed_ns (device
 * uint64, leader only) receives %globaltimer delta over the timed iters. */
int hx_pingpong(int role, const void *src, void *peer_dst, size_t bytes,
                unsigned long long *my_flag, unsigned long long *peer_flag,
                int iters, int warmup, unsigned long long timeout_ns,
                unsigned long long *elapsed_ns, int *err, void *stream);

/* Low-latency variant for small messages (bytes % 4 == 0, <= 1 MiB): each
 * 8-byte word of the LL buffers carries 4 payload bytes plus the 32-bit
 * iteration tag and is written with one single-copy-atomic store, so the
 * receiver polls the data itself (no fence, no separate flag). peer_ll /
 * my_ll: 2*bytes each (my_ll zeroed by the caller); dst_local: bytes. One
 * CTA per GPU; both roles must run concurrently on different GPUs. */
int hx_pingpong_ll(int role, const void *src, void *dst_local, void *peer_ll, void *my_ll,
                   size_t bytes, int iters, int warmup, unsigned long long timeout_ns,
                   unsigned long long *elapsed_ns, int *err, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HX_H */
