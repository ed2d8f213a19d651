// Jacobi3D 6-neighbour relaxation for sm_100a.
//
// Reference: _BlockCore.update, cl/jacobi3d.py:165-173 (and the sequential
// oracle's identical sweep + residual, 192-198):
//   nxt[i,j,k] = (((((c[i-1,j,k] + c[i+1,j,k]) + c[i,j-1,k]) + c[i,j+1,k])
//                 + c[i,j,k-1]) + c[i,j,k+1]) / 6.0
// The adds are issued in exactly this order (no contraction) and the
// quotient is the IEEE correctly rounded t / 6.0, so results are
// bit-identical to numpy. Ghost cells of nxt are never written.
//
// Division by 6 (div6): y = RN(1/6) = 0x3FC5555555555555 has relative error
// 2^-54, so q = RN(t*y) is within 1 ulp of t/6; with the exact FMA remainder
// r = t - 6q, Markstein's theorem gives RN(q + r*y) = RN(t/6) for every t
// whose intermediate values stay normal. Zero, subnormal-range, huge and
// non-finite sums take the library __ddiv_rn. 3 FP64 ops instead of the
// generic divide's ~20 + branch; hx_div6_check verifies it on device.
//
// Primary kernel (HBM-bound, 16 algorithmic bytes per cell): a 2.5-D
// streaming sweep. Each CTA owns a TY x TZ tile of the (j,k) plane and
// marches along x (the slowest axis) over a chunk of planes. Every padded
// plane tile (TY+2) x (TZ+4) is fetched once by a TMA bulk-tensor load into
// an NS-stage shared-memory ring guarded by mbarriers; each input cell
// crosses HBM once (tile halos are served by L2 — ncu: 59.0 GB DRAM for
// 58.0 GB algorithmic at 1536^3). Each thread keeps its columns' x-1 and x
// values in registers (register marching), so per cell it reads only the
// x+1 centre and the four y/z neighbours from shared memory. Outputs are
// stored from registers with coalesced stores through pointers advanced
// one plane per step. The residual max|nxt-cur| uses the register-resident
// centre and is reduced per warp into one atomicMax on the uint64 bit
// pattern (valid for non-negative doubles), skipped when already covered.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "hx_internal.cuh"

namespace {

constexpr int TY = 32;        // tile rows (j)
constexpr int TZ = 64;        // tile columns (k): two 32-lane halves
constexpr int NSTAGE = 4;     // shared-memory ring depth (planes)
constexpr int MIN_CTAS = 3;   // resident CTAs per SM (smem: 3 x 74 KB)
constexpr int THREADS = 256;  // 8 warps; warp w owns rows w, w+8, w+16, w+24
constexpr int NWARP = THREADS / 32;
constexpr int ROWS = TY / NWARP;
constexpr int PTS = ROWS * 2;  // cells per thread per plane
// A box row is TZ+2 doubles (the tile plus its z halo). TMA only accepts
// 16-byte aligned row starts, so when the tile's first input column kb-1 is
// odd (sub-box sweeps starting at an even k) the load starts one element
// earlier and the box is TZ+4 wide (kshift = 1). Full sweeps use TZ+2.
constexpr int BOX_Y = TY + 2, BOX_Z_MAX = TZ + 4;
constexpr unsigned STAGE_STRIDE = (BOX_Y * BOX_Z_MAX * sizeof(double) + 127) / 128 * 128;
constexpr size_t SMEM_BYTES = (size_t)NSTAGE * STAGE_STRIDE + NSTAGE * sizeof(uint64_t);

int g_variant = 0;  // 0 auto, 1 TMA, 2 generic
int g_last_variant = 0;
int g_chunk = 0;  // planes per CTA work item, 0 = auto
int g_num_sms = 0;
int g_l2promo = -1;  // CUtensorMapL2promotion for the plane loads; -1 = default

constexpr double RCP6 = 0.16666666666666666;  // RN(1/6) = 0x3FC5555555555555

// +0.0 is exact on the fast path (q = r = +0) and is by far the most common
// sum early in a hot-wall run, so it must not take the slow path; -0.0
// would come out as +0.0 and goes to the library division.
__device__ __forceinline__ bool div6_fast_ok(double t) {
    const double a = fabs(t);
    return (a >= 0x1p-960 && a <= 0x1p1020) || __double_as_longlong(t) == 0;
}

__device__ __forceinline__ double div6_fast(double t) {
    const double q = __dmul_rn(t, RCP6);
    const double r = __fma_rn(-6.0, q, t);
    return __fma_rn(r, RCP6, q);
}

__device__ __noinline__ double div6_slow(double t) {
    return t == 0.0 ? t : __ddiv_rn(t, 6.0);
}

__device__ __forceinline__ double div6(double t) {
    return div6_fast_ok(t) ? div6_fast(t) : div6_slow(t);
}

__device__ __forceinline__ double sum6(double xm, double xp, double ym, double yp, double zm,
                                       double zp) {
    double t = __dadd_rn(xm, xp);
    t = __dadd_rn(t, ym);
    t = __dadd_rn(t, yp);
    t = __dadd_rn(t, zm);
    return __dadd_rn(t, zp);
}

// Residual max|nxt - cur| into one uint64 word (for non-negative doubles the
// bit-pattern order is the value order). Warp shuffle reduction, then lane 0
// of each warp updates the word: no CTA barrier, so the warps of a short TMA
// work item retire independently. Every warp of a sweep targets the same
// word, and an unconditional atomic would serialise at its L2 slice; the max
// only grows, so lane 0 skips the atomic when the (possibly stale, hence
// lower) current value already covers its w.
// The residual max|nxt - cur| is kept as the bit pattern of |nxt - cur|
// (sign cleared): for non-negative doubles the unsigned integer order is
// the numeric order, so the max is an integer max on the integer pipe (no
// FP64 min/max next to the stencil's own FP64 work), and a NaN difference
// — whose pattern sorts above +inf — propagates like numpy's max
// (cl/jacobi3d.py:197-198).
__device__ __forceinline__ unsigned long long abs_diff_bits(double v, double c) {
    return (unsigned long long)__double_as_longlong(__dsub_rn(v, c)) & 0x7fffffffffffffffull;
}

__device__ __forceinline__ void warp_max_to_global(unsigned long long worst,
                                                   unsigned long long *res) {
    for (int o = 16; o > 0; o >>= 1) worst = max(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    if ((tid & 31) == 0 && worst > 0ull) {
        if (worst > *(volatile unsigned long long *)res) atomicMax(res, worst);
    }
}

// The fused exchange's z faces produced by the interior sweep (round 2,
// the default): the tiles that hold k = 1 (with a -z neighbour) or k = bz
// (+z) wait for that neighbour's flag (>= *step + 1), take the ghost column
// from its slot (packed [i-1][j-1], staged beside each plane by cp.async)
// and copy the face cells into the neighbour's slot. The z faces cost no
// extra DRAM work: the sweep opens those pages anyway, where a separate
// z-face kernel pays a page activation per cell (profiles/r2_zface_dram.md).
struct ZEdge {
    const unsigned long long *flag[2];  // our flags from the -z / +z neighbour (null: none)
    const unsigned long long *step;     // device step counter (hx_zsignal advances it)
    const double *zin[2];               // this step's slots
    double *zout[2];                    // the neighbours' slots for the next step
    unsigned long long timeout_ns;
    int *err;
    // x / y faces in the sweep too (hx_stencil_exchange; null: none): our flags
    // from the -x +x -y +y neighbours, and for each the element distance from
    // a cell of our next field to the matching ghost cell in its next field
    const unsigned long long *xyflag[4];
    long long xydelta[4];
    int bx;  // block extent in x (the +x face is plane bx)
    // in-kernel release (hx_stencil_exchange): the last edge tile to finish
    // releases sig[d] = *step + 2 into the neighbours' arenas and advances
    // *step. Only edge tiles read the ghosts the neighbours overwrite next or
    // store into theirs, so they alone decide when the step is done for the
    // neighbours. edge_counter: zero-initialised, re-armed by the last tile.
    unsigned long long *sig[6];
    unsigned *edge_counter;  // null: release with hx_exchange_signal instead
    unsigned edge_items;
};

// One x plane of a tile from two staged planes: P0 holds plane q (y/z
// neighbours), PP plane q+1; xm/x0 carry planes q-1 and q in registers and
// are advanced. Stores the live cells of plane q and folds their residual.
// ROWSTEP: staged distance between a thread's rows r and r + NWARP; ylo /
// yhi: distance from a cell to its y-1 / y+1 neighbour in P0.
// ZS (1: the tile holds k = 1 with a -z neighbour, 2: k = bz with a +z
// neighbour): on the edge lane (zedge, half zc) the z ghost is zg[row] and
// the cell is also copied to zdst[row] — the z faces produced by the
// interior sweep (ZEdge below).
// CONSEC: the thread's ROWS rows are consecutive (ROWSTEP = one staged
// row), so an inner row's y neighbours are the rows above / below it that
// the thread already holds in registers (x0: plane q's values): 2 of the 8
// y loads per row pair stay in shared memory instead of 8 — 28 shared loads
// per 8 cells instead of 40 (less shared-memory traffic per cell).
template <bool RES, int ROWSTEP, int ZS = 0, bool CONSEC = false, bool XY = false>
__device__ __forceinline__ void relax_plane(const double *P0, const double *PP, int soff, int ylo,
                                            int yhi, double (&xm)[PTS], double (&x0)[PTS],
                                            double *out, int bz, unsigned live,
                                            unsigned long long &worst, bool zedge = false,
                                            int zc = 0, const double *zg = nullptr,
                                            double *zdst = nullptr, const ZEdge *Zx = nullptr,
                                            int P = 0, int jrow = 0, int by = 0) {
    double v[PTS];
    bool fast = true;
    double prev[2] = {0.0, 0.0};  // CONSEC: row t - 1's plane-q values
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
        const int t = p >> 1, c = p & 1;
        const int o = soff + t * ROWSTEP + 32 * c;
        const double xp = PP[o];
        double ym, yp;
        if (CONSEC) {
            ym = t > 0 ? prev[c] : P0[o - ylo];
            yp = t < ROWS - 1 ? x0[p + 2 < PTS ? p + 2 : p] : P0[o + yhi];
            prev[c] = x0[p];
        } else {
            ym = P0[o - ylo];
            yp = P0[o + yhi];
        }
        double zm = P0[o - 1], zp = P0[o + 1];
        // ZS: the edge lane's z ghost comes from the neighbour's slot (zg,
        // staged by cp.async), not from the field's ghost column
        if (ZS == 1 && zedge && c == zc) zm = zg[t];
        if (ZS == 2 && zedge && c == zc) zp = zg[t];
        v[p] = sum6(xm[p], xp, ym, yp, zm, zp);
        xm[p] = x0[p];
        x0[p] = xp;
        fast &= div6_fast_ok(v[p]);
    }
    if (fast) {
#pragma unroll
        for (int p = 0; p < PTS; ++p) v[p] = div6_fast(v[p]);
    } else {
#pragma unroll
        for (int p = 0; p < PTS; ++p) v[p] = div6(v[p]);
    }
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
        if (live & (1u << p)) {
            constexpr int RS = CONSEC ? 1 : NWARP;  // rows between a thread's rows
            out[(size_t)((p >> 1) * RS) * (bz + 2) + 32 * (p & 1)] = v[p];
            if (RES) worst = max(worst, abs_diff_bits(v[p], xm[p]));
            if (ZS && zedge && (p & 1) == zc) zdst[(p >> 1) * RS] = v[p];  // face -> slot
            if (XY) {  // x / y faces: also into the neighbour's ghost plane / row
                double *const o = out + (size_t)((p >> 1) * RS) * (bz + 2) + 32 * (p & 1);
                if (Zx->xyflag[0] && P == 1) o[Zx->xydelta[0]] = v[p];
                if (Zx->xyflag[1] && P == Zx->bx) o[Zx->xydelta[1]] = v[p];
                const int j = jrow + (p >> 1);
                if (Zx->xyflag[2] && j == 1) o[Zx->xydelta[2]] = v[p];
                if (Zx->xyflag[3] && j == by) o[Zx->xydelta[3]] = v[p];
            }
        }
    }
}

// Work item = (tile j, tile k, x chunk) in grouped order: groups of `grows`
// tile rows; inside a group all tiles of chunk c, then chunk c+1, ...
// Concurrent CTAs therefore cover adjacent tiles of the same few planes
// (tile halos hit L2) and chunk c+1 of a tile starts while chunk c's last
// planes are still in L2.
struct Item {
    int jb, kb, ib, nplanes;
};

__device__ __forceinline__ Item work_item(int j0, int k0, int i0, int i1, int ntj, int ntk,
                                          int chunk, int nchunks, int grows) {
    const int items_g = grows * ntk * nchunks;
    const int g = blockIdx.x / items_g;
    const int rem = blockIdx.x - g * items_g;
    const int tiles_g = min(grows, ntj - g * grows) * ntk;
    const int c = rem / tiles_g;
    const int t = rem - c * tiles_g;
    Item it;
    it.jb = j0 + (g * grows + t / ntk) * TY;
    it.kb = k0 + (t % ntk) * TZ;
    it.ib = i0 + c * chunk;
    it.nplanes = min(it.ib + chunk, i1) - it.ib + 2;  // padded planes ib-1 .. ie
    return it;
}

// ------------------------------------------------------- TMA pipeline ----
// Work item = (tile j, tile k, x chunk). Box in interior coordinates:
// [i0,i1) x [j0,j1) x [k0,k1).

// One work item (tile x chunk) of the TMA sweep. ZE: the tile holds k = 1
// with a -z neighbour (zlo) or k = bz with a +z neighbour (zhi) and does the
// z-edge work as well; the kernel picks the instance per tile, so the plain
// tiles of a z-edge launch run the plain code (and registers).
template <bool RES, int BOX_Z, int ZS, bool XY = false>  // ZS: bit 0 the tile holds k = 1 (-z), bit 1 k = bz (+z)
__device__ __forceinline__ void tma_tile(const CUtensorMap &map, double *__restrict__ nxt, int by,
                                         int bz, int j1, int k1, int klive, const Item &it,
                                         unsigned long long *res, const ZEdge &Z,
                                         unsigned xym = 0) {  // XY: sides -x +x -y +y (bits)
    constexpr bool ZE = ZS != 0, zlo = (ZS & 1) != 0, zhi = (ZS & 2) != 0;
    constexpr unsigned STAGE_BYTES = BOX_Y * BOX_Z * sizeof(double);
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + NSTAGE * STAGE_STRIDE);

    const int jb = it.jb, kb = it.kb, ib = it.ib, nplanes = it.nplanes;
    const int kshift = BOX_Z == TZ + 2 ? 0 : (kb - 1) & 1;  // 16-byte aligned TMA rows
    const int kload = kb - 1 - kshift;

    if ((ZE || XY) && threadIdx.x == 0) {
        const unsigned long long want = *(volatile const unsigned long long *)Z.step + 1;
        if (zlo) hx::spin_until(Z.flag[0], want, Z.timeout_ns, Z.err);
        if (zhi) hx::spin_until(Z.flag[1], want, Z.timeout_ns, Z.err);
        if (XY)
            for (int d = 0; d < 4; ++d)
                if ((xym >> d) & 1u) hx::spin_until(Z.xyflag[d], want, Z.timeout_ns, Z.err);
        // the ghost planes / rows were stored by the peers (generic proxy, made
        // visible by the acquires): order them before this tile's TMA reads,
        // as the boundary kernel does
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        hx::prefetch_tmap(&map);
        for (int s = 0; s < NSTAGE; ++s) hx::mbar_init(&bar[s], 1);
        hx::fence_mbar_init();
        const int pre = min(NSTAGE, nplanes);
        for (int p = 0; p < pre; ++p) {
            hx::mbar_expect_tx(&bar[p], STAGE_BYTES);
            hx::tma_load_3d(smem + p * STAGE_STRIDE, &map, kload, jb - 1, ib - 1 + p, &bar[p]);
        }
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row0 = ROWS * warp;  // warp w owns the consecutive tile rows 4w .. 4w + 3
    // shared-memory offset (doubles) of this thread's first cell centre
    const int soff = (row0 + 1) * BOX_Z + lane + 1 + kshift;
    const size_t plane = (size_t)(by + 2) * (bz + 2);
    double *out = nxt + ((size_t)ib * (by + 2) + (jb + row0)) * (bz + 2) + kb + lane;
    unsigned live = 0;  // bit p: cell p of this thread is inside the box
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
        const int r = row0 + (p >> 1), kk = lane + 32 * (p & 1);
        if (jb + r < j1 && kb + kk < k1 && kb + kk >= klive) live |= 1u << p;
    }

    // ZE (ZS = 1: the tile holds k = 1, ZS = 2: k = bz): the neighbour's slot
    // supplies the edge column's z ghost. Warp 0 stages slot rows jb .. jb+31
    // of each relaxed plane with cp.async into the unused tail of that
    // plane's stage (a 66-wide box leaves 608 bytes), two planes ahead; the
    // per-plane CTA barrier publishes them. The TMA never writes the tail,
    // so no proxy fence is needed, and nothing stays in registers.
    constexpr unsigned ZG_OFF = BOX_Y * BOX_Z * sizeof(double);
    static_assert(!ZE || ZG_OFF + TY * sizeof(double) <= STAGE_STRIDE, "stage tail too small");
    const int zcol = ZS == 1 ? 0 : bz - kb;  // the edge column within the tile
    const bool zedge = ZE && lane == (zcol & 31);
    const int zc = ZE ? zcol >> 5 : 0;
    auto zstage = [&](int q) {  // one cp.async group per call (empty past the last plane)
        if (!ZE || warp != 0) return;
        if (q <= nplanes - 2 && jb + lane <= by) {
            const double *src = Z.zin[ZS == 2] + (size_t)(ib - 2 + q) * by + (jb + lane - 1);
            const uint32_t dst = hx::smem_addr(smem + (q % NSTAGE) * STAGE_STRIDE + ZG_OFF) + 8 * lane;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto zwait = [&]() {  // all groups but the newest have landed
        if (ZE && warp == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");
    };
    // the edge lane's face cells also go to the neighbour's slot (offset of
    // this thread's first row there; the pointer is formed at the store)
    unsigned zoff = (unsigned)((ib - 1) * by + (jb + row0 - 1));

    zstage(1);
    zstage(2);

    double xm[PTS], x0[PTS];
    unsigned long long worst = 0;
    int nan_seen = 0;
    {
        const double *s0 = reinterpret_cast<const double *>(smem);
        const double *s1 = reinterpret_cast<const double *>(smem + STAGE_STRIDE);
        hx::mbar_wait(&bar[0], 0);
        hx::mbar_wait(&bar[1], 0);
        zwait();  // plane 1's slot rows (the barrier below publishes them)
#pragma unroll
        for (int p = 0; p < PTS; ++p) {
            const int o = soff + (p >> 1) * BOX_Z + 32 * (p & 1);
            xm[p] = s0[o];
            x0[p] = s1[o];
            nan_seen |= (xm[p] != xm[p]) | (x0[p] != x0[p]);
        }
    }
    // Plane 0 must be in registers before its stage is recycled. A plain
    // bar.sync does not wait for this warp's outstanding shared loads (it
    // blocks lazily), and the refill below is an async-proxy write: under SM
    // contention the TMA can land before a queued LDS is served. The
    // barrier's predicate consumes every loaded value, so each warp's loads
    // have completed when it arrives. (Inside the loop the loaded values feed
    // the stores that precede the barrier, which orders them the same way.)
    (void)__syncthreads_or(nan_seen);
    if (threadIdx.x == 0 && NSTAGE < nplanes) {
        hx::mbar_expect_tx(&bar[0], STAGE_BYTES);
        hx::tma_load_3d(smem, &map, kload, jb - 1, ib - 1 + NSTAGE, &bar[0]);
    }
    int s_c = 1 % NSTAGE;  // stage holding plane q
    for (int q = 1; q <= nplanes - 2; ++q) {
        const int s_n = s_c + 1 == NSTAGE ? 0 : s_c + 1;  // stage holding plane q+1
        hx::mbar_wait(&bar[s_n], ((q + 1) / NSTAGE) & 1);
        relax_plane<RES, BOX_Z, ZS, true, XY>(
            reinterpret_cast<const double *>(smem + s_c * STAGE_STRIDE),
            reinterpret_cast<const double *>(smem + s_n * STAGE_STRIDE), soff, BOX_Z, BOX_Z, xm,
            x0, out, bz, live, worst, zedge, zc,
            reinterpret_cast<const double *>(smem + s_c * STAGE_STRIDE + ZG_OFF) + row0,
            ZE ? Z.zout[ZS == 2] + zoff : nullptr, &Z, ib - 1 + q, jb + row0, by);
        out += plane;
        if (ZE) {
            zoff += by;
            zstage(q + 2);
            zwait();  // plane q + 1's slot rows, published by the barrier below
        }
        __syncthreads();  // all warps are done with stage s_c (plane q)
        if (threadIdx.x == 0) {
            const int p = q + NSTAGE;
            if (p < nplanes) {
                hx::mbar_expect_tx(&bar[s_c], STAGE_BYTES);
                hx::tma_load_3d(smem + s_c * STAGE_STRIDE, &map, kload, jb - 1, ib - 1 + p,
                                &bar[s_c]);
            }
        }
        s_c = s_n;
    }
    if (RES) warp_max_to_global(worst, res);
    if constexpr (ZE || XY) {
        if (Z.edge_counter) {  // the last edge tile releases the step to the neighbours
            __shared__ int last;
            __syncthreads();  // this tile's local and peer stores are issued
            if (threadIdx.x == 0) {
                __threadfence();  // GPU scope per tile; the releases below are cumulative
                last = atomicAdd(Z.edge_counter, 1u) + 1u == Z.edge_items;
                if (last) *Z.edge_counter = 0u;  // re-arm (launches on one stream are ordered)
            }
            __syncthreads();
            if (last) {
                const unsigned long long v = *(volatile const unsigned long long *)Z.step + 2;
                const bool healthy = !Z.err || *(volatile const int *)Z.err == 0;
                if (threadIdx.x < 6 && Z.sig[threadIdx.x] && healthy)
                    hx::st_release_sys(Z.sig[threadIdx.x], v);
                __syncthreads();  // every releasing thread has read *step
                if (threadIdx.x == 0) *(volatile unsigned long long *)Z.step = v - 1;
            }
        }
    }
}

template <bool RES, int BOX_Z, bool ZE>
__global__ void __launch_bounds__(THREADS, MIN_CTAS)
stencil_tma_kernel(const __grid_constant__ CUtensorMap map, double *__restrict__ nxt, int by,
                   int bz, int i0, int i1, int j0, int j1, int k0, int k1, int klive, int ntj,
                   int ntk, int chunk, int nchunks, int grows, unsigned long long *res, ZEdge Z) {
    const Item it = work_item(j0, k0, i0, i1, ntj, ntk, chunk, nchunks, grows);
    if constexpr (ZE) {  // z-edge tile: holds k = 1 (-z neighbour) / k = bz (+z neighbour)
        const bool zlo = Z.flag[0] && it.kb <= 1 && 1 < it.kb + TZ && k0 <= 1;
        const bool zhi = Z.flag[1] && it.kb <= bz && bz < it.kb + TZ && bz < k1;
        // x / y faces this tile holds (the box is the whole block then)
        const unsigned xym = (Z.xyflag[0] && it.ib == 1 ? 1u : 0u) |
                             (Z.xyflag[1] && it.ib + it.nplanes - 3 == Z.bx ? 2u : 0u) |
                             (Z.xyflag[2] && it.jb == 1 ? 4u : 0u) |
                             (Z.xyflag[3] && it.jb <= by && by < it.jb + TY ? 8u : 0u);
        // one instance per side, so a tile keeps one side's state (the host
        // rejects blocks where one tile would hold both z faces, bz <= TZ)
        if (zlo && zhi) {
            if (threadIdx.x == 0 && Z.err) atomicExch(Z.err, HX_E_INVALID);
            return;
        }
        if (xym) {
            if (zlo) return tma_tile<RES, BOX_Z, 1, true>(map, nxt, by, bz, j1, k1, klive, it, res, Z, xym);
            if (zhi) return tma_tile<RES, BOX_Z, 2, true>(map, nxt, by, bz, j1, k1, klive, it, res, Z, xym);
            return tma_tile<RES, BOX_Z, 0, true>(map, nxt, by, bz, j1, k1, klive, it, res, Z, xym);
        }
        if (zlo) return tma_tile<RES, BOX_Z, 1>(map, nxt, by, bz, j1, k1, klive, it, res, Z);
        if (zhi) return tma_tile<RES, BOX_Z, 2>(map, nxt, by, bz, j1, k1, klive, it, res, Z);
    }
    tma_tile<RES, BOX_Z, 0>(map, nxt, by, bz, j1, k1, klive, it, res, Z);
}

// ------------------------------------------- row-pair tensor pipeline ----
// The TMA kernel for row pitches a plain 3-D tensor map cannot describe
// (bz + 2 doubles, not a multiple of 16 bytes: odd bz). The array is viewed
// through four tensor maps, one per (row parity a, plane parity b) class:
//   element (i, j, k) = base + (i>>1) 2 plane + (j>>1) 2 pz + [k + a pz + b plane]
// with strides 2 pz and 2 plane doubles (16-byte multiples for any parity)
// and the bracket as the dim-0 coordinate (dim-0 extent a pz + b plane + pz,
// so past-the-row columns read as out-of-bounds zeros, never past the array).
// Every row of a class starts with the same alignment, so one box per class
// (17 rows x 68 doubles, started one element early when the row start is
// odd) stages the tile's even or odd rows: two tensor loads per plane.
// Measured (tools/prof_stencil.py): 1536^2 x 1535 at 0.999 and 1535^3 at
// 0.997 of the HBM roofline (the generic kernel: 0.58; staging rows with
// 34 separate bulk copies per plane: 0.64, TMA-request bound).
constexpr int PW = TZ + 4;   // box width in doubles (66 needed + alignment shift, 544 B)
constexpr int PH = BOX_Y / 2;  // 17 rows per parity box
constexpr int PREG = (PH * PW * (int)sizeof(double) + 127) / 128 * 128 / (int)sizeof(double);
constexpr unsigned PSTAGE = 2 * PREG * sizeof(double);
constexpr size_t PSMEM_BYTES = (size_t)NSTAGE * PSTAGE + NSTAGE * sizeof(uint64_t);

struct PairMaps {
    CUtensorMap m[4];  // index a + 2 b
};

template <bool RES>
__global__ void __launch_bounds__(THREADS, MIN_CTAS)
stencil_pair_kernel(const __grid_constant__ PairMaps maps, double *__restrict__ nxt, int by, int bz,
                    int i0, int i1, int j0, int j1, int k0, int k1, int ntj, int ntk, int chunk,
                    int nchunks, int grows, unsigned long long *res) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + NSTAGE * PSTAGE);
    const Item it = work_item(j0, k0, i0, i1, ntj, ntk, chunk, nchunks, grows);
    const int jb = it.jb, kb = it.kb, ib = it.ib, nplanes = it.nplanes;
    const long long pz = (long long)bz + 2, plane = (long long)(by + 2) * pz;
    // local row parity l (tile row R = l + 2m) -> global row class a_l
    const int a0 = (jb - 1) & 1, a1 = jb & 1;
    // staging shift of local-parity region l at padded plane P
    auto shift = [&](int l, int P) {
        return (int)(((long long)(kb - 1) + (l ? a1 : a0) * pz + (P & 1) * plane) & 1);
    };
    auto load_plane = [&](int p, int stage) {  // thread 0: both parity boxes of plane ib-1+p
        const int P = ib - 1 + p;
        hx::mbar_expect_tx(&bar[stage], (unsigned)(2 * PH * PW * sizeof(double)));
#pragma unroll
        for (int l = 0; l < 2; ++l) {
            const int a = l ? a1 : a0;
            const int c0 = (kb - 1) + (int)(a * pz + (P & 1) * plane) - shift(l, P);
            hx::tma_load_3d(smem + stage * PSTAGE + l * PREG * sizeof(double), &maps.m[a + 2 * (P & 1)],
                            c0, (jb - 1 + l) >> 1, P >> 1, &bar[stage]);
        }
    };
    if (threadIdx.x == 0) {
        for (int q = 0; q < 4; ++q) hx::prefetch_tmap(&maps.m[q]);
        for (int q = 0; q < NSTAGE; ++q) hx::mbar_init(&bar[q], 1);
        hx::fence_mbar_init();
        for (int p = 0; p < NSTAGE && p < nplanes; ++p) load_plane(p, p);
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // this thread's rows R = warp + 1 + 8m sit in region rc at row (R >> 1);
    // their y-1 / y+1 neighbours in the other region
    const int rc = (warp + 1) & 1;
    const int c_row = (warp + 1) >> 1, lo_row = warp >> 1, hi_row = (warp + 2) >> 1;
    const int soff = rc * PREG + c_row * PW + lane + 1;
    auto ylo = [&](int P) {
        return soff - ((1 - rc) * PREG + lo_row * PW + lane + 1) + shift(rc, P) - shift(1 - rc, P);
    };
    auto yhi = [&](int P) {
        return ((1 - rc) * PREG + hi_row * PW + lane + 1) - soff + shift(1 - rc, P) - shift(rc, P);
    };
    double *out = nxt + ((size_t)ib * (by + 2) + (jb + warp)) * (size_t)pz + kb + lane;
    unsigned live = 0;
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
        const int r = warp + (p >> 1) * NWARP, kk = lane + 32 * (p & 1);
        if (jb + r < j1 && kb + kk < k1) live |= 1u << p;
    }
    double xm[PTS], x0[PTS];
    unsigned long long worst = 0;
    int nan_seen = 0;
    {
        const double *s0 = reinterpret_cast<const double *>(smem) + shift(rc, ib - 1);
        const double *s1 = reinterpret_cast<const double *>(smem + PSTAGE) + shift(rc, ib);
        hx::mbar_wait(&bar[0], 0);
        hx::mbar_wait(&bar[1], 0);
#pragma unroll
        for (int p = 0; p < PTS; ++p) {
            const int o = soff + (p >> 1) * (NWARP / 2) * PW + 32 * (p & 1);
            xm[p] = s0[o];
            x0[p] = s1[o];
            nan_seen |= (xm[p] != xm[p]) | (x0[p] != x0[p]);
        }
    }
    (void)__syncthreads_or(nan_seen);  // consume before stage 0 is refilled (see the TMA kernel)
    if (threadIdx.x == 0 && NSTAGE < nplanes) load_plane(NSTAGE, 0);
    int s_c = 1;
    for (int q = 1; q <= nplanes - 2; ++q) {
        const int s_n = s_c + 1 == NSTAGE ? 0 : s_c + 1;
        hx::mbar_wait(&bar[s_n], ((q + 1) / NSTAGE) & 1);
        const int P = ib - 1 + q;
        relax_plane<RES, (NWARP / 2) * PW>(
            reinterpret_cast<const double *>(smem + s_c * PSTAGE) + shift(rc, P),
            reinterpret_cast<const double *>(smem + s_n * PSTAGE) + shift(rc, P + 1), soff, ylo(P),
            yhi(P), xm, x0, out, bz, live, worst);
        out += plane;
        __syncthreads();  // all warps are done with stage s_c (plane q)
        if (threadIdx.x == 0 && q + NSTAGE < nplanes) load_plane(q + NSTAGE, s_c);
        s_c = s_n;
    }
    if (RES) warp_max_to_global(worst, res);
}

// ----------------------------------------------------------- generic ----
// One thread per cell over a box; read-only cache for the neighbours. Used
// for odd z extents (TMA needs 16-byte strides) and thin boundary shells.
__global__ void __launch_bounds__(256)
stencil_generic_kernel(const double *__restrict__ cur, double *__restrict__ nxt, int by, int bz,
                       int i0, int j0, int j1, int k0, int k1, unsigned long long *res) {
    const hx::Geom g(by, bz);
    const int k = k0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int j = j0 + blockIdx.y * blockDim.y + threadIdx.y;
    const int i = i0 + blockIdx.z;
    unsigned long long worst = 0;
    if (k < k1 && j < j1) {
        const size_t c = g.at(i, j, k);
        const size_t sx = (size_t)g.py * g.pz, sy = g.pz;
        const double v = div6(sum6(__ldg(cur + c - sx), __ldg(cur + c + sx), __ldg(cur + c - sy),
                                   __ldg(cur + c + sy), __ldg(cur + c - 1), __ldg(cur + c + 1)));
        nxt[c] = v;
        if (res) worst = abs_diff_bits(v, __ldg(cur + c));
    }
    if (res) warp_max_to_global(worst, res);
}

// Device self-check of div6 against the library division.
__global__ void div6_check_kernel(const double *in, size_t n, unsigned long long *mismatch) {
    unsigned long long bad = 0;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
         q += (size_t)gridDim.x * blockDim.x) {
        const double t = in[q];
        const double a = div6(t), b = __ddiv_rn(t, 6.0);
        const bool same = (__double_as_longlong(a) == __double_as_longlong(b)) || (a != a && b != b);
        bad += !same;
    }
    if (bad) atomicAdd(mismatch, bad);
}

// ------------------------------------------------------------- init ------
__global__ void init_block_kernel(double *f, int bx, int by, int bz, int hot_wall, double hot,
                                  double background, double fill) {
    const hx::Geom g(by, bz);
    const size_t n = (size_t)(bx + 2) * g.py * g.pz;
    const size_t plane = (size_t)g.py * g.pz;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
         q += (size_t)gridDim.x * blockDim.x) {
        const long i = (long)(q / plane);
        const long rem = (long)(q % plane);
        const long j = rem / g.pz, k = rem % g.pz;
        double v = background;
        if (i >= 1 && i <= bx && j >= 1 && j <= by && k >= 1 && k <= bz) v = fill;
        if (hot_wall && i == 0) v = hot;
        f[q] = v;
    }
}

// ------------------------------------------- fused boundary sweep + put ---
// The halo exchange folded into the stencil that produces it (exchange
// "fused"): the boundary boxes of a block are relaxed here, and every cell
// that lies on a neighbour-facing plane is stored twice — into our nxt and,
// over NVLink, straight into the neighbour's nxt ghost plane, where its
// next sweep reads it. No pack, no staging slot, no unpack: the face bytes
// leave the SM once. One flag per direction orders everything: the
// neighbour's release of flag = it+1 (after its boundary sweep of it-1)
// says both "your ghost plane holds my boundary of it-1" and "I have
// finished reading the ghost plane you are about to overwrite".
struct ShellJob {
    int nbox;
    int box[6][6];          // i0,i1,j0,j1,k0,k1 (1-based, half-open)
    int rows[7];            // prefix row counts; a row runs along k (along j for a z column)
    double *remote[6];      // neighbour's nxt base (same padded shape), or null
    long long shift[6];     // our padded offset + shift[d] = its ghost cell
    int face[6];            // coordinate of our plane facing d (i/j/k by d/2)
    unsigned long long *wait[6];
    unsigned long long *signal[6];
    // z faces through contiguous slots (hx_shell_put_z): zin[h] holds the
    // -z (h = 0) / +z (h = 1) neighbour's face of the previous step, packed
    // [i-1][j-1] (bx x by), read instead of the ghost column; zout[h]
    // receives our face on that side in the neighbour's arena, instead of
    // 8-byte stores into its ghost column 12 KB apart
    const double *zin[2];
    double *zout[2];
};

__global__ void __launch_bounds__(256)
shell_put_kernel(const double *cur, double *__restrict__ nxt, int by, int bz,
                 ShellJob J, unsigned long long wait_value, unsigned long long signal_value,
                 unsigned *counter, unsigned long long timeout_ns, int *err,
                 unsigned long long *res, unsigned long long *step) {
    __shared__ int ok;
    __shared__ unsigned long long base;  // device step counter (graph replays), else 0
    if (threadIdx.x == 0) {
        base = step ? *(volatile unsigned long long *)step : 0ull;
        ok = 1;
        for (int d = 0; d < 6 && ok; ++d)
            if (J.wait[d]) ok = hx::spin_until(J.wait[d], base + wait_value, timeout_ns, err);
    }
    __syncthreads();
    const hx::Geom g(by, bz);
    const size_t sx = (size_t)g.py * g.pz, sy = g.pz;
    unsigned long long worst = 0;
    // One row per CTA iteration: the (box, i, j) decode happens once per row
    // and the threads stream along it (k-contiguous rows coalesce).
    for (int row = blockIdx.x; ok && row < J.rows[J.nbox]; row += gridDim.x) {
        int b = 0;
        while (row >= J.rows[b + 1]) ++b;
        const int *x = J.box[b];
        const int rl = row - J.rows[b];
        const int nj = x[3] - x[2], nk = x[5] - x[4];
        const bool along_k = nk > 1;
        const int i = x[0] + (along_k ? rl / nj : rl);
        const int j = along_k ? x[2] + rl % nj : x[2];
        const int len = along_k ? nk : nj;
        const size_t c0 = g.at(i, j, x[4]);
        const size_t step_c = along_k ? 1 : sy;
        // neighbour-facing planes this whole row lies on (x and y faces; a
        // z face is one k of a k-row, or every cell of a z column)
        unsigned whole = 0, zface = 0;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
            if (!J.remote[d]) continue;
            if (d < 2 ? i == J.face[d] : d < 4 ? (along_k ? j == J.face[d] : false) : false)
                whole |= 1u << d;
            if (d >= 4 || (d >= 2 && !along_k)) zface |= 1u << d;
        }
        // One cell: relax, store locally, fold the residual, and store to
        // every neighbour-facing plane it lies on except `skip` (the row's
        // primary face when the caller stores that one as a pair).
        // One cell in two parts. relax: the six-point update (and the
        // residual) — loads and arithmetic only, so the loads of several
        // cells can be in flight together; put: store it locally and to
        // every neighbour-facing plane it lies on except `skip` (the row's
        // primary face when the caller stores that one as a pair).
        auto relax = [&](int t) -> double {
            const size_t c = c0 + (size_t)t * step_c;
            // Coherent (not .nc) loads: ghost cells were stored by a peer
            // GPU while this kernel may already have been running; the flag
            // acquire above (observed through the barrier) orders the loads.
            double zm, zp;
            const int kc = along_k ? x[4] + t : x[4];
            const int jc = along_k ? j : j + t;
            if (J.zin[0] && kc == 1)
                zm = J.zin[0][(size_t)(i - 1) * by + (jc - 1)];
            else
                zm = cur[c - 1];
            if (J.zin[1] && kc == bz)
                zp = J.zin[1][(size_t)(i - 1) * by + (jc - 1)];
            else
                zp = cur[c + 1];
            const double v = div6(sum6(cur[c - sx], cur[c + sx], cur[c - sy], cur[c + sy], zm, zp));
            if (res) worst = max(worst, abs_diff_bits(v, cur[c]));
            return v;
        };
        auto put = [&](int t, double v, unsigned skip) {
            const size_t c = c0 + (size_t)t * step_c;
            nxt[c] = v;
            unsigned on = whole & ~skip;
            if (zface) {
                const int jj = along_k ? j : j + t, kk = along_k ? x[4] + t : x[4];
#pragma unroll
                for (int d = 2; d < 6; ++d)
                    if ((zface >> d) & 1u)
                        if ((d < 4 ? jj : kk) == J.face[d]) on |= 1u << d;
            }
#pragma unroll
            for (int d = 0; d < 6; ++d)
                if ((on >> d) & 1u) {
                    if (d >= 4 && J.zout[d - 4]) {
                        const int jj = along_k ? j : j + t;
                        J.zout[d - 4][(size_t)(i - 1) * by + (jj - 1)] = v;
                    } else {
                        J.remote[d][(long long)c + J.shift[d]] = v;
                    }
                }
        };
        if (along_k && whole) {
            // The row lies on a face: store it to the neighbour in 16-byte
            // pairs, each warp's 32 pairs one whole run of four 128-byte
            // lines on the neighbour's side (the first `a` cells, up to the
            // first line boundary, go singly) — partial-line NVLink writes
            // cost bandwidth (profiles/r1_pchannel.md). Each thread relaxes
            // up to PAIRS pairs before storing any, so their loads overlap
            // (a store between them would order the next loads behind it).
            constexpr int PAIRS = 3;
            const int dp = __ffs(whole) - 1;
            const unsigned skip = 1u << dp;
            double *r0 = J.remote[dp] + ((long long)c0 + J.shift[dp]);
            const int a = min(len, (int)(((128u - ((uintptr_t)r0 & 127u)) & 127u) >> 3));
            if ((int)threadIdx.x < a) {
                const double v = relax(threadIdx.x);
                put(threadIdx.x, v, skip);
                r0[threadIdx.x] = v;
            }
            const int np = (len - a + 1) >> 1;
            for (int p0 = threadIdx.x; p0 < np; p0 += PAIRS * blockDim.x) {
                double v[PAIRS][2];
#pragma unroll
                for (int u = 0; u < PAIRS; ++u) {
                    const int t = a + 2 * (p0 + u * (int)blockDim.x);
                    if (t < len) {
                        v[u][0] = relax(t);
                        if (t + 1 < len) v[u][1] = relax(t + 1);
                    }
                }
#pragma unroll
                for (int u = 0; u < PAIRS; ++u) {
                    const int t = a + 2 * (p0 + u * (int)blockDim.x);
                    if (t >= len) continue;
                    put(t, v[u][0], skip);
                    if (t + 1 < len) {
                        put(t + 1, v[u][1], skip);
                        *reinterpret_cast<double2 *>(r0 + t) = make_double2(v[u][0], v[u][1]);
                    } else {
                        r0[t] = v[u][0];
                    }
                }
            }
        } else {
#pragma unroll 2
            for (int t = threadIdx.x; t < len; t += blockDim.x) put(t, relax(t), 0u);
        }
    }
    if (res) warp_max_to_global(worst, res);
    __syncthreads();
    if (threadIdx.x == 0) {
        // GPU-scope fence, then the arrival count; the last CTA's system
        // fence and release stores below are cumulative over every CTA's
        // local and remote stores (causality through the count), so the
        // neighbour that acquires the flag sees them all. A system fence
        // per CTA would stall each CTA for its NVLink write acks (the same
        // finding as the persistent channel's sends, profiles/r1_pchannel.md).
        __threadfence();
        const unsigned done = atomicAdd(counter, 1u) + 1u;
        if (done == gridDim.x) {
            *counter = 0u;  // re-arm (launches on one stream are ordered)
            __threadfence_system();
            const bool healthy = !err || *(volatile int *)err == 0;
            for (int d = 0; d < 6 && healthy; ++d)
                if (J.signal[d]) hx::st_release_sys(J.signal[d], base + signal_value);
            if (step) *step = base + 1;  // every CTA read it before this last one counted
        }
    }
}

// ------------------------------------------- TMA boundary faces -------
// The fused exchange for x and y face slabs (the shell of every benchmark
// decomposition without a z split). A face tile is FR rows x FK columns;
// one TMA box brings its three layers (the face and its two neighbours
// along the normal) with a one-cell halo into shared memory. Persistent
// CTAs walk their tiles through an FNST-stage ring, so the loads of the
// next tiles are in flight while 8 warps relax the current one (one tile
// row each, 4 cells per lane, 32 consecutive k per store) and store it
// locally and straight into the neighbour's ghost plane over NVLink. The
// per-row kernel above issues six dependent global loads per cell and is
// latency-bound (16 % warps active, profiles/r1_exchange_kernels.md).
constexpr int FR = 8;                 // tile rows across the face (one warp each)
constexpr int FK = 128;               // tile columns (k): 4 x 32 lanes
constexpr int FBK = FK + 4;           // box width: k-2 .. k+FK+1 (1056 B, a 16-byte multiple)
constexpr int FBR = FR + 2;           // box rows across the face, with the row halo
constexpr int FNST = 2;               // ring stages (3 CTAs/SM)
constexpr unsigned FACE_BYTES = 3u * FBR * FBK * sizeof(double);
constexpr unsigned FACE_STRIDE = (FACE_BYTES + 127u) / 128u * 128u;
constexpr unsigned FACE_STAGE_OUT = 8u * FK * sizeof(double);  // one result row per warp
constexpr size_t FACE_SMEM = (size_t)FNST * FACE_STRIDE + FACE_STAGE_OUT + FNST * sizeof(uint64_t);

// z face tiles: 8 i-rows (one warp each) x 32 j (one lane each) at k = pos;
// the box holds k-cells kstart .. kstart+3 (16-byte aligned start) of 10 x 34
// (i, j) rows
constexpr int ZTJ = 32;
constexpr int ZBK = 4, ZBJ = ZTJ + 2, ZBI = FR + 2;
constexpr unsigned ZFACE_BYTES = (unsigned)(ZBK * ZBJ * ZBI * sizeof(double));

struct FaceJob {
    int nbox;
    int axis[6];   // 0: x slab (plane i = pos), 1: y slab (row j = pos), 2: z slab (k = pos)
    int pos[6];
    int lo[6], hi[6];    // rows: j (x slab) or i (y and z slabs), 1-based, half-open
    int clo[6], chi[6];  // z slab: the j range
    int k0, k1;
    int tiles[7];  // prefix tile counts
    int ntk;
    double *remote[6];
    long long shift[6];
    int face[6];
    unsigned long long *wait[6];
    unsigned long long *signal[6];
    // z neighbours' faces through the arena slots (packed [i-1][j-1], bx x by):
    // zin[h] read instead of the z ghost column, zout[h] written for them
    const double *zin[2];
    double *zout[2];
};

__global__ void __launch_bounds__(256)
face_tma_kernel(const __grid_constant__ CUtensorMap mapx, const __grid_constant__ CUtensorMap mapy,
                const __grid_constant__ CUtensorMap mapz,
                double *__restrict__ nxt, int by, int bz, FaceJob J, int bulk,
                unsigned long long wait_value, unsigned long long signal_value, unsigned *counter,
                unsigned long long timeout_ns, int *err, unsigned long long *res,
                unsigned long long *step) {
    extern __shared__ __align__(128) unsigned char smem[];
    double *outrow = reinterpret_cast<double *>(smem + FNST * FACE_STRIDE);  // [8][FK]
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + FNST * FACE_STRIDE + FACE_STAGE_OUT);
    __shared__ int ok;
    __shared__ unsigned long long base;
    const int total = J.tiles[J.nbox];
    const int count = ((int)blockIdx.x < total) ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    // thread 0: the TMA box of this CTA's n-th tile into stage s
    auto load = [&](int n, int s) {
        const int t = (int)blockIdx.x + n * (int)gridDim.x;
        int b = 0;
        while (t >= J.tiles[b + 1]) ++b;
        const int lt = t - J.tiles[b];
        if (J.axis[b] == 2) {  // z face tile
            const int ntj = (J.chi[b] - J.clo[b] + ZTJ - 1) / ZTJ;
            const int i0 = J.lo[b] + (lt / ntj) * FR, j0 = J.clo[b] + (lt % ntj) * ZTJ;
            const int kstart = J.pos[b] == 1 ? 0 : J.pos[b] - 2;
            hx::mbar_expect_tx(&bar[s], ZFACE_BYTES);
            hx::tma_load_3d(smem + s * FACE_STRIDE, &mapz, kstart, j0 - 1, i0 - 1, &bar[s]);
            return;
        }
        const int r0 = J.lo[b] + (lt / J.ntk) * FR, kb = (lt % J.ntk) * FK;
        // a box row must start 16-byte aligned (an odd start coordinate, or a
        // negative one, is an illegal instruction): from kb - 2, or 0
        const int kbox = kb > 0 ? kb - 2 : 0;
        hx::mbar_expect_tx(&bar[s], FACE_BYTES);
        if (J.axis[b] == 0)
            hx::tma_load_3d(smem + s * FACE_STRIDE, &mapx, kbox, r0 - 1, J.pos[b] - 1, &bar[s]);
        else
            hx::tma_load_3d(smem + s * FACE_STRIDE, &mapy, kbox, J.pos[b] - 1, r0 - 1, &bar[s]);
    };
    if (threadIdx.x == 0) {
        base = step ? *(volatile unsigned long long *)step : 0ull;
        ok = 1;
        for (int d = 0; d < 6 && ok; ++d)
            if (J.wait[d]) ok = hx::spin_until(J.wait[d], base + wait_value, timeout_ns, err);
        // the ghost layers were stored by the peers (generic proxy, made
        // visible by the acquire): order them before the TMA's reads
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (ok && count) {
            hx::prefetch_tmap(&mapx);
            hx::prefetch_tmap(&mapy);
            hx::prefetch_tmap(&mapz);
            for (int s = 0; s < FNST; ++s) hx::mbar_init(&bar[s], 1);
            hx::fence_mbar_init();
            for (int n = 0; n < FNST && n < count; ++n) load(n, n);
        }
    }
    __syncthreads();
    unsigned long long worst = 0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t pz = (size_t)bz + 2;
    for (int n = 0; ok && n < count; ++n) {
        const int s = n % FNST;
        const int t = (int)blockIdx.x + n * (int)gridDim.x;
        int b = 0;
        while (t >= J.tiles[b + 1]) ++b;
        const int lt = t - J.tiles[b];
        if (J.axis[b] == 2) {
            // z face tile: cell (i0 + w, j0 + lane, pos). The neighbour-side
            // z value comes from its slot (packed, coalesced along j); the
            // result goes to nxt (one cell per 12 KB row) and to the
            // neighbour's slot (contiguous).
            const int ntj = (J.chi[b] - J.clo[b] + ZTJ - 1) / ZTJ;
            const int i = J.lo[b] + (lt / ntj) * FR + w, j = J.clo[b] + (lt % ntj) * ZTJ + lane;
            const int kf = J.pos[b], h = kf == 1 ? 0 : 1;
            const bool live = i < J.hi[b] && j < J.chi[b];
            const size_t packed = (size_t)(i - 1) * by + (j - 1);
            const double ghost = live ? J.zin[h][packed] : 0.0;
            const int C = ((w + 1) * ZBJ + lane + 1) * ZBK + (kf == 1 ? 1 : 2);
            hx::mbar_wait(&bar[s], (n / FNST) & 1);
            const double *S = reinterpret_cast<const double *>(smem + s * FACE_STRIDE);
            const double zm = h == 0 ? ghost : S[C - 1], zp = h == 1 ? ghost : S[C + 1];
            double v = div6(sum6(S[C - ZBJ * ZBK], S[C + ZBJ * ZBK], S[C - ZBK], S[C + ZBK], zm, zp));
            if (res && live) worst = max(worst, abs_diff_bits(v, S[C]));
            (void)__syncthreads_or((int)(v != v) | (res ? (int)(worst >> 63) : 0));
            if (threadIdx.x == 0 && n + FNST < count) load(n + FNST, s);
            if (live) {
                nxt[((size_t)i * (by + 2) + j) * pz + kf] = v;
                J.zout[h][packed] = v;
            }
            continue;
        }
        // tiles start at even k, so every row segment [kb, kb + FK) starts on a
        // 16-byte boundary here and on the neighbour (even row pitch)
        const int r0 = J.lo[b] + (lt / J.ntk) * FR, kb = (lt % J.ntk) * FK;
        const bool xs = J.axis[b] == 0;
        const int row = r0 + w;
        const int i = xs ? J.pos[b] : row, j = xs ? row : J.pos[b];
        // this row's destinations: our nxt, and the ghost plane of every
        // neighbour whose face the row lies on (the slab's own face, plus a
        // y face on an x slab's edge rows); no z neighbour on this path
        const long long crow = ((long long)i * (by + 2) + j) * (long long)pz + kb;
        double *dst = nxt + crow;
        double *rd0 = nullptr, *rd1 = nullptr;
#pragma unroll
        for (int d = 0; d < 4; ++d)
            if (J.remote[d] && (d < 2 ? i : j) == J.face[d]) {
                double *r = J.remote[d] + (crow + J.shift[d]);
                if (!rd0) rd0 = r; else rd1 = r;
            }
        // shared-memory strides: x slab S[3][FBR][FBK], y slab S[FBR][3][FBK]
        const int ssx = xs ? FBR * FBK : 3 * FBK;
        // cell kk of the row sits at box column kk + 2 (box from kb - 2), or
        // kk for the first tile (box from 0: its cell k = 0 is not relaxed)
        const int C0 = (xs ? (FBR + w + 1) : (3 * (w + 1) + 1)) * FBK + (kb > 0 ? 2 : 0) + lane;
        // live columns kk in [klo, khi): interior cells k in [k0, k1) of this row
        const int klo = max(0, J.k0 - kb), khi = row < J.hi[b] ? min(FK, J.k1 - kb) : 0;
        hx::mbar_wait(&bar[s], (n / FNST) & 1);
        const double *S = reinterpret_cast<const double *>(smem + s * FACE_STRIDE);
        const int kbox = kb > 0 ? kb - 2 : 0;
        if ((J.zin[0] || J.zin[1]) && row < J.hi[b]) {
            // this row's z ghosts (k = 0, k = bz + 1) come from the z
            // neighbours' slots, not the ghost column; only this warp reads them
            double *Sw = reinterpret_cast<double *>(smem + s * FACE_STRIDE);
            const int rs = C0 - lane - (kb > 0 ? 2 : 0) - kbox;  // (virtual) index of k = 0
            const size_t packed = (size_t)(i - 1) * by + (j - 1);
            if (lane == 0 && J.zin[0] && kb == 0) Sw[rs] = J.zin[0][packed];
            if (lane == 0 && J.zin[1] && kb <= bz && bz < kb + FK) Sw[rs + bz + 1] = J.zin[1][packed];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before any TMA refill
            __syncwarp();
        }
        constexpr int U = FK / 32;
        double v[U];
        bool fast = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int C = C0 + 32 * u;
            v[u] = sum6(S[C - ssx], S[C + ssx], S[C - FBK], S[C + FBK], S[C - 1], S[C + 1]);
            fast &= div6_fast_ok(v[u]);
        }
        if (fast) {
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = div6_fast(v[u]);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = div6(v[u]);
        }
        if (res) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (lane + 32 * u >= klo && lane + 32 * u < khi)
                    worst = max(worst, abs_diff_bits(v[u], S[C0 + 32 * u]));
        }
        // cells outside the interior keep their current value (the bulk
        // segment's end cells; never stored locally)
        int nanp = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int kk = lane + 32 * u;
            if (kk < klo || kk >= khi) v[u] = S[C0 + 32 * u];
            nanp |= v[u] != v[u];
        }
        // every shared load has completed once the barrier is passed: each
        // value fed v, and v and the residual feed the predicate, so the
        // stage may be refilled right after it
        (void)__syncthreads_or(nanp | (res ? (int)(worst >> 63) : 0));
        if (threadIdx.x == 0 && n + FNST < count) load(n + FNST, s);  // refill during the stores
        if ((J.zout[0] || J.zout[1]) && khi > klo) {  // the row's z-face cells, for the z neighbours
            const size_t packed = (size_t)(i - 1) * by + (j - 1);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int kk = lane + 32 * u;
                if (kk < klo || kk >= khi) continue;
                if (J.zout[0] && kb + kk == 1) J.zout[0][packed] = v[u];
                if (J.zout[1] && kb + kk == bz) J.zout[1][packed] = v[u];
            }
        }
        if (bulk == 2 && khi > klo) {
            // paired 16-byte stores: the row is staged in shared memory, then
            // each lane stores two adjacent cells (512 B per warp instruction,
            // 16-byte aligned here and on the neighbour)
            double *row_out = outrow + w * FK;
            __syncwarp();
#pragma unroll
            for (int u = 0; u < U; ++u) row_out[lane + 32 * u] = v[u];
            __syncwarp();
#pragma unroll
            for (int h = 0; h < FK / 64; ++h) {
                const int kk = 2 * lane + 64 * h;
                if (kb + kk >= (int)pz) continue;
                const double2 pr = *reinterpret_cast<const double2 *>(row_out + kk);
                if (rd0) *reinterpret_cast<double2 *>(rd0 + kk) = pr;
                if (rd1) *reinterpret_cast<double2 *>(rd1 + kk) = pr;
                const bool l0 = kk >= klo && kk < khi, l1 = kk + 1 >= klo && kk + 1 < khi;
                if (l0 && l1)
                    *reinterpret_cast<double2 *>(dst + kk) = pr;
                else if (l0)
                    dst[kk] = pr.x;
                else if (l1)
                    dst[kk + 1] = pr.y;
            }
            continue;
        }
        if (bulk == 1 && rd0 && khi > klo) {
            // the neighbour's copy leaves as whole 16-byte-aligned row
            // segments by bulk copy (full 128-byte lines over NVLink; a
            // warp's plain 8-byte stores straddle line boundaries). The
            // segment's end cells k = 0 / bz + 1 land on the neighbour's
            // edge cells (ghost plane x z ghost), which no stencil reads.
            double *row_out = outrow + w * FK;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int kk = lane + 32 * u;
                row_out[kk] = v[u];
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                const unsigned bytes = (unsigned)(min(FK, (int)pz - kb) * sizeof(double));
                const uint32_t src = hx::smem_addr(row_out);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(rd0), "r"(src), "r"(bytes) : "memory");
                if (rd1)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                 ::"l"(rd1), "r"(src), "r"(bytes) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            rd0 = rd1 = nullptr;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int kk = lane + 32 * u;
            if (kk < klo || kk >= khi) continue;
            dst[kk] = v[u];
            if (rd0) rd0[kk] = v[u];
            if (rd1) rd1[kk] = v[u];
        }
    }
    // every bulk store has completed (written, not only read out of shared
    // memory) before this CTA's fence and arrival count
    if (bulk == 1 && (threadIdx.x & 31) == 0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (res) warp_max_to_global(worst, res);
    __syncthreads();
    if (threadIdx.x == 0) {
        // as shell_put_kernel: GPU-scope fence and arrival count per CTA, the
        // last CTA's system fence + releases are cumulative over all of them
        __threadfence();
        const unsigned done = atomicAdd(counter, 1u) + 1u;
        if (done == gridDim.x) {
            *counter = 0u;
            __threadfence_system();
            const bool healthy = !err || *(volatile int *)err == 0;
            for (int d = 0; d < 6 && healthy; ++d)
                if (J.signal[d]) hx::st_release_sys(J.signal[d], base + signal_value);
            if (step) *step = base + 1;
        }
    }
}

// ---------------------------------------------- persistent small blocks --
// Small blocks are launch-bound: a 64^3 sweep is ~1 us of HBM work, while a
// fused step costs two launches plus their gaps even when replayed from a
// CUDA graph. persist_kernel runs `iters` fused iterations of ONE block in
// one launch: every iteration waits for the neighbours' flags (their
// boundary of it-1 is in our ghost planes, and they are done reading the
// ghosts we are about to write), relaxes the whole block — storing each
// neighbour-facing cell also into the neighbour's next-buffer ghost plane,
// as hx_shell_put does — then a grid barrier, and CTA 0 releases
// flag = it + 2 to every neighbour. Grid-wide barriers need every CTA
// resident: the host sizes the grid to fit (hx_persist_run).
struct PersistJob {
    double *field[2];        // our two padded fields
    double *peer[6][2];      // each neighbour's two fields (null: no neighbour)
    long long shift[6];      // our padded offset + shift[d] = its ghost cell
    int face[6];
    unsigned long long *wait[6];
    unsigned long long *signal[6];
    // z faces through the arena slots, as the fused steps (hx_shell_put_z):
    // for an iteration of parity q, zin[q][h] is our slot on side h (parity
    // q) and zout[q][h] the neighbour's slot it writes (parity q ^ 1)
    const double *zin[2][2];
    double *zout[2][2];
};

// One grid-wide barrier: the last CTA to arrive resets the count and bumps
// the generation (release); the others spin on it (acquire).
__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g, prev;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                     : "=r"(prev) : "l"(count) : "memory");
        if (prev + 1u == gridDim.x) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
        } else {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
            } while (v == g);
        }
    }
    __syncthreads();
}

// One grid barrier per iteration. Every CTA acquires the neighbours' flags
// itself (threads 0-5, one flag each), so no barrier is needed to hand
// CTA 0's acquires to the grid; the barrier after the sweep orders every
// CTA's local and peer stores before CTA 0's release, and also closes the
// iteration for the local buffers (the next one writes what this one read).
// A timed-out wait skips the sweep but still arrives, so nobody hangs.
__global__ void __launch_bounds__(256)
persist_kernel(PersistJob J, int bx, int by, int bz, int parity, unsigned long long it0, int iters,
               unsigned *bar_count, unsigned *bar_gen, unsigned long long timeout_ns, int *err) {
    const hx::Geom g(by, bz);
    const unsigned sx = (unsigned)(g.py * g.pz), sy = (unsigned)g.pz;
    const unsigned cells = (unsigned)bx * by * bz;  // the host keeps blocks below 2^31 cells
    for (int n = 0; n < iters; ++n) {
        const unsigned long long it = it0 + n;
        const int p = (parity + n) & 1;
        int ok = 1;
        if (threadIdx.x < 6 && J.wait[threadIdx.x])
            ok = hx::spin_until(J.wait[threadIdx.x], it + 1, timeout_ns, err, 32);
        ok = __syncthreads_and(ok);
        if (ok && !(err && *(volatile int *)err)) {
            const double *cur = J.field[p];
            double *nxt = J.field[p ^ 1];
            const int qi = (int)(it & 1);  // zin[qi]: this iteration's slots; zout[qi]: the
                                           // neighbour's slots for the next one
            for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < cells;
                 q += gridDim.x * blockDim.x) {
                const unsigned r = q / (unsigned)bz;
                const int k = 1 + (int)(q - r * (unsigned)bz);
                const unsigned i0 = r / (unsigned)by;
                const int j = 1 + (int)(r - i0 * (unsigned)by), i = 1 + (int)i0;
                const size_t c = (size_t)i * sx + (size_t)j * sy + k;
                const unsigned packed = r;  // (i - 1) * by + (j - 1)
                const double zm = (k == 1 && J.zin[qi][0]) ? J.zin[qi][0][packed] : cur[c - 1];
                const double zp = (k == bz && J.zin[qi][1]) ? J.zin[qi][1][packed] : cur[c + 1];
                const double v = div6(sum6(cur[c - sx], cur[c + sx], cur[c - sy], cur[c + sy], zm, zp));
                nxt[c] = v;
                const int at[3] = {i, j, k};
#pragma unroll
                for (int d = 0; d < 6; ++d)
                    if (J.peer[d][p ^ 1] && at[d >> 1] == J.face[d]) {
                        if (d >= 4 && J.zout[qi][d - 4])
                            J.zout[qi][d - 4][packed] = v;
                        else
                            J.peer[d][p ^ 1][(long long)c + J.shift[d]] = v;
                    }
            }
        }
        grid_barrier(bar_count, bar_gen);  // every CTA's local + peer stores are done
        if (err && *(volatile int *)err) return;  // a timed-out wait: everyone stops
        // CTA 0 releases the six flags in parallel (each st.release.sys is
        // cumulative over the stores the grid barrier ordered before it)
        if (blockIdx.x == 0 && threadIdx.x < 6 && J.signal[threadIdx.x])
            hx::st_release_sys(J.signal[threadIdx.x], it + 2);
    }
}

__global__ void fill_kernel(double *p, size_t n, double v) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
         q += (size_t)gridDim.x * blockDim.x)
        p[q] = v;
}

// ------------------------------------------------------ host helpers -----
std::mutex g_map_mu;
std::map<std::tuple<const void *, int, int, int, int, int>, CUtensorMap> g_maps;

int l2_promotion() {
    if (g_l2promo < 0) {
        // 0 none, 1 64B, 2 128B, 3 256B. Measured (tools/sweep_tma_knobs.sh):
        // 256-byte promotion is fastest for every sweep shape — 1536^3
        // 8.883 ms vs 8.927 (64B), 1535^3 8.831 vs 8.877, 768x1536x3072
        // 8.816 vs 8.862.
        const char *e = getenv("HX_TMA_L2PROMO");
        g_l2promo = e ? atoi(e) : 3;
        if (g_l2promo < 0 || g_l2promo > 3) g_l2promo = 3;
    }
    return g_l2promo;
}

int tensor_map_for(const double *cur, int bx, int by, int bz, int box_z, CUtensorMap *out) {
    const int promo = l2_promotion();
    auto key = std::make_tuple((const void *)cur, bx, by, bz, box_z, promo);
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        auto it = g_maps.find(key);
        if (it != g_maps.end()) {
            *out = it->second;
            return 0;
        }
    }
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)hx_internal_driver_sym("cuTensorMapEncodeTiled");
    if (!encode) return HX_E_NODRIVER;
    const cuuint64_t pz = (cuuint64_t)bz + 2, py = (cuuint64_t)by + 2, px = (cuuint64_t)bx + 2;
    cuuint64_t dims[3] = {pz, py, px};
    cuuint64_t strides[2] = {pz * sizeof(double), py * pz * sizeof(double)};
    cuuint32_t box[3] = {(cuuint32_t)box_z, BOX_Y, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)cur, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return HX_E_TMA;
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 256) g_maps.clear();
    g_maps[key] = m;
    *out = m;
    return 0;
}

// Tensor map over the padded block with an arbitrary 3-D box (the face
// kernel's x-slab, y-slab and z-tile boxes), cached like tensor_map_for's.
// promo is the L2 promotion (0 none .. 3 256 B): the x/y boxes read whole
// 132-double row segments (256 B, as the stencil), but a z-tile row is 4
// doubles 12 KB from the next, and promoting it to 256 B would fetch 8x
// the bytes it uses from DRAM.
std::map<std::tuple<const void *, int, int, int, int, int, int, int>, CUtensorMap> g_face_maps;

int face_map_for(const double *cur, int bx, int by, int bz, int b0, int b1, int b2, int promo,
                 CUtensorMap *out) {
    auto key = std::make_tuple((const void *)cur, bx, by, bz, b0, b1, b2, promo);
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        auto it = g_face_maps.find(key);
        if (it != g_face_maps.end()) {
            *out = it->second;
            return 0;
        }
    }
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)hx_internal_driver_sym("cuTensorMapEncodeTiled");
    if (!encode) return HX_E_NODRIVER;
    const cuuint64_t pz = (cuuint64_t)bz + 2, py = (cuuint64_t)by + 2, px = (cuuint64_t)bx + 2;
    cuuint64_t dims[3] = {pz, py, px};
    cuuint64_t strides[2] = {pz * sizeof(double), py * pz * sizeof(double)};
    cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)cur, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return HX_E_TMA;
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_face_maps.size() > 256) g_face_maps.clear();
    g_face_maps[key] = m;
    *out = m;
    return 0;
}

bool tma_eligible(const double *cur, int bz) {
    return ((bz + 2) % 2 == 0) && (((uintptr_t)cur & 15) == 0);
}

int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

// Function attributes live in each device's context: set them once per
// device (a process driving several GPUs launches on each; `done` holds a
// bit per ordinal) and ask for the full shared-memory carveout so that
// 3 CTAs of ~74 KB fit per SM.
template <typename Kernel>
int ensure_smem(Kernel kernel, size_t bytes, unsigned long long &done) {
    int dev = 0;
    HX_TRY(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(done & bit)) {
        HX_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        HX_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    (int)cudaSharedmemCarveoutMaxShared));
        done |= bit;
    }
    return 0;
}

template <bool RES, int BOX_Z, bool ZE>
int launch_tma_t(const CUtensorMap &map, double *nxt, int by, int bz, int i0, int i1, int j0,
                 int j1, int k0, int k1, int klive, int ntj, int ntk, int chunk, int nchunks,
                 int grows, long items, unsigned long long *res, const ZEdge &Z, cudaStream_t st) {
    static unsigned long long attr_set = 0;
    if (int rc = ensure_smem(stencil_tma_kernel<RES, BOX_Z, ZE>, SMEM_BYTES, attr_set)) return rc;
    stencil_tma_kernel<RES, BOX_Z, ZE><<<(unsigned)items, THREADS, SMEM_BYTES, st>>>(
        map, nxt, by, bz, i0, i1, j0, j1, k0, k1, klive, ntj, ntk, chunk, nchunks, grows, res, Z);
    HX_LAUNCH_CHECK();
    return 0;
}

// Tile / chunk / group schedule shared by the TMA and row-bulk-copy pipelines.
struct Schedule {
    int ntj, ntk, chunk, nchunks, grows;
    long items;
};

Schedule make_schedule(int i0, int i1, int j0, int j1, int k0, int k1) {
    Schedule sc;
    const int ni = i1 - i0, nj = j1 - j0, nk = k1 - k0;
    sc.ntj = (nj + TY - 1) / TY;
    sc.ntk = (nk + TZ - 1) / TZ;
    int chunk = g_chunk;
    if (chunk <= 0) {
        // Short chunks keep neighbouring CTAs in step (their tile halos are
        // L2 hits); the grouped order makes the 2 boundary planes a chunk
        // shares with the next one L2 hits too.
        // Tuned on B200 at 1536^3 (tools/prof_stencil.py sweeps, profiles/):
        // chunk 4 with ~288-tile groups reaches ~99% of the measured copy
        // bandwidth; chunk 10 / ungrouped was 87%, chunk 96 70%.
        const char *e = getenv("HX_STENCIL_CHUNK");
        chunk = e ? atoi(e) : 4;
        if (chunk <= 0) chunk = 4;
    }
    sc.chunk = std::min(chunk, ni);
    sc.nchunks = (ni + sc.chunk - 1) / sc.chunk;
    int grows = std::max(1, (288 + sc.ntk / 2) / sc.ntk);  // tile rows per scheduling group
    if (const char *e = getenv("HX_STENCIL_GROUP")) grows = std::max(1, atoi(e));
    sc.grows = std::min(grows, sc.ntj);
    sc.items = (long)sc.ntj * sc.ntk * sc.nchunks;
    return sc;
}

int launch_tma(const double *cur, double *nxt, int bx, int by, int bz, int i0, int i1, int j0,
               int j1, int k0, int k1, unsigned long long *res, cudaStream_t st,
               const ZEdge *zedge = nullptr) {
    ZEdge Z;
    memset(&Z, 0, sizeof(Z));
    if (zedge) Z = *zedge;
    const bool ze = zedge && (Z.flag[0] || Z.flag[1] || Z.xyflag[0] || Z.xyflag[1] ||
                              Z.xyflag[2] || Z.xyflag[3]);
    // every tile starts at kb = kt + t*TZ (TZ even): one box width per launch. A
    // box whose first column k0 is even (a sweep trimmed by a -z neighbour)
    // uses the 68-wide box shifted to a 16-byte-aligned start; its stores then
    // start on even k. HX_TMA_KEEP_GRID=1 keeps the full sweep's tile grid
    // instead (66-wide box from k0 - 1, stores below k0 masked via klive):
    // measured slower, 8.90 vs 8.77 ms for a 1536^3 block trimmed at k = 2
    // (tools/prof_box.py) — the shifted tiles' stores are 16-byte aligned
    static int keep_grid = -1;
    if (keep_grid < 0) {
        const char *e = getenv("HX_TMA_KEEP_GRID");
        keep_grid = e ? atoi(e) : 0;
    }
    const int kt = (((k0 - 1) & 1) && keep_grid) ? k0 - 1 : k0;
    const bool shifted = ((kt - 1) & 1) != 0;
    const int box_z = shifted ? TZ + 4 : TZ + 2;
    CUtensorMap map;
    int rc = tensor_map_for(cur, bx, by, bz, box_z, &map);
    if (rc) return rc;
    const Schedule sc = make_schedule(i0, i1, j0, j1, kt, k1);
    if (sc.items > 0x7fffffffL) return HX_E_INVALID;
#define HX_TMA_LAUNCH(R, W, E)                                                             \
    launch_tma_t<R, W, E>(map, nxt, by, bz, i0, i1, j0, j1, kt, k1, k0, sc.ntj, sc.ntk, sc.chunk, \
                          sc.nchunks, sc.grows, sc.items, res, Z, st)
    if (ze) {  // the z-edge variant: only unshifted boxes starting at k = 1 reach it (halo.py)
        if (shifted) return HX_E_INVALID;
        return res ? HX_TMA_LAUNCH(true, TZ + 2, true) : HX_TMA_LAUNCH(false, TZ + 2, true);
    }
    if (shifted)
        return res ? HX_TMA_LAUNCH(true, TZ + 4, false) : HX_TMA_LAUNCH(false, TZ + 4, false);
    return res ? HX_TMA_LAUNCH(true, TZ + 2, false) : HX_TMA_LAUNCH(false, TZ + 2, false);
#undef HX_TMA_LAUNCH
}

// The four (row parity, plane parity) class maps of stencil_pair_kernel.
std::map<std::tuple<const void *, int, int, int, int>, PairMaps> g_pair_maps;

int pair_maps_for(const double *cur, int bx, int by, int bz, PairMaps *out) {
    const int promo = l2_promotion();
    auto key = std::make_tuple((const void *)cur, bx, by, bz, promo);
    {
        std::lock_guard<std::mutex> lk(g_map_mu);
        auto it = g_pair_maps.find(key);
        if (it != g_pair_maps.end()) {
            *out = it->second;
            return 0;
        }
    }
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)hx_internal_driver_sym("cuTensorMapEncodeTiled");
    if (!encode) return HX_E_NODRIVER;
    const cuuint64_t pz = (cuuint64_t)bz + 2, py = (cuuint64_t)by + 2, px = (cuuint64_t)bx + 2;
    const cuuint64_t plane = py * pz;
    PairMaps pm;
    for (int b = 0; b < 2; ++b)
        for (int a = 0; a < 2; ++a) {
            cuuint64_t dims[3] = {a * pz + b * plane + pz, (py - a + 1) / 2, (px - b + 1) / 2};
            cuuint64_t strides[2] = {2 * pz * sizeof(double), 2 * plane * sizeof(double)};
            cuuint32_t box[3] = {(cuuint32_t)PW, (cuuint32_t)PH, 1};
            cuuint32_t estr[3] = {1, 1, 1};
            CUresult r = encode(&pm.m[a + 2 * b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)cur,
                                dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return HX_E_TMA;
        }
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_pair_maps.size() > 64) g_pair_maps.clear();
    g_pair_maps[key] = pm;
    *out = pm;
    return 0;
}

template <bool RES>
int launch_pair_t(const PairMaps &pm, double *nxt, int by, int bz, int i0, int i1, int j0, int j1,
                  int k0, int k1, const Schedule &sc, unsigned long long *res, cudaStream_t st) {
    static unsigned long long attr_set = 0;
    if (int rc = ensure_smem(stencil_pair_kernel<RES>, PSMEM_BYTES, attr_set)) return rc;
    stencil_pair_kernel<RES><<<(unsigned)sc.items, THREADS, PSMEM_BYTES, st>>>(
        pm, nxt, by, bz, i0, i1, j0, j1, k0, k1, sc.ntj, sc.ntk, sc.chunk, sc.nchunks, sc.grows,
        res);
    HX_LAUNCH_CHECK();
    return 0;
}

int launch_pair(const double *cur, double *nxt, int bx, int by, int bz, int i0, int i1, int j0,
                int j1, int k0, int k1, unsigned long long *res, cudaStream_t st) {
    if (((uintptr_t)cur & 15) != 0) return HX_E_INVALID;  // tensor maps need a 16-byte base
    const long long plane = (long long)(by + 2) * (bz + 2);
    if (plane + 2LL * (bz + 2) + PW >= 0x7fffffffLL) return HX_E_INVALID;  // int box coordinates
    PairMaps pm;
    int rc = pair_maps_for(cur, bx, by, bz, &pm);
    if (rc) return rc;
    const Schedule sc = make_schedule(i0, i1, j0, j1, k0, k1);
    if (sc.items > 0x7fffffffL) return HX_E_INVALID;
    return res ? launch_pair_t<true>(pm, nxt, by, bz, i0, i1, j0, j1, k0, k1, sc, res, st)
               : launch_pair_t<false>(pm, nxt, by, bz, i0, i1, j0, j1, k0, k1, sc, res, st);
}

// Thin boundary slabs of the overlap split (one plane / row / column thick):
// one thread per cell over the flattened box, consecutive threads along the
// box's longest fast axis (k if the slab spans k, else j) so the centre
// loads coalesce; neighbours come through L1/L2.
__global__ void __launch_bounds__(256)
stencil_slab_kernel(const double *__restrict__ cur, double *__restrict__ nxt, int by, int bz,
                    int i0, int j0, int k0, int ni, int nj, int nk, int k_fast,
                    unsigned long long *res) {
    const hx::Geom g(by, bz);
    const long long n = (long long)ni * nj * nk;
    unsigned long long worst = 0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        if (k_fast) {
            k = k0 + (int)(q % nk);
            const long long r = q / nk;
            j = j0 + (int)(r % nj);
            i = i0 + (int)(r / nj);
        } else {
            j = j0 + (int)(q % nj);
            const long long r = q / nj;
            k = k0 + (int)(r % nk);
            i = i0 + (int)(r / nk);
        }
        const size_t c = g.at(i, j, k);
        const size_t sx = (size_t)g.py * g.pz, sy = g.pz;
        const double v = div6(sum6(__ldg(cur + c - sx), __ldg(cur + c + sx), __ldg(cur + c - sy),
                                   __ldg(cur + c + sy), __ldg(cur + c - 1), __ldg(cur + c + 1)));
        nxt[c] = v;
        if (res) worst = max(worst, abs_diff_bits(v, __ldg(cur + c)));
    }
    if (res) warp_max_to_global(worst, res);
}

// One z column (k = kcol) over an (i, j) box: the z-face boundary shell of
// the overlap split. Every (i, j) row segment is one 32-byte sector, so each
// lane loads the aligned 4-double quad holding c[k-1..k+1] with two 16-byte
// loads, takes y neighbours from adjacent lanes by shuffle (lanes run along
// j), and loads only the two x neighbours separately. ~3 loads per cell
// instead of 7 scattered 8-byte ones.
__global__ void __launch_bounds__(256)
stencil_zcol_kernel(const double *__restrict__ cur, double *__restrict__ nxt, int by, int bz,
                    int i0, int i1, int j0, int j1, int kcol, unsigned long long *res) {
    const hx::Geom g(by, bz);
    const int ka = ((kcol - 1) & 1) ? kcol - 2 : kcol - 1;  // 16-byte aligned quad start
    const int c = kcol - ka;                                 // centre index in the quad (1 or 2)
    const int lane = threadIdx.x & 31;
    const int j = j0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int i = i0 + blockIdx.y;
    unsigned long long worst = 0;
    const bool live = j < j1;
    const int jj = live ? j : j1 - 1;  // keep every lane active for the shuffles
    const double2 *row = reinterpret_cast<const double2 *>(cur + g.at(i, jj, ka));
    const double2 lo = __ldg(row), hi = __ldg(row + 1);
    const double q[4] = {lo.x, lo.y, hi.x, hi.y};
    const double ctr = q[c], zm = q[c - 1], zp = q[c + 1];
    double ym = __shfl_up_sync(0xffffffffu, ctr, 1);
    double yp = __shfl_down_sync(0xffffffffu, ctr, 1);
    if (lane == 0 || jj - 1 < j0) ym = __ldg(cur + g.at(i, jj - 1, kcol));
    if (lane == 31 || jj + 1 >= j1) yp = __ldg(cur + g.at(i, jj + 1, kcol));
    const size_t sx = (size_t)g.py * g.pz;
    const size_t at = g.at(i, jj, kcol);
    const double v = div6(sum6(__ldg(cur + at - sx), __ldg(cur + at + sx), ym, yp, zm, zp));
    if (live) {
        nxt[at] = v;
        if (res) worst = abs_diff_bits(v, ctr);
    }
    if (res) warp_max_to_global(worst, res);
}

int launch_zcol(const double *cur, double *nxt, int by, int bz, int i0, int i1, int j0, int j1,
                int kcol, unsigned long long *res, cudaStream_t st) {
    dim3 grd((j1 - j0 + 255) / 256, i1 - i0);
    if (grd.y > 65535) return HX_E_INVALID;
    stencil_zcol_kernel<<<grd, 256, 0, st>>>(cur, nxt, by, bz, i0, i1, j0, j1, kcol, res);
    HX_LAUNCH_CHECK();
    return 0;
}

int launch_slab(const double *cur, double *nxt, int by, int bz, int i0, int i1, int j0, int j1,
                int k0, int k1, unsigned long long *res, cudaStream_t st) {
    const int ni = i1 - i0, nj = j1 - j0, nk = k1 - k0;
    const long long n = (long long)ni * nj * nk;
    const int k_fast = (nk >= 32 || nk >= nj) ? 1 : 0;
    const long long want = (n + 255) / 256;
    const unsigned grid = (unsigned)std::min<long long>(want, 16LL * num_sms());
    stencil_slab_kernel<<<grid, 256, 0, st>>>(cur, nxt, by, bz, i0, j0, k0, ni, nj, nk, k_fast,
                                              res);
    HX_LAUNCH_CHECK();
    return 0;
}

int launch_generic(const double *cur, double *nxt, int by, int bz, int i0, int i1, int j0, int j1,
                   int k0, int k1, unsigned long long *res, cudaStream_t st) {
    dim3 blk(32, 8, 1);
    dim3 grd((k1 - k0 + 31) / 32, (j1 - j0 + 7) / 8, i1 - i0);
    if (grd.y > 65535 || grd.z > 65535) return HX_E_INVALID;
    stencil_generic_kernel<<<grd, blk, 0, st>>>(cur, nxt, by, bz, i0, j0, j1, k0, k1, res);
    HX_LAUNCH_CHECK();
    return 0;
}

}  // namespace

extern "C" {

int hx_stencil_set_variant(int variant) {
    int prev = g_variant;
    g_variant = variant;
    return prev;
}

int hx_stencil_last_variant(void) { return g_last_variant; }

int hx_stencil_set_chunk(int planes) {
    int prev = g_chunk;
    g_chunk = planes;
    return prev;
}

int hx_stencil_box(const double *cur, double *nxt, int bx, int by, int bz, int i0, int i1, int j0,
                   int j1, int k0, int k1, unsigned long long *res, void *stream) {
    if (!cur || !nxt || bx < 1 || by < 1 || bz < 1) return HX_E_INVALID;
    if (i0 < 1 || j0 < 1 || k0 < 1 || i1 > bx + 1 || j1 > by + 1 || k1 > bz + 1) return HX_E_INVALID;
    if (i0 >= i1 || j0 >= j1 || k0 >= k1) return 0;  // empty box
    cudaStream_t st = (cudaStream_t)stream;
    int want = g_variant;
    if (want == 0) {
        // thin slabs (the overlap split's boundary shell) would waste most of
        // a 32x64 TMA tile: single z columns get the quad-load kernel, other
        // thin boxes the flattened slab kernel
        const bool thin = (j1 - j0) < 8 || (k1 - k0) < 16;
        const int ka = ((k0 - 1) & 1) ? k0 - 2 : k0 - 1;
        const bool zcol = k1 - k0 == 1 && (j1 - j0) >= 32 && tma_eligible(cur, bz) &&
                          ka >= 0 && ka + 3 <= bz + 1;
        want = zcol ? 4 : thin ? 3 : (tma_eligible(cur, bz) ? 1 : 5);
    }
    if (want == 4) {
        const int ka = ((k0 - 1) & 1) ? k0 - 2 : k0 - 1;
        if (k1 - k0 != 1 || !tma_eligible(cur, bz) || ka < 0 || ka + 3 > bz + 1) return HX_E_INVALID;
        g_last_variant = 4;
        return launch_zcol(cur, nxt, by, bz, i0, i1, j0, j1, k0, res, st);
    }
    if (want == 3) {
        g_last_variant = 3;
        return launch_slab(cur, nxt, by, bz, i0, i1, j0, j1, k0, k1, res, st);
    }
    if (want == 5 || (want == 1 && !tma_eligible(cur, bz) && g_variant == 0)) {
        g_last_variant = 5;
        return launch_pair(cur, nxt, bx, by, bz, i0, i1, j0, j1, k0, k1, res, st);
    }
    if (want == 1 && !tma_eligible(cur, bz)) return HX_E_INVALID;
    if (want == 1) {
        int rc = launch_tma(cur, nxt, bx, by, bz, i0, i1, j0, j1, k0, k1, res, st);
        if (rc == 0) {
            g_last_variant = 1;
            return 0;
        }
        if (g_variant == 1) return rc;  // forced: report, do not fall back
        g_last_variant = 5;             // no tensor map (driver entry point): same pipeline
        return launch_pair(cur, nxt, bx, by, bz, i0, i1, j0, j1, k0, k1, res, st);
    }
    g_last_variant = 2;
    return launch_generic(cur, nxt, by, bz, i0, i1, j0, j1, k0, k1, res, st);
}

// The interior sweep of the fused exchange with the z faces (see ZEdge).
int hx_stencil_box_z(const double *cur, double *nxt, int bx, int by, int bz, int i0, int i1,
                     int j0, int j1, int k0, int k1, unsigned long long *res,
                     const unsigned long long *const zflag[2], const unsigned long long *zstep,
                     const double *const zin[2], double *const zout[2],
                     unsigned long long timeout_ns, int *err, void *stream) {
    if (!cur || !nxt || bx < 1 || by < 1 || bz < 1 || !zstep || !zflag) return HX_E_INVALID;
    if (i0 < 1 || j0 < 1 || k0 != 1 || i1 > bx + 1 || j1 > by + 1 || k1 != bz + 1)
        return HX_E_INVALID;  // whole rows in z: the box holds both z faces
    if (i0 >= i1 || j0 >= j1) return 0;
    if (!tma_eligible(cur, bz)) return HX_E_INVALID;
    if (zflag[0] && zflag[1] && bz <= TZ) return HX_E_INVALID;  // a tile would hold both faces
    ZEdge Z;
    memset(&Z, 0, sizeof(Z));
    for (int h = 0; h < 2; ++h) {
        Z.flag[h] = zflag[h];
        if (zflag[h] && (!zin || !zout || !zin[h] || !zout[h])) return HX_E_INVALID;
        Z.zin[h] = zflag[h] ? zin[h] : nullptr;
        Z.zout[h] = zflag[h] ? zout[h] : nullptr;
    }
    Z.step = zstep;
    Z.timeout_ns = timeout_ns;
    Z.err = err;
    g_last_variant = 1;
    cudaStream_t st = (cudaStream_t)stream;
    // One sweep over whole rows: the tiles that hold k = 1 (with a -z
    // neighbour) or k = bz (+z) take the z-edge work (flag wait, slot patches,
    // face copies) at run time; the rest run the plain path. Keeping the edge
    // tiles in the main sweep's schedule shares their DRAM pages with the
    // neighbouring tiles: a separate 64-wide strip sweep runs at about half
    // the HBM rate (profiles/r2_zface_dram.md). HX_ZE_STRIPS=1 restores the
    // split launches (middle, then edge strips) for comparison.
    static int strips = -1;
    if (strips < 0) {
        const char *e = getenv("HX_ZE_STRIPS");
        strips = e ? atoi(e) : 0;
    }
    const int klo_end = 1 + TZ;                       // the first tile column: [1, 1 + TZ)
    const int khi_beg = 1 + ((bz - 1) / TZ) * TZ;     // the tile column holding k = bz
    if (!strips || khi_beg <= klo_end)
        return launch_tma(cur, nxt, bx, by, bz, i0, i1, j0, j1, 1, bz + 1, res, st, &Z);
    const int mid0 = Z.flag[0] ? klo_end : 1, mid1 = Z.flag[1] ? khi_beg : bz + 1;
    if (int rc = launch_tma(cur, nxt, bx, by, bz, i0, i1, j0, j1, mid0, mid1, res, st)) return rc;
    ZEdge lo = Z, hi = Z;
    lo.flag[1] = nullptr;
    hi.flag[0] = nullptr;
    if (Z.flag[0])
        if (int rc = launch_tma(cur, nxt, bx, by, bz, i0, i1, j0, j1, 1, klo_end, res, st, &lo))
            return rc;
    if (Z.flag[1])
        return launch_tma(cur, nxt, bx, by, bz, i0, i1, j0, j1, khi_beg, bz + 1, res, st, &hi);
    return 0;
}

// After a fused step's interior and boundary kernels: release the z
// neighbours' flags (= *step + 2, cumulative over both kernels' slot
// writes, which precede this launch on the stream) and advance *step.
// Work items of the one-sweep fused step that hold a face (host only): the
// kernel's own rule (stencil_tma_kernel) — tile columns holding k = 1 / bz,
// tile rows holding j = 1 / by, chunks holding i = 1 / bx, for the sides
// in mask (bit d: neighbour d) — over the same schedule (make_schedule).
// The last of them to finish releases the step, so the count must match.
int hx_exchange_edge_items(int bx, int by, int bz, int mask, unsigned *out) {
    if (bx < 1 || by < 1 || bz < 1 || !out || (mask & ~63)) return HX_E_INVALID;
    const Schedule sc = make_schedule(1, bx + 1, 1, by + 1, 1, bz + 1);
    const long long ntk = sc.ntk, ntj = sc.ntj, nch = sc.nchunks;
    const bool xl = mask & 1, xh = mask & 2, yl = mask & 4, yh = mask & 8, zl = mask & 16,
               zh = mask & 32;
    // edge in some axis = all - edge in no axis (a side's tiles: the first or
    // the last column / row / chunk; both sides may share one when there is one)
    const long long kin = ntk - (zl ? 1 : 0) - (zh && (!zl || ntk > 1) ? 1 : 0);
    const long long jin = ntj - (yl ? 1 : 0) - (yh && (!yl || ntj > 1) ? 1 : 0);
    const long long iin = nch - (xl ? 1 : 0) - (xh && (!xl || nch > 1) ? 1 : 0);
    const long long edge =
        ntk * ntj * nch - std::max(0LL, kin) * std::max(0LL, jin) * std::max(0LL, iin);
    if (edge < 0 || edge > 0xffffffffLL) return HX_E_INVALID;
    *out = (unsigned)edge;
    return 0;
}

// The fused step as ONE sweep: every face of the block is produced and
// consumed by the interior sweep's edge tiles (x / y: the neighbours store
// straight into our ghost planes / rows and we into theirs; z: through the
// slots, as hx_stencil_box_z). flag[d]: our flag from neighbour d (null: no
// neighbour); peer_nxt[d]: neighbour d's next field (x / y only). The box is
// the whole block. Release with hx_exchange_signal after the launch.
int hx_stencil_exchange(const double *cur, double *nxt, int bx, int by, int bz,
                        unsigned long long *res, const unsigned long long *const flag[6],
                        double *const peer_nxt[6], unsigned long long *step,
                        const double *const zin[2], double *const zout[2],
                        unsigned long long *const signal[6], unsigned *counter,
                        unsigned long long timeout_ns, int *err, void *stream) {
    if (!cur || !nxt || bx < 1 || by < 1 || bz < 1 || !step || !flag || !peer_nxt)
        return HX_E_INVALID;
    if (counter && !signal) return HX_E_INVALID;
    if (!tma_eligible(cur, bz)) return HX_E_INVALID;
    if (flag[4] && flag[5] && bz <= TZ) return HX_E_INVALID;  // a tile would hold both z faces
    if (flag[2] && flag[3] && by <= TY) return HX_E_INVALID;  // ... both y faces
    if (flag[0] && flag[1] && bx < 2) return HX_E_INVALID;    // one plane, both x faces
    ZEdge Z;
    memset(&Z, 0, sizeof(Z));
    for (int h = 0; h < 2; ++h) {
        Z.flag[h] = flag[4 + h];
        if (flag[4 + h] && (!zin || !zout || !zin[h] || !zout[h])) return HX_E_INVALID;
        Z.zin[h] = flag[4 + h] ? zin[h] : nullptr;
        Z.zout[h] = flag[4 + h] ? zout[h] : nullptr;
    }
    const long long sx = (long long)(by + 2) * (bz + 2), sy = bz + 2;
    const long long span[2] = {sx * bx, sy * by};
    for (int d = 0; d < 4; ++d) {
        Z.xyflag[d] = flag[d];
        if (!flag[d]) continue;
        if (!peer_nxt[d]) return HX_E_INVALID;
        const long long shift = (d & 1) ? -span[d >> 1] : span[d >> 1];  // our face -> its ghost
        Z.xydelta[d] = ((long long)(intptr_t)peer_nxt[d] - (long long)(intptr_t)nxt) /
                           (long long)sizeof(double) + shift;
    }
    Z.bx = bx;
    Z.step = step;
    Z.timeout_ns = timeout_ns;
    Z.err = err;
    if (counter) {
        int mask = 0;
        for (int d = 0; d < 6; ++d) mask |= flag[d] ? 1 << d : 0;
        if (int rc = hx_exchange_edge_items(bx, by, bz, mask, &Z.edge_items)) return rc;
        if (Z.edge_items == 0) return HX_E_INVALID;  // no neighbour: nothing would release
        Z.edge_counter = counter;
        for (int d = 0; d < 6; ++d) Z.sig[d] = signal[d];
    }
    g_last_variant = 1;
    return launch_tma(cur, nxt, bx, by, bz, 1, bx + 1, 1, by + 1, 1, bz + 1, res,
                      (cudaStream_t)stream, &Z);
}

struct Flags6 {
    unsigned long long *f[6];
};

// After a step's sweep (and boundary kernel, if any), stream-ordered behind
// them: threads 0-5 release their flag = *step + 2 in parallel (each
// st.release.sys is cumulative over the sweep's peer stores, which precede
// this launch on the stream); then *step += 1.
__global__ void signal_flags_kernel(Flags6 F, unsigned long long *step, const int *err) {
    const unsigned long long v = *(volatile unsigned long long *)step + 2;
    const bool healthy = !err || *(volatile const int *)err == 0;
    if (threadIdx.x < 6 && F.f[threadIdx.x] && healthy) hx::st_release_sys(F.f[threadIdx.x], v);
    __syncthreads();  // every thread has read *step
    if (threadIdx.x == 0) *step = v - 1;
}

int hx_exchange_signal(unsigned long long *const flag[6], unsigned long long *step, const int *err,
                       void *stream) {
    if (!flag || !step) return HX_E_INVALID;
    Flags6 F;
    for (int d = 0; d < 6; ++d) F.f[d] = flag[d];
    signal_flags_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(F, step, err);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_zsignal(unsigned long long *const flag[2], unsigned long long *step, const int *err,
               void *stream) {
    if (!flag) return HX_E_INVALID;
    unsigned long long *f6[6] = {nullptr, nullptr, nullptr, nullptr, flag[0], flag[1]};
    return hx_exchange_signal(f6, step, err, stream);
}

int hx_preload_halo_kernels();  // hx_halo.cu

// See hx_preload_halo_kernels: the exchange's spinning kernels, loaded up
// front on the current device (the stencil variants are launched alone or
// concurrently with the fused shell, which needs no other kernel to finish).
int hx_preload() {
    if (const char *e = getenv("HX_L2_FETCH"))  // measurement knob: L2 fetch granularity (bytes)
        HX_TRY(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(e)));
    cudaFuncAttributes a;
    HX_TRY(cudaFuncGetAttributes(&a, (const void *)shell_put_kernel));
    HX_TRY(cudaFuncGetAttributes(&a, (const void *)face_tma_kernel));
    HX_TRY(cudaFuncGetAttributes(&a, (const void *)signal_flags_kernel));
    HX_TRY(cudaFuncGetAttributes(&a, (const void *)fill_kernel));
    return hx_preload_halo_kernels();
}

int hx_shell_put(const double *cur, double *nxt, int bx, int by, int bz, int nbox,
                 const int *boxes, double *const remote[6], unsigned long long *const wait_flag[6],
                 unsigned long long wait_value, unsigned long long *const signal_flag[6],
                 unsigned long long signal_value, unsigned int *counter,
                 unsigned long long timeout_ns, int *err, unsigned long long *res,
                 unsigned long long *step, void *stream) {
    return hx_shell_put_z(cur, nxt, bx, by, bz, nbox, boxes, remote, wait_flag, wait_value,
                          signal_flag, signal_value, counter, timeout_ns, err, res, step, nullptr,
                          nullptr, stream);
}

int hx_shell_put_z(const double *cur, double *nxt, int bx, int by, int bz, int nbox,
                   const int *boxes, double *const remote[6], unsigned long long *const wait_flag[6],
                   unsigned long long wait_value, unsigned long long *const signal_flag[6],
                   unsigned long long signal_value, unsigned int *counter,
                   unsigned long long timeout_ns, int *err, unsigned long long *res,
                   unsigned long long *step, const double *const zin[2], double *const zout[2],
                   void *stream) {
    if (!cur || !nxt || !counter || bx < 1 || by < 1 || bz < 1 || nbox < 0 || nbox > 6)
        return HX_E_INVALID;
    if (nbox > 0 && !boxes) return HX_E_INVALID;
    ShellJob J;
    memset(&J, 0, sizeof(J));
    const long long sx = (long long)(by + 2) * (bz + 2), sy = bz + 2;
    const long long span[3] = {sx * bx, sy * by, (long long)bz};  // block extent per axis
    const int ext[3] = {bx, by, bz};
    for (int d = 0; d < 6; ++d) {
        J.remote[d] = remote ? remote[d] : nullptr;
        J.wait[d] = wait_flag ? wait_flag[d] : nullptr;
        J.signal[d] = signal_flag ? signal_flag[d] : nullptr;
        // our plane 1 (d even) is the neighbour's ghost plane ext+1, our
        // plane ext (d odd) its ghost plane 0
        J.face[d] = (d & 1) ? ext[d >> 1] : 1;
        J.shift[d] = (d & 1) ? -span[d >> 1] : span[d >> 1];
    }
    for (int h = 0; h < 2; ++h) {
        // a z slot only together with that z neighbour
        J.zin[h] = (zin && J.remote[4 + h]) ? zin[h] : nullptr;
        J.zout[h] = (zout && J.remote[4 + h]) ? zout[h] : nullptr;
    }
    J.rows[0] = 0;
    long long n = 0;
    for (int q = 0; q < nbox; ++q) {
        const int *x = boxes + 6 * q;
        if (x[0] < 1 || x[2] < 1 || x[4] < 1 || x[1] > bx + 1 || x[3] > by + 1 || x[5] > bz + 1)
            return HX_E_INVALID;
        const int ni = std::max(0, x[1] - x[0]), nj = std::max(0, x[3] - x[2]),
                  nk = std::max(0, x[5] - x[4]);
        if ((long long)ni * nj * nk == 0) continue;
        for (int e = 0; e < 6; ++e) J.box[J.nbox][e] = x[e];
        const long long rows = nk > 1 ? (long long)ni * nj : ni;
        if (J.rows[J.nbox] + rows > 0x7fffffffLL) return HX_E_INVALID;
        J.rows[J.nbox + 1] = J.rows[J.nbox] + (int)rows;
        n += (long long)ni * nj * nk;
        ++J.nbox;
    }
    // x / y face slabs only (no z column) on a TMA-describable block: the
    // face kernel (HX_SHELL_FACE_TMA=0 keeps the per-row kernel, for A/B)
    static int face_tma = -1;
    if (face_tma < 0) {
        const char *e = getenv("HX_SHELL_FACE_TMA");
        face_tma = e ? atoi(e) : 1;
    }
    // x / y slabs over whole rows and z slabs at k = 1 / bz; z neighbours only
    // through their slots; a row then lies on at most two x / y faces
    bool faces_only = face_tma && J.nbox > 0 && tma_eligible(cur, bz) &&
                      ((uintptr_t)nxt & 15) == 0 && (!J.remote[4] || J.zin[0]) &&
                      (!J.remote[5] || J.zin[1]) && bx >= 2 && by >= 2 && bz >= 2;
    for (int q = 0; q < J.nbox && faces_only; ++q) {
        const int *x = J.box[q];
        const bool xslab = x[1] - x[0] == 1 && x[4] == 1 && x[5] == bz + 1;
        const bool yslab = x[3] - x[2] == 1 && x[1] - x[0] > 1 && x[4] == 1 && x[5] == bz + 1;
        const bool zslab = x[5] - x[4] == 1 && (x[4] == 1 || x[4] == bz) && x[1] - x[0] >= 1 &&
                           x[3] - x[2] > 1;
        faces_only = xslab || yslab || zslab;
    }
    if (faces_only) {
        FaceJob F;
        memset(&F, 0, sizeof(F));
        F.nbox = J.nbox;
        F.k0 = J.box[0][4];
        F.k1 = J.box[0][5];
        F.ntk = (bz + 2 + FK - 1) / FK;  // tiles over padded k [0, bz + 2), starting at even k
        F.tiles[0] = 0;
        for (int q = 0; q < J.nbox; ++q) {
            const int *x = J.box[q];
            long long t;
            if (x[5] - x[4] == 1) {  // z slab
                F.axis[q] = 2;
                F.pos[q] = x[4];
                F.lo[q] = x[0];
                F.hi[q] = x[1];
                F.clo[q] = x[2];
                F.chi[q] = x[3];
                t = (long long)((x[1] - x[0] + FR - 1) / FR) * ((x[3] - x[2] + ZTJ - 1) / ZTJ);
            } else {
                const bool xslab = x[1] - x[0] == 1;
                F.axis[q] = xslab ? 0 : 1;
                F.pos[q] = xslab ? x[0] : x[2];
                F.lo[q] = xslab ? x[2] : x[0];
                F.hi[q] = xslab ? x[3] : x[1];
                t = (long long)((F.hi[q] - F.lo[q] + FR - 1) / FR) * F.ntk;
            }
            if (F.tiles[q] + t > 0x7fffffffLL) return HX_E_INVALID;
            F.tiles[q + 1] = F.tiles[q] + (int)t;
        }
        for (int h = 0; h < 2; ++h) {
            F.zin[h] = J.zin[h];
            F.zout[h] = J.zout[h];
        }
        for (int d = 0; d < 6; ++d) {
            F.remote[d] = J.remote[d];
            F.shift[d] = J.shift[d];
            F.face[d] = J.face[d];
            F.wait[d] = J.wait[d];
            F.signal[d] = J.signal[d];
        }
        CUtensorMap mx, my, mz;
        static int zpromo = -1;  // z-tile L2 promotion (HX_FACE_ZPROMO, 0..3; default none)
        if (zpromo < 0) {
            const char *e = getenv("HX_FACE_ZPROMO");
            zpromo = e ? std::min(3, std::max(0, atoi(e))) : 0;
        }
        if (int rc = face_map_for(cur, bx, by, bz, FBK, FBR, 3, l2_promotion(), &mx)) return rc;
        if (int rc = face_map_for(cur, bx, by, bz, FBK, 3, FBR, l2_promotion(), &my)) return rc;
        if (int rc = face_map_for(cur, bx, by, bz, ZBK, ZBJ, ZBI, zpromo, &mz)) return rc;
        static unsigned long long attr_set = 0;
        if (int rc = ensure_smem(face_tma_kernel, FACE_SMEM, attr_set)) return rc;
        static int face_bulk = -1;  // bulk-copy row segments to the peer (HX_FACE_BULK=0: plain stores)
        if (face_bulk < 0) {
            const char *e = getenv("HX_FACE_BULK");
            face_bulk = e ? atoi(e) : 1;
        }
        static int fmult = 0;
        if (!fmult) {
            const char *e = getenv("HX_FACE_GRID_MULT");  // persistent CTAs per SM (tuning)
            fmult = e && atoi(e) > 0 ? atoi(e) : 3;
        }
        const unsigned grid = (unsigned)std::max(1, std::min(F.tiles[F.nbox], fmult * num_sms()));
        if (F.tiles[F.nbox] > 0) {
            face_tma_kernel<<<grid, 256, FACE_SMEM, (cudaStream_t)stream>>>(
                mx, my, mz, nxt, by, bz, F, face_bulk, wait_value, signal_value, counter, timeout_ns,
                err, res,
                step);
            HX_LAUNCH_CHECK();
            return 0;
        }
    }
    static int mult = 0;
    if (!mult) {
        const char *e = getenv("HX_SHELL_GRID_MULT");  // CTAs per SM (tuning)
        mult = e && atoi(e) > 0 ? atoi(e) : 4;  // 4: 0.112 -> 0.076 ms concurrent shell at 1536^2, step unchanged
    }
    const unsigned grid = (unsigned)std::max<long long>(
        1, std::min<long long>(std::min<long long>((n + 255) / 256, J.rows[J.nbox]),
                               (long long)mult * num_sms()));
    shell_put_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        cur, nxt, by, bz, J, wait_value, signal_value, counter, timeout_ns, err, res, step);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_persist_run(double *const field[2], double *const peer[12], int bx, int by, int bz,
                   int parity, unsigned long long it0, int iters,
                   unsigned long long *const wait_flag[6], unsigned long long *const signal_flag[6],
                   const double *const zin[4], double *const zout[4], unsigned *barrier,
                   int max_ctas, unsigned long long timeout_ns, int *err, void *stream) {
    if (!field || !field[0] || !field[1] || !barrier || bx < 1 || by < 1 || bz < 1 ||
        iters < 0 || (parity & ~1) || (long long)bx * by * bz > (1LL << 31))
        return HX_E_INVALID;
    if (iters == 0) return 0;
    PersistJob J;
    memset(&J, 0, sizeof(J));
    const long long sx = (long long)(by + 2) * (bz + 2), sy = bz + 2;
    const long long span[3] = {sx * bx, sy * by, (long long)bz};
    const int ext[3] = {bx, by, bz};
    J.field[0] = field[0];
    J.field[1] = field[1];
    for (int d = 0; d < 6; ++d) {
        J.peer[d][0] = peer ? peer[2 * d] : nullptr;
        J.peer[d][1] = peer ? peer[2 * d + 1] : nullptr;
        J.wait[d] = wait_flag ? wait_flag[d] : nullptr;
        J.signal[d] = signal_flag ? signal_flag[d] : nullptr;
        J.face[d] = (d & 1) ? ext[d >> 1] : 1;
        J.shift[d] = (d & 1) ? -span[d >> 1] : span[d >> 1];
    }
    for (int q = 0; q < 2; ++q)
        for (int h = 0; h < 2; ++h) {  // only with that z neighbour
            J.zin[q][h] = (zin && J.peer[4 + h][0]) ? zin[2 * q + h] : nullptr;
            J.zout[q][h] = (zout && J.peer[4 + h][0]) ? zout[2 * q + h] : nullptr;
        }
    // every CTA must be resident for the grid barriers: one CTA of 256
    // threads per SM at most (the caller may lower it for blocks sharing a GPU)
    const long long cells = (long long)bx * by * bz;
    long long want = (cells + 1023) / 1024;
    int grid = (int)std::max<long long>(1, std::min<long long>(want, num_sms()));
    if (max_ctas > 0) grid = std::min(grid, max_ctas);
    persist_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(J, bx, by, bz, parity, it0, iters,
                                                           barrier, barrier + 1, timeout_ns, err);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_stencil(const double *cur, double *nxt, int bx, int by, int bz, unsigned long long *res,
               void *stream) {
    return hx_stencil_box(cur, nxt, bx, by, bz, 1, bx + 1, 1, by + 1, 1, bz + 1, res, stream);
}

int hx_div6_check(const double *in, size_t n, unsigned long long *mismatches, void *stream) {
    if (!in || !mismatches) return HX_E_INVALID;
    if (!n) return 0;
    div6_check_kernel<<<4 * num_sms(), 256, 0, (cudaStream_t)stream>>>(in, n, mismatches);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_init_block(double *field, int bx, int by, int bz, int hot_wall, double hot,
                  double background, double fill, void *stream) {
    if (!field || bx < 1 || by < 1 || bz < 1) return HX_E_INVALID;
    init_block_kernel<<<4 * num_sms(), 256, 0, (cudaStream_t)stream>>>(field, bx, by, bz, hot_wall,
                                                                       hot, background, fill);
    HX_LAUNCH_CHECK();
    return 0;
}

int hx_fill_f64(double *dst, size_t n, double value, void *stream) {
    if (!dst) return HX_E_INVALID;
    if (!n) return 0;
    fill_kernel<<<4 * num_sms(), 256, 0, (cudaStream_t)stream>>>(dst, n, value);
    HX_LAUNCH_CHECK();
    return 0;
}

}  // extern "C"
