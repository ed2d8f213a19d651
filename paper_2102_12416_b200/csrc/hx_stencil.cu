// Jacobi3D 6-neighbour relaxation for sm_100a.
//
// Reference: _BlockCore.update, cl/jacobi3d.py:165-173 (and the sequential
// oracle's identical sweep + residual, 192-198):
//   nxt[i,j,k] = (((((c[i-1,j,k] + c[i+1,j,k]) + c[i,j-1,k]) + c[i,j+1,k])
//                 + c[i,j,k-1]) + c[i,j,k+1]) / 6.0
// The adds are issued in exactly this order and the division is the IEEE
// correctly rounded div.rn.f64 (never a multiply by 1/6), so results are
// bit-identical to numpy. Ghost cells of nxt are never written.
//
// Primary kernel (HBM-bound, 16 algorithmic bytes per cell): a 2.5-D
// streaming sweep. Each CTA owns a TY x TZ tile of the (j,k) plane and
// marches along x (the slowest axis) over a chunk of planes. Every padded
// plane tile (TY+2) x (TZ+2) is fetched exactly once by a TMA bulk-tensor
// load into an S-stage shared-memory ring guarded by mbarriers, so each
// input cell crosses HBM once (plus the thin tile halos, which L2 serves);
// the x-neighbours come from the adjacent ring stages and the y/z
// neighbours from the current stage. Outputs are stored straight from
// registers with coalesced 8-byte stores. The residual max|nxt-cur| reuses
// the centre value already in shared memory (no extra traffic) and is
// reduced warp -> CTA -> one atomicMax on the uint64 bit pattern (valid
// for non-negative doubles).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "hx_internal.cuh"

namespace {

constexpr int TY = 32;           // tile rows (j)
constexpr int TZ = 64;           // tile columns (k)
constexpr int NSTAGE = 6;        // shared-memory ring depth (planes)
constexpr int THREADS = 256;     // 8 warps; warp w owns rows w, w+8, w+16, w+24
constexpr int ROWS_PER_WARP = TY / (THREADS / 32);
constexpr int BOX_Y = TY + 2, BOX_Z = TZ + 2;
constexpr unsigned STAGE_BYTES = BOX_Y * BOX_Z * sizeof(double);             // 17952
constexpr unsigned STAGE_STRIDE = (STAGE_BYTES + 127) / 128 * 128;           // TMA: 128 B aligned
constexpr size_t SMEM_BYTES = (size_t)NSTAGE * STAGE_STRIDE + NSTAGE * sizeof(uint64_t);

int g_variant = 0;     // 0 auto, 1 TMA, 2 generic
int g_last_variant = 0;
int g_chunk = 0;       // planes per CTA work item, 0 = auto
int g_num_sms = 0;

__device__ __forceinline__ double relax(double xm, double xp, double ym, double yp, double zm,
                                        double zp) {
    double t = __dadd_rn(xm, xp);
    t = __dadd_rn(t, ym);
    t = __dadd_rn(t, yp);
    t = __dadd_rn(t, zm);
    t = __dadd_rn(t, zp);
    return __ddiv_rn(t, 6.0);
}

__device__ __forceinline__ void cta_max_to_global(double worst, unsigned long long *res) {
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nwarps = (int)(blockDim.x * blockDim.y * blockDim.z) >> 5;
    const int lane = tid & 31, warp = tid >> 5;
    if (lane == 0) red[warp] = worst;
    __syncthreads();
    if (tid == 0) {
        double w = red[0];
        for (int q = 1; q < nwarps; ++q) w = fmax(w, red[q]);
        if (w > 0.0) atomicMax(res, (unsigned long long)__double_as_longlong(w));
    }
}

// ------------------------------------------------------- TMA pipeline ----
// Work item = (tile j, tile k, x chunk). Box in interior coordinates:
// [i0,i1) x [j0,j1) x [k0,k1).
__global__ void __launch_bounds__(THREADS, 2)
stencil_tma_kernel(const __grid_constant__ CUtensorMap map, double *__restrict__ nxt, int by,
                   int bz, int i0, int i1, int j0, int j1, int k0, int k1, int ntj, int ntk,
                   int chunk, unsigned long long *res) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + NSTAGE * STAGE_STRIDE);

    int item = blockIdx.x;
    const int tk = item % ntk;
    item /= ntk;
    const int tj = item % ntj;
    const int c = item / ntj;
    const int jb = j0 + tj * TY, kb = k0 + tk * TZ;
    const int ib = i0 + c * chunk;
    const int ie = min(ib + chunk, i1);
    const int nplanes = ie - ib + 2;  // padded planes ib-1 .. ie

    if (threadIdx.x == 0) {
        hx::prefetch_tmap(&map);
        for (int s = 0; s < NSTAGE; ++s) hx::mbar_init(&bar[s], 1);
        hx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int pre = min(NSTAGE, nplanes);
        for (int p = 0; p < pre; ++p) {
            hx::mbar_expect_tx(&bar[p], STAGE_BYTES);
            hx::tma_load_3d(smem + p * STAGE_STRIDE, &map, kb - 1, jb - 1, ib - 1 + p, &bar[p]);
        }
    }

    const hx::Geom g(by, bz);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bool kok[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) kok[h] = kb + lane + 32 * h < k1;
    double worst = 0.0;

    hx::mbar_wait(&bar[0], 0);
    hx::mbar_wait(&bar[1 % NSTAGE], 0);
    for (int q = 1; q <= nplanes - 2; ++q) {
        const int sm = (q - 1) % NSTAGE, s0 = q % NSTAGE, sp = (q + 1) % NSTAGE;
        hx::mbar_wait(&bar[sp], ((q + 1) / NSTAGE) & 1);
        const double *pm = reinterpret_cast<const double *>(smem + sm * STAGE_STRIDE);
        const double *p0 = reinterpret_cast<const double *>(smem + s0 * STAGE_STRIDE);
        const double *pp = reinterpret_cast<const double *>(smem + sp * STAGE_STRIDE);
        const int i = ib - 1 + q;
#pragma unroll
        for (int rr = 0; rr < ROWS_PER_WARP; ++rr) {
            const int r = warp + rr * (THREADS / 32);
            const int j = jb + r;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int kk = lane + 32 * h;
                const int ctr = (r + 1) * BOX_Z + kk + 1;
                const double v = relax(pm[ctr], pp[ctr], p0[ctr - BOX_Z], p0[ctr + BOX_Z],
                                       p0[ctr - 1], p0[ctr + 1]);
                if (j < j1 && kok[h]) {
                    nxt[g.at(i, j, kb + kk)] = v;
                    if (res) worst = fmax(worst, fabs(__dsub_rn(v, p0[ctr])));
                }
            }
        }
        __syncthreads();  // every thread is done with stage sm
        if (threadIdx.x == 0) {
            const int p = q - 1 + NSTAGE;
            if (p < nplanes) {
                hx::mbar_expect_tx(&bar[sm], STAGE_BYTES);
                hx::tma_load_3d(smem + sm * STAGE_STRIDE, &map, kb - 1, jb - 1, ib - 1 + p, &bar[sm]);
            }
        }
    }
    if (res) cta_max_to_global(worst, res);
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
    double worst = 0.0;
    if (k < k1 && j < j1) {
        const size_t c = g.at(i, j, k);
        const size_t sx = (size_t)g.py * g.pz, sy = g.pz;
        const double v = relax(__ldg(cur + c - sx), __ldg(cur + c + sx), __ldg(cur + c - sy),
                               __ldg(cur + c + sy), __ldg(cur + c - 1), __ldg(cur + c + 1));
        nxt[c] = v;
        if (res) worst = fabs(__dsub_rn(v, __ldg(cur + c)));
    }
    if (res) cta_max_to_global(worst, res);
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

__global__ void fill_kernel(double *p, size_t n, double v) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
         q += (size_t)gridDim.x * blockDim.x)
        p[q] = v;
}

// ------------------------------------------------------ host helpers -----
std::mutex g_map_mu;
std::map<std::tuple<const void *, int, int, int>, CUtensorMap> g_maps;

int tensor_map_for(const double *cur, int bx, int by, int bz, CUtensorMap *out) {
    auto key = std::make_tuple((const void *)cur, bx, by, bz);
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
    cuuint32_t box[3] = {BOX_Z, BOX_Y, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMap m;
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void *)cur, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return HX_E_TMA;
    std::lock_guard<std::mutex> lk(g_map_mu);
    if (g_maps.size() > 256) g_maps.clear();
    g_maps[key] = m;
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

int launch_tma(const double *cur, double *nxt, int bx, int by, int bz, int i0, int i1, int j0,
               int j1, int k0, int k1, unsigned long long *res, cudaStream_t st) {
    CUtensorMap map;
    int rc = tensor_map_for(cur, bx, by, bz, &map);
    if (rc) return rc;
    static bool attr_set = false;
    if (!attr_set) {
        HX_TRY(cudaFuncSetAttribute(stencil_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SMEM_BYTES));
        attr_set = true;
    }
    const int ni = i1 - i0, nj = j1 - j0, nk = k1 - k0;
    const int ntj = (nj + TY - 1) / TY, ntk = (nk + TZ - 1) / TZ;
    int chunk = g_chunk;
    if (chunk <= 0) {
        // ~24 waves of 2 CTAs/SM keeps the tail short; chunk-boundary planes
        // are re-read once per chunk (2/chunk extra read traffic).
        const long target = 24L * 2 * num_sms();
        const long tiles = (long)ntj * ntk;
        chunk = (int)std::max<long>(8, ((long)ni * tiles + target - 1) / target);
    }
    chunk = std::min(chunk, ni);
    const int nchunks = (ni + chunk - 1) / chunk;
    const long items = (long)ntj * ntk * nchunks;
    if (items > 0x7fffffffL) return HX_E_INVALID;
    stencil_tma_kernel<<<(unsigned)items, THREADS, SMEM_BYTES, st>>>(
        map, nxt, by, bz, i0, i1, j0, j1, k0, k1, ntj, ntk, chunk, res);
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
    if (want == 0) want = tma_eligible(cur, bz) ? 1 : 2;
    if (want == 1 && !tma_eligible(cur, bz)) return HX_E_INVALID;
    if (want == 1) {
        int rc = launch_tma(cur, nxt, bx, by, bz, i0, i1, j0, j1, k0, k1, res, st);
        if (rc == 0) {
            g_last_variant = 1;
            return 0;
        }
        if (g_variant == 1) return rc;  // forced: report, do not fall back
    }
    g_last_variant = 2;
    return launch_generic(cur, nxt, by, bz, i0, i1, j0, j1, k0, k1, res, st);
}

int hx_stencil(const double *cur, double *nxt, int bx, int by, int bz, unsigned long long *res,
               void *stream) {
    return hx_stencil_box(cur, nxt, bx, by, bz, 1, bx + 1, 1, by + 1, 1, bz + 1, res, stream);
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
