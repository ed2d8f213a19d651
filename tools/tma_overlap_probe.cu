// Probe: can a TMA tensor map describe an odd-pitch padded array through a
// row-pair / plane-pair view whose dim-0 extent overlaps the next dims?
//   element (i, j, k) = base + (i>>1)*2*plane + (j>>1)*2*pz + [k + (j&1)*pz + (i&1)*plane]
// dims {D0, ceil(py/2), ceil(px/2)}, strides {2*pz*8, 2*plane*8} (16-byte
// multiples whatever the parities), dim-0 coordinate = k + (j&1)*pz + (i&1)*plane.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o gpurun_out/tma_probe tools/tma_overlap_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void probe_kernel(const __grid_constant__ CUtensorMap map, double *out, int c0, int c1,
                             int c2, int boxw, int boxh) {
    __shared__ __align__(128) double tile[17 * 72];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                     "r"(boxw * boxh * 8) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"((unsigned)__cvta_generic_to_shared(tile)),
            "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(b) : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(b)
        : "memory");
    for (int t = threadIdx.x; t < boxw * boxh; t += blockDim.x) out[t] = tile[t];
}

int main() {
    const int bx = 9, by = 11, bz = 29;  // every parity odd
    const long pz = bz + 2, py = by + 2, px = bx + 2, plane = py * pz, n = px * plane;
    std::vector<double> h(n);
    for (long e = 0; e < n; ++e) h[e] = (double)e;
    double *d, *o;
    cudaMalloc(&d, n * 8 + 4096);
    cudaMalloc(&o, 17 * 72 * 8);
    cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q);
    const int boxw = 16, boxh = 4;  // 14 wanted + 1 shift, rounded to 16 B rows
    cuuint64_t dims[3] = {(cuuint64_t)(2 * pz + plane), (cuuint64_t)((py + 1) / 2), (cuuint64_t)((px + 1) / 2)};
    cuuint64_t strides[2] = {(cuuint64_t)(2 * pz * 8), (cuuint64_t)(2 * plane * 8)};
    cuuint32_t box[3] = {(cuuint32_t)boxw, (cuuint32_t)boxh, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUtensorMap map;
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    if (r != CUDA_SUCCESS) return 1;
    int bad = 0, cases = 0;
    for (int i = 0; i < px; ++i)
        for (int j = 0; j + 2 * (boxh - 1) < py; ++j)
            for (int k = 0; k + 14 <= pz; k += 3) {
                const int want0 = k + (j & 1) * (int)pz + (i & 1) * (int)plane;
                const int sh = want0 & 1;  // box rows must start 16-byte aligned
                probe_kernel<<<1, 64>>>(map, o, want0 - sh, j >> 1, i >> 1, boxw, boxh);
                std::vector<double> got(boxw * boxh);
                cudaMemcpy(got.data(), o, boxw * boxh * 8, cudaMemcpyDeviceToHost);
                for (int rr = 0; rr < boxh; ++rr)
                    for (int c = 0; c < 14; ++c) {
                        const long want = i * plane + (j + 2 * rr) * pz + k + c;
                        bad += got[rr * boxw + c + sh] != (double)want;
                    }
                ++cases;
            }
    printf("cases %d, mismatches %d, err %s\n", cases, bad, cudaGetErrorString(cudaDeviceSynchronize()));
    return bad != 0;
}
