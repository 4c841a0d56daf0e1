// Probe: does cp.async.bulk.tensor (SWIZZLE_NONE) accept a shared-memory
// destination that is 16-byte but not 128-byte aligned?
// nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tma_align probe_tma_align.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int off_bytes) {
    __shared__ __align__(1024) unsigned char sm[8192];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + off_bytes);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(16 * 8 * 8));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(&map), "r"(0), "r"(0), "r"(b)
                     : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(b) : "memory");
    }
    __syncthreads();
    const double* s = reinterpret_cast<const double*>(sm + off_bytes);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) out[i] = s[i];
}

int main() {
    double* g;
    double* o;
    cudaMalloc(&g, 64 * 64 * 8);
    cudaMalloc(&o, 128 * 8);
    std::vector<double> h(64 * 64);
    for (int i = 0; i < 64 * 64; ++i) h[i] = i;
    cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[2] = {64, 64};
    cuuint64_t strides[1] = {64 * 8};
    cuuint32_t box[2] = {8, 16}, es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int off : {0, 128, 64, 16}) {
        cudaMemset(o, 0, 128 * 8);
        k<<<1, 128>>>(map, o, off);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> r(128);
        cudaMemcpy(r.data(), o, 128 * 8, cudaMemcpyDeviceToHost);
        bool ok = e == cudaSuccess;
        for (int row = 0; row < 16; ++row)
            for (int l = 0; l < 8; ++l) ok &= r[row * 8 + l] == h[row * 64 + l];
        printf("dst offset %4d B: %s (%s)\n", off, ok ? "OK" : "WRONG", cudaGetErrorString(e));
        if (e != cudaSuccess) break;
    }
    return 0;
}
