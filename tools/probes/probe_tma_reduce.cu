// Probe: does the TMA engine add fp64 into global memory?
//   (1) cp.reduce.async.bulk .add.f64 (contiguous)
//   (2) cp.reduce.async.bulk.tensor .add on a FLOAT64 tensor map, 128B swizzle
// nvcc -gencode arch=compute_100a,code=sm_100a -o probe probe_tma_reduce.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void k_bulk(double* g) {
    __shared__ __align__(128) double s[256];
    s[threadIdx.x] = threadIdx.x + 0.5;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(g), "r"(sa), "r"(2048) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

__global__ void k_tensor(const __grid_constant__ CUtensorMap map) {
    __shared__ __align__(1024) double s[16 * 16];   // box 16 x 16, 128B swizzle
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = i;   // swizzled order irrelevant: all 1s test below
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
        asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&map), "r"(sa), "r"(0), "r"(0) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    double* g;
    cudaMalloc(&g, 1 << 16);
    std::vector<double> h(256, 1.0);
    cudaMemcpy(g, h.data(), 2048, cudaMemcpyHostToDevice);
    k_bulk<<<1, 256>>>(g);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h.data(), g, 2048, cudaMemcpyDeviceToHost);
    bool ok = e == cudaSuccess;
    for (int i = 0; i < 256; ++i) ok &= h[i] == 1.0 + i + 0.5;
    printf("bulk add.f64: %s (%s)\n", ok ? "OK" : "WRONG", cudaGetErrorString(e));

    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap map;
    cuuint64_t dims[2] = {16, 64};
    cuuint64_t strides[1] = {16 * 8};
    cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    std::vector<double> z(16 * 64, 2.0);
    cudaMemcpy(g, z.data(), z.size() * 8, cudaMemcpyHostToDevice);
    k_tensor<<<1, 256>>>(map);
    e = cudaDeviceSynchronize();
    cudaMemcpy(z.data(), g, z.size() * 8, cudaMemcpyDeviceToHost);
    ok = cr == CUDA_SUCCESS && e == cudaSuccess;
    for (int i = 0; i < 256; ++i) ok &= z[i] == 3.0;
    for (int i = 256; i < 1024; ++i) ok &= z[i] == 2.0;
    printf("tensor add f64 (128B swizzle): %s (encode %d, %s)\n", ok ? "OK" : "WRONG", (int)cr,
           cudaGetErrorString(e));
    return 0;
}
