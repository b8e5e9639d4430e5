// Copy micro (dev tool): the fused K1's data movement without the FNV chain, to
// price its store path. 2 GiB -> 2 GiB, 148 CTAs x 16 warps, warp task = 32
// pages x 4 KiB, one 8 KiB stage per warp (256 B of each page, cp.async in,
// 128B-swizzled like a TMA box), then the stage goes out either as lane stores
// (LDS + STG.128, the current kernel) or as two TMA tensor stores of 16 rows x
// 256 B (one per 64 KiB chunk) issued by one lane.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int kWarps = 16;
constexpr int kStage = 32 * 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// unit u (16 B) of row j: half u >> 3, chunk (u & 7) ^ ((2 j + half) & 7)
__device__ __forceinline__ uint32_t sw_off(uint32_t j, uint32_t u) {
  const uint32_t h = u >> 3;
  return j * 256 + h * 128 + ((((u & 7) ^ ((2 * j + h) & 7))) << 4);
}

template <bool TMA>
__global__ void __launch_bounds__(kWarps * 32, 1)
k(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t nbytes,
  const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* buf = smem + warp * kStage;
  const uint32_t bu = smem_u32(buf);
  const size_t ntasks = nbytes / (32ull * 4096);
  const size_t nw = size_t(gridDim.x) * kWarps;
  const uint32_t u = lane & 15, q = lane >> 4;  // 16 lanes per page, 2 pages per instr
  for (size_t t = size_t(blockIdx.x) * kWarps + warp; t < ntasks; t += nw) {
    const size_t base = t * 32 * 4096;
    for (int s = 0; s < 16; ++s) {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const uint32_t j = kk * 2 + q;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(bu + sw_off(j, u)),
                     "l"(src + base + size_t(j) * 4096 + s * 256 + u * 16)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      if (TMA) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const uint64_t row0 = base / 4096;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int32_t c0 = 0, c1 = 2 * s, c2 = int32_t(row0 + 16 * c);
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                ::"l"(&tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bu + c * 16 * 256)
                : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const uint32_t j = kk * 2 + q;
          const uint4 v = *reinterpret_cast<const uint4*>(buf + sw_off(j, u));
          __stcs(reinterpret_cast<uint4*>(dst + base + size_t(j) * 4096 + s * 256 + u * 16), v);
        }
        __syncwarp();
      }
    }
  }
  if (TMA && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t n = 2ull << 30;
  uint8_t *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  cudaMemset(a, 7, n);
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  EncodeFn encode = reinterpret_cast<EncodeFn>(fn);
  CUtensorMap tm;
  const cuuint64_t dims[3] = {128, 32, n / 4096};
  const cuuint64_t strides[2] = {128, 4096};
  const cuuint32_t box[3] = {128, 2, 16};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, b, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return 1; }
  const int smem = kWarps * kStage;
  cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    float best = 1e9;
    for (int rep = 0; rep < 8; ++rep) {
      cudaMemset(b, 0, 4096);
      cudaEventRecord(e0);
      kern<<<148, kWarps * 32, smem>>>(a, b, n, tm);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    // spot check
    uint8_t h[4096];
    cudaMemcpy(h, b + n - 4096, 4096, cudaMemcpyDeviceToHost);
    printf("%-20s %7.3f ms  %7.1f GB/s (R+W)  %s  last page byte %d\n", name, best,
           2.0 * n / best / 1e6, cudaGetErrorString(e), int(h[100]));
  };
  for (int i = 0; i < 2; ++i) {
    run(k<false>, "LDS + STG.128");
    run(k<true>, "TMA tensor store");
  }
  return 0;
}
