// The fused K1 DRAM pattern (32 pages x 256-B segments per step, 4 KiB page pitch, read then
// written to the same offsets of a staging image) moved by TMA 2D tensor loads and stores
// (box 32 rows x 128 B, two per segment), vs the LDG/STG version (pattern_bw2: 5.96 TB/s).
#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int ST, int SEGB>
__global__ void __launch_bounds__(32) k(const __grid_constant__ CUtensorMap src, const __grid_constant__ CUtensorMap dst, int ntasks) {
  constexpr int NB = SEGB / 128, STEP = NB * 4096;  // boxes per segment, bytes per step
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[ST];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < ST; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int spt = 4096 / SEGB;  // steps per task
  const long total = (long)((ntasks - blockIdx.x + gridDim.x - 1) / gridDim.x) * spt;
  auto coords = [&](long it, int& x, int& y) {
    const long t = blockIdx.x + (it / spt) * gridDim.x;
    x = int(it % spt) * SEGB;
    y = int(t * 32);
  };
  uint32_t ph[ST] = {};
  long issued = 0;
  auto load = [&](long it) {
    const int k = int(it % ST);
    int x, y;
    coords(it, x, y);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[k])), "r"(STEP));
    for (int b = 0; b < NB; ++b)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su(sm + k * STEP + b * 4096)), "l"(&src), "r"(x + b * 128), "r"(y), "r"(su(&bar[k])) : "memory");
  };
  for (; issued < ST && issued < total; ++issued) load(issued);
  for (long it = 0; it < total; ++it) {
    const int k = int(it % ST);
    asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}"
                 ::"r"(su(&bar[k])), "r"(ph[k]) : "memory");
    ph[k] ^= 1;
    int x, y;
    coords(it, x, y);
    for (int b = 0; b < NB; ++b)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"(&dst), "r"(x + b * 128), "r"(y), "r"(su(sm + k * STEP + b * 4096)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (issued < total) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(0) : "memory");
      load(issued++);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t n = 2ull << 30;
  uint8_t *a, *b;
  cudaMalloc(&a, n);
  cudaMalloc(&b, n);
  cudaMemset(a, 1, n);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap ms, md;
  cuuint64_t dims[2] = {4096, n / 4096}, strides[1] = {4096};
  cuuint32_t box[2] = {128, 32}, es[2] = {1, 1};
  enc(&ms, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&md, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, b, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int ntasks = int(n / (32 * 4096));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, int ctas, int smem, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<ctas, 32, smem>>>(ms, md, ntasks);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<ctas, 32, smem>>>(ms, md, ntasks);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float t;
    cudaEventElapsedTime(&t, e0, e1);
    t /= 5;
    printf("%-40s %7.3f ms %7.1f GB/s (R+W)  %s\n", name, t, 2.0 * n / t / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run(k<4, 256>, 148 * 4, 4 * 8192 + 1024, "TMA seg 256, 4 CTA/SM, ring 4");
  run(k<8, 256>, 148 * 2, 8 * 8192 + 1024, "TMA seg 256, 2 CTA/SM, ring 8");
  run(k<6, 256>, 148 * 4, 6 * 8192 + 1024, "TMA seg 256, 4 CTA/SM, ring 6");
  run(k<8, 128>, 148 * 4, 8 * 4096 + 1024, "TMA seg 128, 4 CTA/SM, ring 8");
  run(k<4, 512>, 148 * 2, 4 * 16384 + 1024, "TMA seg 512, 2 CTA/SM, ring 4");
  return 0;
}
