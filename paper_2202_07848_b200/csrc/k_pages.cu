// k_pages.cu — host-page snapshot classification (build_manifest host section,
// ckpt.cpp:116-130): for every 4 KiB page digest of a rank's paged host words,
//   fresh = first occurrence in this call and not in the store index (known set)
//           (BlobStore::put's `fresh`, ckpt.cpp:18-20, in put order)
//   inc   = digest absent from the previous manifest's page set of the rank
//           (s_cr_inc, ckpt.cpp:127-128)
// Two passes over the digest vector: insert (atomicMin of the page index per
// digest), then classify + block-reduced counts.
#include "table.cuh"

namespace snap {
namespace {

constexpr int kThreads = 256;

__global__ void k_page_insert(TableDev pages, TableDev known, int use_known,
                              const uint64_t* __restrict__ dig, uint64_t n,
                              uint64_t* __restrict__ slot) {
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long d = dig[p];
    uint64_t s = ~0ull;
    if (!(use_known && table_find(known, d) != ~0ull)) {
      s = table_find_or_insert(pages, d);
      atomicMin(pages.vals + s, static_cast<unsigned long long>(p));
    }
    slot[p] = s;
  }
}

__global__ void __launch_bounds__(kThreads)
    k_page_classify(TableDev pages, TableDev prev, int use_prev, const uint64_t* __restrict__ dig,
                    const uint64_t* __restrict__ slot, uint64_t n, uint8_t* __restrict__ flags,
                    unsigned long long* __restrict__ counts) {
  unsigned fresh = 0, inc = 0;
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t s = slot[p];
    const bool f = s != ~0ull && pages.vals[s] == p;
    const bool i = !use_prev || table_find(prev, dig[p]) == ~0ull;
    flags[p] = uint8_t((f ? 1 : 0) | (i ? 2 : 0));
    fresh += f;
    inc += i;
  }
  for (int o = 16; o; o >>= 1) {
    fresh += __shfl_xor_sync(0xffffffffu, fresh, o);
    inc += __shfl_xor_sync(0xffffffffu, inc, o);
  }
  __shared__ unsigned sf[kThreads / 32], si[kThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    sf[threadIdx.x >> 5] = fresh;
    si[threadIdx.x >> 5] = inc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, b = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      a += sf[w];
      b += si[w];
    }
    atomicAdd(counts, a);
    atomicAdd(counts + 1, b);
  }
}

unsigned grid_for(uint64_t n) {
  const uint64_t b = (n + kThreads - 1) / kThreads;
  return unsigned(b < 148 * 8 ? (b ? b : 1) : 148 * 8);
}

}  // namespace

int launch_page_classify(TableDev pages, TableDev known, bool use_known, TableDev prev,
                         bool use_prev, const uint64_t* dig, uint64_t n, uint64_t* slot,
                         uint8_t* flags, unsigned long long* counts, cudaStream_t s) {
  if (n == 0) return 0;
  k_page_insert<<<grid_for(n), kThreads, 0, s>>>(pages, known, use_known ? 1 : 0, dig, n, slot);
  k_page_classify<<<grid_for(n), kThreads, 0, s>>>(pages, prev, use_prev ? 1 : 0, dig, slot, n,
                                                   flags, counts);
  return 2;
}

}  // namespace snap
