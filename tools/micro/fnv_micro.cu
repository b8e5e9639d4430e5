// Raw FNV-1a throughput ceiling on B200: data synthesized in registers (no
// memory traffic), CH independent chains per thread, several step variants.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void stepA(uint32_t& lo, uint32_t& hi, uint32_t b) {
  const uint32_t x = lo ^ (b & 0xffu);
  const uint64_t t = (uint64_t)x * 0x1b3u;
  uint32_t y;
  asm("{\n\t.reg .u32 s;\n\tshl.b32 s, %1, 8;\n\tadd.u32 %0, s, %2;\n\t}" : "=r"(y) : "r"(x), "r"((uint32_t)(t >> 32)));
  hi = hi * 0x1b3u + y;
  lo = (uint32_t)t;
}
// lo via IMAD.LO and carry via IMAD.HI (no IMAD.WIDE)
__device__ __forceinline__ void stepB(uint32_t& lo, uint32_t& hi, uint32_t b) {
  const uint32_t x = lo ^ (b & 0xffu);
  uint32_t y;
  asm("mad.hi.u32 %0, %1, 435, %2;" : "=r"(y) : "r"(x), "r"(x << 8));
  hi = hi * 0x1b3u + y;
  lo = x * 0x1b3u;
}
// 64-bit mul by the full prime (compiler's own lowering)
__device__ __forceinline__ void stepC(uint32_t& lo, uint32_t& hi, uint32_t b) {
  uint64_t h = ((uint64_t)hi << 32) | lo;
  h ^= (b & 0xff);
  h *= 1099511628211ull;
  lo = (uint32_t)h; hi = (uint32_t)(h >> 32);
}


// hi folded into the wide multiply's 64-bit addend: Y = hi*P + (x<<8) (shift via PRMT on the
// ALU pipe), {lo,hi} = x*P + (Y<<32): one IMAD + one IMAD.WIDE per byte, no add
__device__ __forceinline__ void stepD(uint32_t& lo, uint32_t& hi, uint32_t b, uint32_t z) {
  const uint32_t x = lo ^ (b & 0xffu);
  uint32_t s;
  asm("prmt.b32 %0, %1, 0, 0x2104;" : "=r"(s) : "r"(x));
  const uint32_t y = hi * 0x1b3u + s;
  uint64_t t;
  asm("{\n\t.reg .u64 c;\n\tmov.b64 c, {%2, %3};\n\tmad.wide.u32 %0, %1, 435, c;\n\t}"
      : "=l"(t) : "r"(x), "r"(z), "r"(y));
  lo = (uint32_t)t;
  hi = (uint32_t)(t >> 32);
}
// same with a plain shift (ptxas picks the unit)
__device__ __forceinline__ void stepE(uint32_t& lo, uint32_t& hi, uint32_t b) {
  const uint32_t x = lo ^ (b & 0xffu);
  const uint32_t y = hi * 0x1b3u + (x << 8);
  const uint64_t t = (uint64_t)x * 0x1b3u + ((uint64_t)y << 32);
  lo = (uint32_t)t;
  hi = (uint32_t)(t >> 32);
}

// shift via PRMT (ALU only), then a plain add
__device__ __forceinline__ void stepF(uint32_t& lo, uint32_t& hi, uint32_t b) {
  const uint32_t x = lo ^ (b & 0xffu);
  uint32_t s;
  asm("prmt.b32 %0, %1, 0, 0x2104;" : "=r"(s) : "r"(x));
  const uint64_t t = (uint64_t)x * 0x1b3u;
  hi = hi * 0x1b3u + (uint32_t)(t >> 32) + s;
  lo = (uint32_t)t;
}
// lo by IMAD, carry + shifted x by IMAD.HI with the PRMT'd shift as addend
__device__ __forceinline__ void stepH(uint32_t& lo, uint32_t& hi, uint32_t b) {
  const uint32_t x = lo ^ (b & 0xffu);
  uint32_t s, y;
  asm("prmt.b32 %0, %1, 0, 0x2104;" : "=r"(s) : "r"(x));
  asm("mad.hi.u32 %0, %1, 435, %2;" : "=r"(y) : "r"(x), "r"(s));
  hi = hi * 0x1b3u + y;
  lo = x * 0x1b3u;
}

// byte pairs: hi2 = hi*P^2 + (t0.hi*P + t1.hi) + 256*(lo1 + x1), because x0*P = lo1 (mod 2^32)
__device__ __forceinline__ void stepG2(uint32_t& lo, uint32_t& hi, uint32_t b0, uint32_t b1) {
  const uint32_t x0 = lo ^ (b0 & 0xffu);
  const uint64_t t0 = (uint64_t)x0 * 0x1b3u;
  const uint32_t l1 = (uint32_t)t0;
  const uint32_t x1 = l1 ^ (b1 & 0xffu);
  const uint64_t t1 = (uint64_t)x1 * 0x1b3u;
  const uint32_t a = (uint32_t)(t0 >> 32) * 0x1b3u + (uint32_t)(t1 >> 32);
  uint32_t bb;
  asm("{\n\t.reg .u32 u;\n\tadd.u32 u, %1, %2;\n\tshl.b32 u, u, 8;\n\tadd.u32 %0, u, %3;\n\t}"
      : "=r"(bb) : "r"(l1), "r"(x1), "r"(a));
  hi = hi * 189225u + bb;
  lo = (uint32_t)t1;
}

template <int V, int CH>
__global__ void __launch_bounds__(512) k(uint64_t* out, int iters, uint32_t z) {
  uint32_t lo[CH], hi[CH];
  for (int c = 0; c < CH; ++c) { lo[c] = 0x84222325u + c; hi[c] = 0xcbf29ce4u; }
  uint32_t w = threadIdx.x * 2654435761u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      w = w * 1664525u + 1013904223u;  // one LCG per 4 words x CH chains
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        uint32_t ww = w ^ c;
        if (V == 7) {
          stepG2(lo[c], hi[c], ww, ww >> 8);
          stepG2(lo[c], hi[c], ww >> 16, ww >> 24);
        }
#pragma unroll
        for (int bb = 0; bb < 4 && V != 7; ++bb) {
          if (V == 0) stepA(lo[c], hi[c], ww >> (8 * bb));
          if (V == 1) stepB(lo[c], hi[c], ww >> (8 * bb));
          if (V == 2) stepC(lo[c], hi[c], ww >> (8 * bb));
          if (V == 3) stepD(lo[c], hi[c], ww >> (8 * bb), z);
          if (V == 4) stepE(lo[c], hi[c], ww >> (8 * bb));
          if (V == 5) stepF(lo[c], hi[c], ww >> (8 * bb));
          if (V == 6) stepH(lo[c], hi[c], ww >> (8 * bb));
        }
      }
    }
  }
  uint64_t r = 0;
  for (int c = 0; c < CH; ++c) r ^= ((uint64_t)hi[c] << 32) | lo[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int V, int CH>
void run(const char* name, int threads, int blocksPerSM) {
  uint64_t* d;
  cudaMalloc(&d, 148 * 4 * 1024 * 8);
  int iters = 2048;
  int blocks = 148 * blocksPerSM;
  k<V, CH><<<blocks, threads>>>(d, 16, 0u);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<V, CH><<<blocks, threads>>>(d, iters, 0u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double bytes = double(blocks) * threads * CH * iters * 16.0;
  printf("%-8s CH=%d threads/SM=%4d : %8.1f GB/s-equivalent\n", name, CH, threads * blocksPerSM,
         bytes / ms / 1e6);
  cudaFree(d);
}

int main() {
  run<0, 1>("A", 512, 1); run<0, 2>("A", 512, 1); run<0, 4>("A", 256, 1); run<0, 1>("A", 1024, 1); run<0, 2>("A", 1024, 1);
  run<1, 1>("B-hi", 512, 1); run<1, 2>("B-hi", 512, 1); run<1, 2>("B-hi", 1024, 1);
  run<2, 1>("C-64", 512, 1); run<2, 2>("C-64", 512, 1); run<2, 2>("C-64", 1024, 1);
  run<3, 1>("D-prmt", 512, 1); run<3, 2>("D-prmt", 512, 1); run<3, 4>("D-prmt", 256, 1); run<3, 2>("D-prmt", 1024, 1);
  run<4, 1>("E-wide", 512, 1); run<4, 2>("E-wide", 512, 1); run<4, 2>("E-wide", 1024, 1);
  run<5, 1>("F-prmt+", 512, 1); run<5, 2>("F-prmt+", 512, 1); run<5, 2>("F-prmt+", 1024, 1);
  run<6, 1>("H-hi", 512, 1); run<6, 2>("H-hi", 512, 1); run<6, 2>("H-hi", 1024, 1);
  run<7, 1>("G-pair", 512, 1); run<7, 2>("G-pair", 512, 1); run<7, 4>("G-pair", 256, 1);
  return 0;
}
