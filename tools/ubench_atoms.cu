// Shared-memory atomic throughput microbenchmarks for k_bound's histogram
// design (not part of the product).  Each CTA: 512 threads, a 128 KB
// [64 bins][512 slots] u32 histogram (k_bound's footprint), conflict-free
// addresses (slot = thread), 1 CTA per SM, 148 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ua tools/ubench_atoms.cu && /tmp/ua
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// MODE 0: red.u32 all lanes; 1: red.u32 with `active` of 32 lanes (predicated);
// 2: red.u64; 3: red.u32 two lanes per bank (2-way conflict); 4: lds.32 (reads);
// 5: one address per thread (all 8 in flight hit it); 6: every warp on the
// same 32 slots, bins varying; 7: every warp on the same 32 words (one bin)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(long iters, int active, unsigned* out) {
  extern __shared__ unsigned h[];
  for (int x = threadIdx.x; x < 64 * 512; x += 512) h[x] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    unsigned hsh = (threadIdx.x * 2654435761u) ^ (u * 40503u + 12345u);
    hsh ^= hsh >> 13;
    hsh *= 0x5bd1e995u;
    hsh ^= hsh >> 15;
    // MODE 15: random bins; 16: half the lanes in bins 0 / 63 (k_bound's below / above slots)
    const int rbin = MODE == 16 ? ((hsh & 3) == 0 ? 0 : ((hsh & 3) == 1 ? 63 : (int)((hsh >> 8) % 62) + 1))
                                : (int)((hsh >> 8) & 63);
    const int bin = MODE == 5 || MODE == 7 ? 5 : (MODE >= 15 ? rbin : ((threadIdx.x * 7 + u * 13) & 63));
    const int slot = MODE == 3 ? ((threadIdx.x & ~31) | ((lane & 15) << 1)) : (MODE >= 6 ? lane : threadIdx.x);
    a[u] = smem_u32(h + bin * 512 + (MODE == 2 ? (slot & ~1) : slot));
  }
  const bool on = lane < active;
  unsigned accv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0 || MODE == 3 || (MODE >= 5 && MODE <= 7) || MODE >= 15) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u]), "r"((unsigned)i + u));
      if (MODE == 1 && on) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u]), "r"((unsigned)i + u));
      if (MODE == 2)
        asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a[u]), "l"((unsigned long long)i + u));
      if (MODE == 8) {  // one red + one lds.32 (other address)
        unsigned v;
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u]), "r"((unsigned)i + u));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(h) + ((a[(u + 3) & 7] - smem_u32(h) + 0x4000u) & 0x1fffcu)));
        accv[u] ^= v;
      }
      if (MODE == 9) {  // one red + one broadcast lds.128
        unsigned v0, v1, v2, v3;
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u]), "r"((unsigned)i + u));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                     : "r"(smem_u32(h) + ((((unsigned)i * 8 + u) * 16) & 0xfff0u)));
        accv[u] ^= v0 ^ v1 ^ v2 ^ v3;
      }
      if (MODE == 10) {  // broadcast lds.128 only
        unsigned v0, v1, v2, v3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                     : "r"(smem_u32(h) + ((((unsigned)i * 8 + u) * 16) & 0xfff0u)));
        accv[u] ^= v0 ^ v1 ^ v2 ^ v3;
      }
      if (MODE == 11) {  // lds.64, 32 lanes consecutive
        unsigned v0, v1;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1)
                     : "r"(smem_u32(h) + ((((unsigned)i * 8 + u) * 256 + (threadIdx.x & 31) * 8) & 0xffffu)));
        accv[u] ^= v0 ^ v1;
      }
      if (MODE == 12 || MODE == 13) {  // shfl.idx broadcast (13: plus one red)
        const unsigned v = __shfl_sync(0xffffffffu, accv[u] + (unsigned)i, (u + (int)i) & 31);
        accv[u] ^= v;
        if (MODE == 13) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u]), "r"((unsigned)i + u));
      }
      if (MODE == 14) {  // three reds per broadcast lds.128 (k_bound's mix, roughly)
        unsigned v0, v1, v2, v3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                     : "r"(smem_u32(h) + ((((unsigned)i * 8 + u) * 16) & 0xfff0u)));
        accv[u] ^= v0 ^ v1 ^ v2 ^ v3;
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u]), "r"((unsigned)i + u));
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[(u + 1) & 7]), "r"((unsigned)i + u));
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[(u + 2) & 7]), "r"((unsigned)i + u));
      }
      if (MODE == 4) {
        unsigned v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a[u] ^ ((unsigned)i & 4u)));
        accv[u] ^= v;
      }
    }
  }
  unsigned acc = 0;
  for (int u = 0; u < 8; ++u) acc ^= accv[u];
  __syncthreads();
  if (h[threadIdx.x] == 0x12345678u || acc == 0x12345u) out[0] = h[threadIdx.x] + acc;
}

template <int MODE>
float run(long iters, int active) {
  unsigned* d;
  cudaMalloc(&d, 4);
  const int sm = 64 * 512 * 4;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<MODE><<<148, 512, sm>>>(iters / 10, active, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148, 512, sm>>>(iters, active, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  if (cudaGetLastError() != cudaSuccess) { printf("mode %d failed\n", MODE); exit(1); }
  cudaFree(d);
  return ms;
}

int main() {
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const long it = 20000;
  const double warp_instr_per_sm = (double)it * 8 * 16;  // 16 warps x 8 per iteration
  auto rep = [&](const char* what, float ms) {
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-44s %8.3f ms  %6.3f SM-cycles per warp instruction\n", what, ms, cyc / warp_instr_per_sm);
  };
  rep("red.shared.add.u32, 32 lanes", run<0>(it, 32));
  for (int a : {24, 16, 8, 1}) {
    char b[64];
    snprintf(b, sizeof b, "red.shared.add.u32, %d lanes active", a);
    rep(b, run<1>(it, a));
  }
  rep("red.shared.add.u64, 32 lanes (16 words pairs)", run<2>(it, 32));
  rep("red.shared.add.u32, 2-way bank conflict", run<3>(it, 32));
  rep("ld.shared.u32, 32 lanes", run<4>(it, 32));
  rep("red.u32, each thread one address x8 in flight", run<5>(it, 32));
  rep("red.u32, 16 warps on the same 32 slots, bins vary", run<6>(it, 32));
  rep("red.u32, 16 warps on the same 32 words", run<7>(it, 32));
  rep("red.u32 + lds.32 (pair per instruction slot)", run<8>(it, 32));
  rep("red.u32 + broadcast lds.128", run<9>(it, 32));
  rep("broadcast lds.128 alone", run<10>(it, 32));
  rep("lds.64 32 lanes consecutive alone", run<11>(it, 32));
  rep("shfl.idx alone", run<12>(it, 32));
  rep("shfl.idx + red.u32", run<13>(it, 32));
  rep("broadcast lds.128 + 3 red.u32", run<14>(it, 32));
  rep("red.u32, random bins per lane", run<15>(it, 32));
  rep("red.u32, 50% of lanes in bins 0/63", run<16>(it, 32));
  return 0;
}
