// Microbenchmark: scatter-add throughput options for spike delivery (SURVEY §8(a) a3 design space).
// Measures (1) HBM stream read of u32 records, (2) global red.add.u32 scattered into an
// L2-resident slot driven by a record stream (column-major sorted rows, like synth),
// (3) shared-memory atomicAdd scattered, (4) shared-memory non-atomic RMW (upper bound).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void stream_read(const uint4* __restrict__ p, size_t n4, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p+i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}
// rows: n_sp rows each of len L (padded to multiple of 128), column-major warp schedule
__global__ void deliver_red(const uint32_t* __restrict__ tgt, int n_sp, int L, uint32_t* slot) {
  int lane = threadIdx.x & 31;
  int warps = gridDim.x * blockDim.x / 32;
  int chunks = L / 128;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32; w < n_sp * chunks; w += warps) {
    int s = w % n_sp, c = w / n_sp;
    const uint4* p = reinterpret_cast<const uint4*>(tgt + (size_t)s * L + c * 128) + lane;
    uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.x));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.y));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.z));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.w));
  }
}
// same but row-major (warp handles whole row sequentially)
__global__ void deliver_red_rowmajor(const uint32_t* __restrict__ tgt, int n_sp, int L, uint32_t* slot) {
  int lane = threadIdx.x & 31;
  int warps = gridDim.x * blockDim.x / 32;
  int chunks = L / 128;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32; w < n_sp * chunks; w += warps) {
    int s = w / chunks, c = w % chunks;
    const uint4* p = reinterpret_cast<const uint4*>(tgt + (size_t)s * L + c * 128) + lane;
    uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.x));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.y));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.z));
    asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + v.w));
  }
}
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template<int MODE>
__global__ void smem_scatter(int iters, int words, uint32_t* out) {
  extern __shared__ uint32_t sm[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t seed = blockIdx.x * 977 + threadIdx.x * 131;
  for (int it = 0; it < iters; it++) {
    uint32_t h = hsh(seed + it * 0x9e3779b9u);
    uint32_t a = h % words;   // words is power of two -> cheap
    if (MODE == 0) atomicAdd(&sm[a], 1u);
    else if (MODE == 1) sm[a] += 1u;
    else { uint32_t a2 = (h >> 7) % words; atomicAdd(&sm[a], 1u); atomicAdd(&sm[a2], 1u);} 
  }
  __syncthreads();
  uint32_t acc = 0; for (int i = threadIdx.x; i < words; i += blockDim.x) acc += sm[i];
  atomicAdd(out, acc);
}
template<int MODE>
__global__ void hash_only(int iters, int words, uint32_t* out) {
  uint32_t seed = blockIdx.x * 977 + threadIdx.x * 131; uint32_t acc=0;
  for (int it = 0; it < iters; it++) { uint32_t h = hsh(seed + it * 0x9e3779b9u); acc += h % words; }
  if (acc == 7) out[0] = acc;
}
__global__ void gl_scatter(int iters, uint32_t words, uint32_t* slot) {
  uint32_t seed = blockIdx.x * 977 + threadIdx.x * 131;
  for (int it = 0; it < iters; it++) { uint32_t h = hsh(seed + it * 0x9e3779b9u); asm volatile("red.global.add.u32 [%0], 1;" :: "l"(slot + (h % words))); }
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d L2 %d\n", nsm, l2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  // synth-like: N=1386750 targets, n_sp=6934 rows of 2163 -> pad to 2176 (mult of 128 = 2176? 2176=17*128)
  const int N = 1386750, NSP = 6934, L = 2176;
  std::vector<uint32_t> h((size_t)NSP * L);
  std::mt19937 rng(1);
  for (int s = 0; s < NSP; s++) { for (int k = 0; k < L; k++) h[(size_t)s*L+k] = rng() % N; std::sort(&h[(size_t)s*L], &h[(size_t)s*L] + L); }
  uint32_t *d_t, *d_slot, *d_out, *d_flush;
  CK(cudaMalloc(&d_t, h.size() * 4)); CK(cudaMemcpy(d_t, h.data(), h.size()*4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d_slot, N * 4)); CK(cudaMemset(d_slot, 0, N*4)); CK(cudaMalloc(&d_out, 64));
  size_t flushn = 512ull<<20; CK(cudaMalloc(&d_flush, flushn));
  double events = (double)NSP * L, bytes = events * 4;
  for (int grid_mult : {4, 8, 16, 32}) for (int bs : {256, 512}) {
    int grid = nsm * grid_mult * 256 / bs;
    for (int rep = 0; rep < 3; rep++) {
      cudaMemset(d_flush, rep, flushn);
      cudaEventRecord(a); deliver_red<<<grid, bs>>>(d_t, NSP, L, d_slot); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("deliver_red colmajor grid=%d bs=%d: %.2f us  %.3e ev/s  %.0f GB/s\n", grid, bs, ms*1e3, events/(ms*1e-3), bytes/(ms*1e-3)/1e9);
      cudaMemset(d_flush, rep, flushn);
      cudaEventRecord(a); deliver_red_rowmajor<<<grid, bs>>>(d_t, NSP, L, d_slot); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("deliver_red rowmajor grid=%d bs=%d: %.2f us  %.3e ev/s\n", grid, bs, ms*1e3, events/(ms*1e-3));
      cudaMemset(d_flush, rep, flushn);
      cudaEventRecord(a); stream_read<<<grid, bs>>>((const uint4*)d_t, h.size()/4, d_out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("stream_read grid=%d bs=%d: %.2f us  %.0f GB/s\n", grid, bs, ms*1e3, bytes/(ms*1e-3)/1e9);
    }
  }
  // smem scatter: per-SM throughput
  for (int words : {16384, 32768, 49152 > 0 ? 32768 : 0}) {
    int iters = 4096; int bs = 1024; int grid = nsm;
    cudaFuncSetAttribute(smem_scatter<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
    cudaFuncSetAttribute(smem_scatter<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a); smem_scatter<0><<<grid, bs, words*4>>>(iters, words, d_out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); double ev = (double)grid*bs*iters;
      if (rep) printf("smem atomicAdd words=%d: %.2f us %.3e ev/s (%.2f ev/clk/SM @1.9GHz)\n", words, ms*1e3, ev/(ms*1e-3), ev/(ms*1e-3)/nsm/1.9e9);
      cudaEventRecord(a); smem_scatter<1><<<grid, bs, words*4>>>(iters, words, d_out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("smem RMW words=%d: %.2f us %.3e ev/s (%.2f ev/clk/SM)\n", words, ms*1e3, ev/(ms*1e-3), ev/(ms*1e-3)/nsm/1.9e9);
      cudaEventRecord(a); hash_only<0><<<grid, bs>>>(iters, words, d_out); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("hash only: %.2f us\n", ms*1e3);
    }
  }
  for (uint32_t words : {1u<<16, 1u<<20, 1386750u, 1u<<23}) {
    int iters = 256; int bs = 512; int grid = nsm * 4;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a); gl_scatter<<<grid, bs>>>(iters, words, d_slot /*size N*/ ); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b); double ev = (double)grid*bs*iters;
      if (rep) printf("global red random words=%u: %.2f us %.3e ev/s\n", words, ms*1e3, ev/(ms*1e-3));
    }
    if (words >= (uint32_t)N) break;
  }
  CK(cudaGetLastError());
  return 0;
}
