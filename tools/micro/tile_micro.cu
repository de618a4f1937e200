// Microbenchmark 2 for the delivery design: smem atomic rate,
// tiled segment gathers, bulk-reduce flush throughput, grid barrier latency.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int MODE>
__global__ void smem_rate(int iters, uint32_t mask, uint32_t* out) {
  extern __shared__ uint32_t sm[];
  for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t x = blockIdx.x * 977u + threadIdx.x * 131u + 7;
#pragma unroll 8
  for (int it = 0; it < iters; it++) {
    x = x * 1664525u + 1013904223u;
    uint32_t a = (x >> 8) & mask;
    if (MODE == 0) atomicAdd(&sm[a], 1u);
    else if (MODE == 1) atomicAdd(&sm[a >> 1], 1u << ((a & 1) * 16));
    else if (MODE == 2) sm[a] += 1u;
    else sm[a] = x;
  }
  __syncthreads();
  uint32_t acc = 0; for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) acc += sm[i];
  atomicAdd(out, acc);
}

// Tiled segment gather: CTA b handles tile b; for each spike s the segment starts at
// rowstart[s] + b*L (u16 entries), length L. Thread-per-spike, 16B aligned loads.
__global__ void seg_gather_tps(const uint16_t* __restrict__ ent, const uint64_t* __restrict__ rowstart,
                               int n_sp, int L, uint32_t tile_mask, uint32_t* out) {
  extern __shared__ uint32_t cnt[];
  for (uint32_t i = threadIdx.x; i <= tile_mask; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  for (int s = threadIdx.x; s < n_sp; s += blockDim.x) {
    uint64_t beg = rowstart[s] + (uint64_t)blockIdx.x * L, end = beg + L;
    uint64_t a = beg & ~7ull;
    for (; a < end; a += 8) {
      uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(ent + a));
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 8; q++) {
        uint64_t e = a + q;
        if (e >= beg && e < end) { uint32_t off = (w[q >> 1] >> ((q & 1) * 16)) & 0xFFFF; atomicAdd(&cnt[off & tile_mask], 1u); }
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i <= tile_mask; i += blockDim.x) if (cnt[i] == 0xFFFFFFFF) out[0] = i;
}
// warp-per-spike variant (good for long segments)
__global__ void seg_gather_wps(const uint16_t* __restrict__ ent, const uint64_t* __restrict__ rowstart,
                               int n_sp, int L, uint32_t tile_mask, uint32_t* out) {
  extern __shared__ uint32_t cnt[];
  for (uint32_t i = threadIdx.x; i <= tile_mask; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int s = warp; s < n_sp; s += nw) {
    uint64_t beg = rowstart[s] + (uint64_t)blockIdx.x * L, end = beg + L;
    for (uint64_t a = (beg & ~7ull) + lane * 8; a < end; a += 256) {
      uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(ent + a));
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 8; q++) {
        uint64_t e = a + q;
        if (e >= beg && e < end) { uint32_t off = (w[q >> 1] >> ((q & 1) * 16)) & 0xFFFF; atomicAdd(&cnt[off & tile_mask], 1u); }
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i <= tile_mask; i += blockDim.x) if (cnt[i] == 0xFFFFFFFF) out[0] = i;
}

__global__ void bulk_flush(uint32_t* dst, int words, int share, int reps) {
  extern __shared__ __align__(128) uint32_t sm[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 1;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  uint32_t* d = dst + (size_t)(blockIdx.x / share) * words;
  for (int r = 0; r < reps; r++) {
    if (threadIdx.x == 0) {
      const int chunk = 16384; // bytes
      for (int off = 0; off < words * 4; off += chunk) {
        uint32_t saddr = (uint32_t)__cvta_generic_to_shared(sm) + off;
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;" :: "l"((char*)d + off), "r"(saddr), "r"(chunk) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// plain coalesced add-store flush (exclusive owner)
__global__ void plain_flush(uint32_t* dst, int words, int reps) {
  extern __shared__ __align__(128) uint32_t sm[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sm[i] = 1;
  __syncthreads();
  uint32_t* d = dst + (size_t)blockIdx.x * words;
  for (int r = 0; r < reps; r++) {
    for (int i = threadIdx.x * 4; i < words; i += blockDim.x * 4) {
      uint4 o = *reinterpret_cast<uint4*>(d + i);
      o.x += sm[i]; o.y += sm[i+1]; o.z += sm[i+2]; o.w += sm[i+3];
      *reinterpret_cast<uint4*>(d + i) = o;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g = *gen;
    __threadfence();
    unsigned arrived = atomicAdd(count, 1u);
    if (arrived == nblocks - 1) { *count = 0; __threadfence(); atomicAdd((unsigned*)gen, 1u); }
    else { while (*gen == g) { __nanosleep(20); } }
    __threadfence();
  }
  __syncthreads();
}
__global__ void barrier_loop(unsigned* count, unsigned* gen, int iters) {
  for (int i = 0; i < iters; i++) grid_barrier(count, gen, gridDim.x);
}
__global__ void empty_kernel() {}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  uint32_t* d_out; CK(cudaMalloc(&d_out, 64));
  // ---- A: smem atomic rate
  for (int mode = 0; mode < 4; mode++) {
    for (uint32_t words : {16384u, 32768u}) {
      int iters = 1 << 14, bs = 1024;
      void (*k)(int, uint32_t, uint32_t*) = mode == 0 ? smem_rate<0> : mode == 1 ? smem_rate<1> : mode == 2 ? smem_rate<2> : smem_rate<3>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a); k<<<nsm, bs, words * 4>>>(iters, words - 1, d_out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double ev = (double)nsm * bs * iters;
        if (rep) printf("smem mode=%d(%s) words=%u: %.1f us, %.3e op/s, %.2f op/clk/SM @1.92GHz\n", mode,
          mode==0?"atomicAdd":mode==1?"atomicAdd packed16":mode==2?"plain RMW":"store", words, ms*1e3, ev/(ms*1e-3), ev/(ms*1e-3)/nsm/1.92e9);
      }
    }
  }
  CK(cudaGetLastError());
  // ---- B: segment gather
  size_t NE = 1ull << 30; uint16_t* d_ent; CK(cudaMalloc(&d_ent, NE * 2));
  CK(cudaMemset(d_ent, 0x35, NE * 2));
  uint32_t* d_flushbuf; size_t flushn = 512ull << 20; CK(cudaMalloc(&d_flushbuf, flushn));
  uint64_t* d_rs; CK(cudaMalloc(&d_rs, 40000 * 8));
  std::mt19937_64 rng(5);
  for (int n_sp : {6934, 19612}) for (int L : {5, 15, 60, 100, 400}) for (int tiles : {148, 296}) {
    if ((size_t)L * tiles > 60000) continue;
    std::vector<uint64_t> rs(n_sp); for (auto& x : rs) x = rng() % (NE - (size_t)L * tiles - 16);
    CK(cudaMemcpy(d_rs, rs.data(), n_sp * 8, cudaMemcpyHostToDevice));
    uint32_t tmask = 8191; int smem = (tmask + 1) * 4;
    for (int variant = 0; variant < 2; variant++) {
      float best = 1e9;
      for (int rep = 0; rep < 3; rep++) {
        cudaMemset(d_flushbuf, rep, flushn);
        cudaEventRecord(a);
        if (variant == 0) seg_gather_tps<<<tiles, 512, smem>>>(d_ent, d_rs, n_sp, L, tmask, d_out);
        else seg_gather_wps<<<tiles, 512, smem>>>(d_ent, d_rs, n_sp, L, tmask, d_out);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (rep) best = std::min(best, ms);
      }
      double ev = (double)n_sp * L * tiles;
      printf("seg_gather %s n_sp=%d L=%d tiles=%d: %.2f us  %.3e ev/s  payload %.0f GB/s (u16)\n", variant ? "warp/spike" : "thread/spike",
             n_sp, L, tiles, best * 1e3, ev / (best * 1e-3), ev * 2 / (best * 1e-3) / 1e9);
    }
  }
  CK(cudaGetLastError());
  // ---- C: flush
  uint32_t* d_dst; CK(cudaMalloc(&d_dst, 64ull << 20));
  for (int words : {8192, 32768}) for (int share : {1, 4, 8}) {
    cudaFuncSetAttribute(bulk_flush, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int reps = 20;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a); bulk_flush<<<nsm, 256, words * 4>>>(d_dst, words, share, reps); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      double bytes = (double)nsm * words * 4 * reps;
      if (rep) printf("bulk reduce flush words=%d share=%d: %.1f us per flush-round, %.0f GB/s\n", words, share, ms * 1e3 / reps, bytes / (ms * 1e-3) / 1e9);
    }
  }
  for (int words : {8192, 32768}) {
    cudaFuncSetAttribute(plain_flush, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int reps = 20;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a); plain_flush<<<nsm, 512, words * 4>>>(d_dst, words, reps); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      double bytes = (double)nsm * words * 4 * reps;
      if (rep) printf("plain add-store flush words=%d: %.2f us per round, %.0f GB/s\n", words, ms * 1e3 / reps, bytes / (ms * 1e-3) / 1e9);
    }
  }
  CK(cudaGetLastError());
  // ---- D: grid barrier
  unsigned *d_cnt, *d_gen; CK(cudaMalloc(&d_cnt, 4)); CK(cudaMalloc(&d_gen, 4)); cudaMemset(d_cnt, 0, 4); cudaMemset(d_gen, 0, 4);
  for (int per : {1, 2, 4}) {
    int iters = 10000;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a); barrier_loop<<<nsm * per, 256>>>(d_cnt, d_gen, iters); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("grid barrier %d CTAs: %.3f us per barrier\n", nsm * per, ms * 1e3 / iters);
    }
  }
  // launch overhead: graph of 100 empty kernels
  {
    cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; i++) empty_kernel<<<nsm, 256, 0, s>>>();
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("graph of 100 empty kernels: %.3f us per kernel\n", ms * 1e3 / 100);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
