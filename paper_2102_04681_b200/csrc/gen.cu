// gen.cu — on-device network generator (SURVEY §8(a) a0'; §III-B,
// "the layout description is then uploaded to the GPU where it is expanded").
//
// Each rank expands only the edges whose target it owns (the descriptor split of
// {range1, range2 ∩ owned, p}), directly into the destination-tiled,
// source-major CSR used by delivery (rows stay contiguous so that the segments of
// neighbouring tiles share DRAM sectors through L2 — the Fig. 1 column-wise idea):
//   row_ptr[s]            start of source s's row (global source IDs, all N rows)
//   bnd[s*(NT+1) + b]     start of tile b's segment within row s (bnd[..NT] = row length)
//   ent[row_ptr[s] + e]   tile-local target offset (u16), ascending within each segment
// Pipeline: count per (row, tile) -> scan -> fill -> (fixed in-degree only) sort segments.
// Fixed probability rows come out sorted because every warp appends its row segment in
// ascending target order (ballot/prefix ordered append).
#include "spice_internal.cuh"
#include "spice_launch.h"

namespace spice {

__device__ __forceinline__ uint32_t warp_incl_scan_g(uint32_t x, uint32_t lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    return x;
}

// Bits of the 4 targets of local 4-block q of tile b that receive an edge from s.
__device__ __forceinline__ uint32_t prob_bits4(const GenGeom &g, const GenRule &r, uint32_t s,
                                               uint32_t i0) {
    if (i0 >= g.n_own) return 0u;
    // (32-bit index math: a 64-bit division per Philox call cost more than the Philox call)
    const uint32_t j0 = g.G == 1 ? i0 : (i0 / g.S * g.G + g.rank) * g.S + i0 % g.S;   // multiple of 4
    const uint4 x = philox4x32_10(make_uint4(s, j0 >> 2, r.index, kTagConn), g.key0, g.key1);
    uint32_t m = 0;
#pragma unroll
    for (uint32_t e = 0; e < 4; ++e) {
        const uint32_t j = j0 + e;
        const bool ok = (i0 + e < g.n_own) && j >= r.dst_begin && j < r.dst_end &&
                        (uint64_t)word_of(x, e) < r.thr;
        m |= (ok ? 1u : 0u) << e;
    }
    return m;
}

__device__ __forceinline__ bool tile_hits_dst(const GenGeom &g, const GenRule &r, uint32_t b) {
    const uint32_t lo = b * g.TW;
    if (lo >= g.n_own) return false;
    const uint32_t hi = min(lo + g.TW, g.n_own) - 1u;
    const uint64_t jlo = local_to_global(lo, g.rank, g.G, g.S);
    const uint64_t jhi = local_to_global(hi, g.rank, g.G, g.S);
    return !(jhi < r.dst_begin || jlo >= r.dst_end);
}

__global__ void __launch_bounds__(256) count_prob_kernel(GenGeom g, GenRule r, uint32_t *cnt) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * 8;
    const uint64_t npairs = (uint64_t)(r.src_end - r.src_begin) * g.NT;
    for (uint64_t w = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); w < npairs; w += nwarps) {
        const uint32_t s = r.src_begin + (uint32_t)(w / g.NT), b = (uint32_t)(w % g.NT);
        if (!tile_hits_dst(g, r, b)) continue;
        const uint32_t len = min(g.TW, g.n_own - b * g.TW);
        const uint32_t nblk = (len + 3u) / 4u;
        uint32_t c = 0;
        for (uint32_t q = lane; q < nblk; q += 32) c += __popc(prob_bits4(g, r, s, b * g.TW + 4u * q));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        if (lane == 0) cnt[(uint64_t)s * (g.NT + 1) + b] += c;
    }
}

__global__ void __launch_bounds__(256) fill_prob_kernel(GenGeom g, GenRule r, const uint64_t *row_ptr,
                                                        const uint32_t *bnd, uint32_t *cursor,
                                                        uint16_t *ent) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * 8;
    const uint64_t npairs = (uint64_t)(r.src_end - r.src_begin) * g.NT;
    for (uint64_t w = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); w < npairs; w += nwarps) {
        const uint32_t s = r.src_begin + (uint32_t)(w / g.NT), b = (uint32_t)(w % g.NT);
        if (!tile_hits_dst(g, r, b)) continue;
        const uint64_t seg = (uint64_t)s * (g.NT + 1) + b;
        uint64_t pos = row_ptr[s] + bnd[seg] + cursor[seg];
        const uint32_t len = min(g.TW, g.n_own - b * g.TW);
        const uint32_t nblk = (len + 3u) / 4u;
        uint32_t written = 0;
        for (uint32_t q0 = 0; q0 < nblk; q0 += 32) {
            const uint32_t q = q0 + lane;
            const uint32_t m = q < nblk ? prob_bits4(g, r, s, b * g.TW + 4u * q) : 0u;
            const uint32_t c = __popc(m);
            const uint32_t incl = warp_incl_scan_g(c, lane);
            uint64_t p = pos + incl - c;
            for (uint32_t e = 0; e < 4; ++e)
                if (m >> e & 1u) ent[p++] = (uint16_t)((4u * q + e) << g.eshift);
            const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
            pos += tot;
            written += tot;
        }
        if (lane == 0) cursor[seg] += written;
    }
}

// Fixed in-degree: target j (owned, in range2) draws k sources; r64 from
// Philox(ctr = (j, k>>1, rule, TAG_INDEG)) words 2(k&1), 2(k&1)+1; source =
// src_begin + floor(r64 |src| / 2^64) (reading R9).
template <bool FILL>
__global__ void __launch_bounds__(256) indeg_kernel(GenGeom g, GenRule r, const uint64_t *row_ptr,
                                                    const uint32_t *bnd, uint32_t *cnt_or_cursor,
                                                    uint16_t *ent) {
    const uint32_t kp = (r.k + 1u) / 2u;
    const uint64_t total = (uint64_t)g.n_own * kp;
    const uint64_t nsrc = (uint64_t)r.src_end - r.src_begin;
    const bool narrow = total < (1ull << 32);            // 32-bit index math when it fits
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = narrow ? (uint32_t)w / kp : (uint32_t)(w / kp);
        const uint32_t pr = narrow ? (uint32_t)w - i * kp : (uint32_t)(w % kp);
        const uint32_t j = g.G == 1 ? i : (i / g.S * g.G + g.rank) * g.S + i % g.S;
        if (j < r.dst_begin || j >= r.dst_end) continue;
        const uint4 x = philox4x32_10(make_uint4(j, pr, r.index, kTagIndeg), g.key0, g.key1);
        const uint32_t b = i / g.TW;
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t kk = 2u * pr + h;
            if (kk >= r.k) break;
            const uint64_t r64 = h ? (((uint64_t)x.w << 32) | x.z) : (((uint64_t)x.y << 32) | x.x);
            const uint32_t s = r.src_begin + (uint32_t)__umul64hi(r64, nsrc);
            const uint64_t seg = (uint64_t)s * (g.NT + 1) + b;
            const uint32_t slot = atomicAdd(&cnt_or_cursor[seg], 1u);
            if (FILL) ent[row_ptr[s] + bnd[seg] + slot] = (uint16_t)((i - b * g.TW) << g.eshift);
        }
    }
}

// Per row: exclusive prefix of the NT segment counts (in place), row length into rowlen.
// Padded layout (g.pad8): every segment is padded to a multiple of 8 entries (one aligned
// 16-byte window each), so the prefix runs over padded lengths and the true row length
// (out-degree on this rank) goes to deg[s].
__global__ void __launch_bounds__(256) row_prefix_kernel(GenGeom g, uint32_t *cnt, uint64_t *rowlen,
                                                         uint32_t *deg) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * 8;
    for (uint64_t s = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); s < g.N; s += nwarps) {
        uint32_t *row = cnt + s * (g.NT + 1);
        uint32_t carry = 0, ctrue = 0;
        for (uint32_t b0 = 0; b0 < g.NT; b0 += 32) {
            const uint32_t b = b0 + lane;
            const uint32_t c = b < g.NT ? row[b] : 0u;
            const uint32_t cp = g.pad8 ? (c + kWin - 1u) & ~(kWin - 1u) : c;
            const uint32_t incl = warp_incl_scan_g(cp, lane);
            if (b < g.NT) row[b] = carry + incl - cp;
            carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
            uint32_t ct = c;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ct += __shfl_xor_sync(0xFFFFFFFFu, ct, o);
            ctrue += ct;
        }
        if (lane == 0) { row[g.NT] = carry; rowlen[s] = carry; if (deg) deg[s] = ctrue; }
    }
}

// Padded layout: entries [cursor, padded length) of every segment get sentinel offsets
// TW + (window index mod 64) -- dummy counters past the tile, one per window, so that the
// sentinels of the 32 windows of one delivery round spread over distinct shared banks.
__global__ void __launch_bounds__(256) pad_segments_kernel(GenGeom g, const uint64_t *row_ptr,
                                                           const uint32_t *bnd, const uint32_t *cursor,
                                                           uint16_t *ent) {
    const uint64_t total = (uint64_t)g.N * g.NT;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)(w / g.NT), b = (uint32_t)(w % g.NT);
        const uint64_t seg = (uint64_t)s * (g.NT + 1) + b;
        const uint64_t base = row_ptr[s] + bnd[seg];
        const uint32_t padded = bnd[seg + 1] - bnd[seg];
        for (uint32_t e = cursor[seg]; e < padded; ++e)
            ent[base + e] = (uint16_t)((g.TW + (((base + e) >> kWinShift) & 63u)) << g.eshift);
    }
}

__global__ void sum_u32_kernel(const uint32_t *x, uint64_t n, unsigned long long *out) {
    unsigned long long t = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        t += x[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, t);
}

// Exclusive scan of n u64 values (in place, out[n] = total); 3 kernels.
constexpr int kScanBlock = 1024;
__global__ void scan_block_sums(const uint64_t *in, uint64_t n, uint64_t *sums) {
    __shared__ uint64_t red[32];
    const uint64_t i = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
    uint64_t v = i < n ? in[i] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < kScanBlock / 32; ++w) t += red[w];
        sums[blockIdx.x] = t;
    }
}
__global__ void scan_sums_serial(uint64_t *sums, uint64_t nb) {
    // single block: chunked exclusive scan of the block sums
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < nb; base += kScanBlock) {
        __shared__ uint64_t buf[kScanBlock];
        const uint64_t i = base + threadIdx.x;
        buf[threadIdx.x] = i < nb ? sums[i] : 0;
        __syncthreads();
        for (int o = 1; o < kScanBlock; o <<= 1) {
            const uint64_t y = threadIdx.x >= (unsigned)o ? buf[threadIdx.x - o] : 0;
            __syncthreads();
            buf[threadIdx.x] += y;
            __syncthreads();
        }
        const uint64_t incl = buf[threadIdx.x];
        const uint64_t excl = incl - (i < nb ? sums[i] : 0);
        __syncthreads();
        if (i < nb) sums[i] = carry + excl;
        __syncthreads();
        if (threadIdx.x == kScanBlock - 1) carry += incl;
        __syncthreads();
    }
}
__global__ void scan_apply(const uint64_t *in, uint64_t n, const uint64_t *sums, uint64_t *out) {
    __shared__ uint64_t buf[kScanBlock];
    const uint64_t i = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
    const uint64_t v = i < n ? in[i] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kScanBlock; o <<= 1) {
        const uint64_t y = threadIdx.x >= (unsigned)o ? buf[threadIdx.x - o] : 0;
        __syncthreads();
        buf[threadIdx.x] += y;
        __syncthreads();
    }
    if (i < n) out[i] = sums[blockIdx.x] + buf[threadIdx.x] - v;
    if (i == n - 1) out[n] = sums[blockIdx.x] + buf[threadIdx.x];
}

// Segment sort, one warp per (row, tile) segment of length in (lo, 32 R]: a bitonic
// network over 32 R keys in registers (key lane + 32 r in k[r]; missing keys are 0x10000
// and sort last).  R = 2 takes segments of 2..64 entries, R = 4 those of 65..128, and
// sort_segments_kernel the rest (fixed in-degree fills segments out of order).
template <int R>
__global__ void __launch_bounds__(256) sort_segments_warp_kernel(GenGeom g, const uint64_t *row_ptr,
                                                                 const uint32_t *bnd, uint16_t *ent,
                                                                 uint32_t lo) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t total = (uint64_t)g.N * g.NT;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; w < total; w += nwarps) {
        const uint32_t s = (uint32_t)(w / g.NT), b = (uint32_t)(w % g.NT);
        const uint64_t seg = (uint64_t)s * (g.NT + 1) + b;
        const uint32_t b0 = bnd[seg], b1 = bnd[seg + 1];
        const uint32_t len = b1 - b0;
        if (len <= lo || len > 32u * R) continue;            // warp-uniform
        uint16_t *p = ent + row_ptr[s] + b0;
        uint32_t k[R];
#pragma unroll
        for (int r = 0; r < R; ++r) k[r] = lane + 32u * r < len ? p[lane + 32u * r] : 0x10000u;
#pragma unroll
        for (uint32_t size = 2; size <= 32u * R; size <<= 1) {
#pragma unroll
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                if (stride >= 32) {                          // partner in register r ^ (stride / 32)
                    const uint32_t rs = stride / 32;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        if (r & rs) continue;
                        const int r2 = r | (int)rs;
                        const bool up = ((lane + 32u * r) & size) == 0;
                        const uint32_t a = min(k[r], k[r2]), z = max(k[r], k[r2]);
                        k[r] = up ? a : z;
                        k[r2] = up ? z : a;
                    }
                } else {
                    const bool lower = (lane & stride) == 0;     // this element has the lower index
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const uint32_t o = __shfl_xor_sync(0xFFFFFFFFu, k[r], stride);
                        const bool up = ((lane + 32u * r) & size) == 0;
                        k[r] = (lower == up) ? min(k[r], o) : max(k[r], o);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) if (lane + 32u * r < len) p[lane + 32u * r] = (uint16_t)k[r];
    }
}

// Insertion sort, one thread per (row, tile) segment longer than 128 entries.
__global__ void __launch_bounds__(256) sort_segments_kernel(GenGeom g, const uint64_t *row_ptr,
                                                            const uint32_t *bnd, uint16_t *ent) {
    const uint64_t total = (uint64_t)g.N * g.NT;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)(w / g.NT), b = (uint32_t)(w % g.NT);
        const uint64_t seg = (uint64_t)s * (g.NT + 1) + b;
        const uint32_t b0 = bnd[seg], b1 = bnd[seg + 1];
        if (b1 - b0 <= 128) continue;                        // (sorted by the warp kernels)
        uint16_t *p = ent + row_ptr[s] + b0;
        const uint32_t len = b1 - b0;
        for (uint32_t x = 1; x < len; ++x) {
            const uint16_t key = p[x];
            uint32_t y = x;
            while (y > 0 && p[y - 1] > key) { p[y] = p[y - 1]; --y; }
            p[y] = key;
        }
    }
}

__global__ void init_uniform_kernel(GenGeom g, uint32_t field, float lo, float hi, float *out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n_own) return;
    const uint32_t j = (uint32_t)local_to_global(i, g.rank, g.G, g.S);
    const uint4 x = philox4x32_10(make_uint4(j >> 2, field, 0u, kTagInit), g.key0, g.key1);
    // u = (x >> 8) 2^-24 exactly; value = lo + u (hi - lo) (reading R15)
    const float u = __fmul_rn(__uint2float_rn(word_of(x, j & 3) >> 8), 5.9604644775390625e-08f);
    out[i] = __fadd_rn(lo, __fmul_rn(u, __fsub_rn(hi, lo)));
}

static int grid_for(uint64_t work, int per_block) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (work + per_block - 1) / per_block;
    const uint64_t cap = (uint64_t)nsm * 16;
    return (int)(want < cap ? (want ? want : 1) : cap);
}

cudaError_t gen_count(const GenGeom &g, const GenRule &r, uint32_t *cnt, cudaStream_t s) {
    if (r.src_end <= r.src_begin || r.dst_end <= r.dst_begin) return cudaSuccess;
    if (r.kind == 0) {
        if (r.thr == 0) return cudaSuccess;
        count_prob_kernel<<<grid_for((uint64_t)(r.src_end - r.src_begin) * g.NT, 8), 256, 0, s>>>(g, r, cnt);
    } else {
        if (r.k == 0) return cudaSuccess;
        indeg_kernel<false><<<grid_for((uint64_t)g.n_own * ((r.k + 1) / 2), 256), 256, 0, s>>>(
            g, r, nullptr, nullptr, cnt, nullptr);
    }
    return cudaGetLastError();
}

cudaError_t gen_scan(const GenGeom &g, uint32_t *cnt_bnd, uint64_t *row_ptr, uint64_t *nnz,
                     uint32_t *deg, cudaStream_t s) {
    cudaError_t e;
    row_prefix_kernel<<<grid_for(g.N, 8), 256, 0, s>>>(g, cnt_bnd, row_ptr, deg);
    if ((e = cudaGetLastError())) return e;
    const uint64_t n = g.N;
    const uint64_t nb = (n + kScanBlock - 1) / kScanBlock;
    uint64_t *sums = nullptr;
    if ((e = cudaMallocAsync(&sums, nb * sizeof(uint64_t), s))) return e;
    scan_block_sums<<<(unsigned)nb, kScanBlock, 0, s>>>(row_ptr, n, sums);
    scan_sums_serial<<<1, kScanBlock, 0, s>>>(sums, nb);
    scan_apply<<<(unsigned)nb, kScanBlock, 0, s>>>(row_ptr, n, sums, row_ptr);
    if ((e = cudaGetLastError())) return e;
    if ((e = cudaFreeAsync(sums, s))) return e;
    if ((e = cudaMemcpyAsync(nnz, row_ptr + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s))) return e;
    return cudaStreamSynchronize(s);
}

cudaError_t gen_scan_u64(uint64_t *data, uint64_t n, cudaStream_t s) {
    cudaError_t e;
    const uint64_t nb = (n + kScanBlock - 1) / kScanBlock;
    uint64_t *sums = nullptr;
    if (n == 0) return cudaMemsetAsync(data, 0, 8, s);
    if ((e = cudaMallocAsync(&sums, nb * sizeof(uint64_t), s))) return e;
    scan_block_sums<<<(unsigned)nb, kScanBlock, 0, s>>>(data, n, sums);
    scan_sums_serial<<<1, kScanBlock, 0, s>>>(sums, nb);
    scan_apply<<<(unsigned)nb, kScanBlock, 0, s>>>(data, n, sums, data);
    if ((e = cudaGetLastError())) return e;
    return cudaFreeAsync(sums, s);
}

cudaError_t gen_fill(const GenGeom &g, const GenRule &r, const uint64_t *row_ptr,
                     const uint32_t *bnd, uint32_t *cursor, uint16_t *ent, cudaStream_t s) {
    if (r.src_end <= r.src_begin || r.dst_end <= r.dst_begin) return cudaSuccess;
    if (r.kind == 0) {
        if (r.thr == 0) return cudaSuccess;
        fill_prob_kernel<<<grid_for((uint64_t)(r.src_end - r.src_begin) * g.NT, 8), 256, 0, s>>>(
            g, r, row_ptr, bnd, cursor, ent);
    } else {
        if (r.k == 0) return cudaSuccess;
        indeg_kernel<true><<<grid_for((uint64_t)g.n_own * ((r.k + 1) / 2), 256), 256, 0, s>>>(
            g, r, row_ptr, bnd, cursor, ent);
    }
    return cudaGetLastError();
}

cudaError_t gen_pad_segments(const GenGeom &g, const uint64_t *row_ptr, const uint32_t *bnd,
                             const uint32_t *cursor, uint16_t *ent, cudaStream_t s) {
    pad_segments_kernel<<<grid_for((uint64_t)g.N * g.NT, 256), 256, 0, s>>>(g, row_ptr, bnd, cursor, ent);
    return cudaGetLastError();
}

cudaError_t gen_sum_u32(const uint32_t *x, uint64_t n, uint64_t *out_host, cudaStream_t s) {
    cudaError_t e;
    unsigned long long *d = nullptr;
    if ((e = cudaMallocAsync(&d, 8, s))) return e;
    if ((e = cudaMemsetAsync(d, 0, 8, s))) return e;
    if (n) sum_u32_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, d);
    if ((e = cudaMemcpyAsync(out_host, d, 8, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaFreeAsync(d, s))) return e;
    return cudaStreamSynchronize(s);
}

cudaError_t gen_sort_segments(const GenGeom &g, const uint64_t *row_ptr, const uint32_t *bnd,
                              uint16_t *ent, cudaStream_t s) {
    sort_segments_warp_kernel<2><<<grid_for((uint64_t)g.N * g.NT * 32, 256), 256, 0, s>>>(g, row_ptr, bnd, ent, 1u);
    sort_segments_warp_kernel<4><<<grid_for((uint64_t)g.N * g.NT * 32, 256), 256, 0, s>>>(g, row_ptr, bnd, ent, 64u);
    sort_segments_kernel<<<grid_for((uint64_t)g.N * g.NT, 256), 256, 0, s>>>(g, row_ptr, bnd, ent);
    return cudaGetLastError();
}

// ---- Brunel+ plastic synapses: weights and the per-target in-synapse index ----
__device__ __forceinline__ bool is_plastic(const PlasticBoxes &pb, uint32_t s, uint32_t j) {
    for (uint32_t q = 0; q < pb.n; ++q)
        if (s >= pb.box[q][0] && s < pb.box[q][1] && j >= pb.box[q][2] && j < pb.box[q][3]) return true;
    return false;
}
__global__ void __launch_bounds__(256) plastic_weights_kernel(GenGeom g, PlasticBoxes pb, const uint64_t *row_ptr,
                                                              const uint32_t *bnd, const uint16_t *ent, float *w,
                                                              float w0) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * 8;
    for (uint64_t q = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); q < (uint64_t)g.N * g.NT; q += nwarps) {
        const uint32_t s = (uint32_t)(q / g.NT), b = (uint32_t)(q % g.NT);
        const uint32_t *bp = bnd + (uint64_t)s * (g.NT + 1) + b;
        const uint64_t st = row_ptr[s] + bp[0];
        const uint32_t len = bp[1] - bp[0];
        for (uint32_t e = lane; e < len; e += 32) {
            const uint32_t il = b * g.TW + (ent[st + e] >> g.eshift);
            w[st + e] = is_plastic(pb, s, (uint32_t)local_to_global(il, g.rank, g.G, g.S)) ? w0 : -1.0f;
        }
    }
}

cudaError_t gen_plastic_weights(const GenGeom &g, const PlasticBoxes &pb, const uint64_t *row_ptr,
                                const uint32_t *bnd, const uint16_t *ent, float *w, float w0, cudaStream_t s) {
    plastic_weights_kernel<<<grid_for((uint64_t)g.N * g.NT, 8), 256, 0, s>>>(g, pb, row_ptr, bnd, ent, w, w0);
    return cudaGetLastError();
}

// ---- per-synapse delays (reading R19) ----
__global__ void __launch_bounds__(256) delays_kernel(GenGeom g, DelayRules dr, uint32_t dmin, const uint64_t *row_ptr,
                                                     const uint32_t *bnd, const uint16_t *ent, uint8_t *dly) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * 8;
    for (uint64_t q = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); q < (uint64_t)g.N * g.NT; q += nwarps) {
        const uint32_t s = (uint32_t)(q / g.NT), b = (uint32_t)(q % g.NT);
        const uint32_t *bp = bnd + (uint64_t)s * (g.NT + 1) + b;
        const uint64_t st = row_ptr[s] + bp[0];
        const uint32_t len = bp[1] - bp[0];
        for (uint32_t e = lane; e < len; e += 32) {
            const uint32_t off = ent[st + e] >> g.eshift;
            uint32_t d = dmin;                                  // (padding sentinels: the fast path)
            if (off < g.TW) {
                const uint32_t j = (uint32_t)local_to_global((uint64_t)b * g.TW + off, g.rank, g.G, g.S);
                for (uint32_t r = 0; r < dr.n; ++r)
                    if (s >= dr.box[r][0] && s < dr.box[r][1] && j >= dr.box[r][2] && j < dr.box[r][3]) {
                        d = dr.lo[r];
                        if (dr.hi[r] > dr.lo[r]) {
                            const uint4 x = philox4x32_10(make_uint4(s, j >> 2, dr.index[r], kTagDelay), g.key0, g.key1);
                            d += (uint32_t)(((uint64_t)word_of(x, j & 3) * (dr.hi[r] - dr.lo[r] + 1)) >> 32);
                        }
                        break;
                    }
            }
            dly[st + e] = (uint8_t)d;
        }
    }
}

cudaError_t gen_delays(const GenGeom &g, const DelayRules &dr, uint32_t dmin, const uint64_t *row_ptr,
                       const uint32_t *bnd, const uint16_t *ent, uint8_t *dly, cudaStream_t s) {
    delays_kernel<<<grid_for((uint64_t)g.N * g.NT, 8), 256, 0, s>>>(g, dr, dmin, row_ptr, bnd, ent, dly);
    return cudaGetLastError();
}

cudaError_t gen_init_uniform(const GenGeom &g, uint32_t field, float lo, float hi, float *out,
                             cudaStream_t s) {
    if (g.n_own == 0) return cudaSuccess;
    init_uniform_kernel<<<(g.n_own + 255) / 256, 256, 0, s>>>(g, field, lo, hi, out);
    return cudaGetLastError();
}

}  // namespace spice
