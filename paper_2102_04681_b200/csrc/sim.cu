// sim.cu — per-step kernels of the Spice hot path on sm_100a.
//
//   update_kernel<MODEL>   neuron update + warp-ballot spike bitmap + block-prefix spike
//                          compaction (Listing 1)
//   deliver_tiled<GS>      destination-tiled spike delivery: every CTA owns a tile of
//                          targets, walks the tile's segment of each spiking row (rows
//                          pre-split at tile pivots, the split of P:273-275) and
//                          accumulates receptor counts with shared-memory atomics; the
//                          tile is then added to the L2-resident input ring slot
//                          (a3; "delivered to all neighbors in said row")
//   deliver_global_atomics paper-style column-wise warps with global atomics (P:200,
//                          P:436 "bottlenecked by atomic operations"): the A/B baseline
//   bitmap_to_list         gathered per-rank bitmaps -> global spike list (a2, G > 1)
//
// Floating point: every operation of the neuron update is an explicit round-to-nearest
// intrinsic in the order fixed by DESIGN.md readings R3-R5 (no contraction), so results
// are bit-identical to the fp32 oracle.
#include "spice_internal.cuh"
#include "spice_launch.h"

namespace spice {

__device__ __forceinline__ uint32_t philox_pick(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                                uint32_t k0, uint32_t k1, uint32_t which) {
    return word_of(philox4x32_10(make_uint4(w0, w1, w2, w3), k0, k1), which);
}

template <int MODEL>
__global__ void __launch_bounds__(kUpdateBlock) update_kernel(SimArgs a, uint32_t k, int produce_list) {
    const uint64_t t = *a.t0 + k;
    const uint32_t i = blockIdx.x * kUpdateBlock + threadIdx.x;   // local index
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool valid = i < a.n_own;
    const uint32_t j = valid ? (uint32_t)local_to_global(i, a.rank, a.G, a.S) : 0u;
    bool spiked = false;
    if (valid) {
        uint32_t *slot = a.ring + (t % a.D) * a.ring_stride + i;
        const uint32_t c = *slot;
        *slot = 0u;
        const ModelConst &m = a.mc;
        int forced = 0;
        bool fbit = false;
        if (a.force_ctl[0] == t) {
            forced = (int)a.force_ctl[1];
            fbit = (a.force_bits[i >> 5] >> (i & 31)) & 1u;
        }
        if (MODEL == 4) {                           // Synth (reading R12)
            a.acc[i] = a.acc[i] + c;
            const uint32_t x = philox_pick(j >> 2, (uint32_t)t, 0u, kTagFire, a.key0, a.key1, j & 3);
            spiked = (uint64_t)x < m.thr_fire;
            if (forced == 1) spiked = fbit; else if (forced == 2) spiked = spiked || fbit;
        } else if (MODEL == 1) {                    // Vogels-Abbott COBA (readings R3-R5)
            const uint32_t ne = c & 0xFFFFu, ni = c >> 16;
            float ge = a.ge[i], gi = a.gi[i], v = a.v[i];
            uint32_t ref = a.ref[i];
            ge = __fadd_rn(ge, __fmul_rn(m.dge, __uint2float_rn(ne)));
            gi = __fadd_rn(gi, __fmul_rn(m.dgi, __uint2float_rn(ni)));
            if (ref > 0u) {
                ref -= 1u;
                v = m.Vr;
            } else {
                const float ta = __fsub_rn(m.EL, v);
                const float tb = __fmul_rn(ge, __fsub_rn(m.Ee, v));
                const float tc = __fmul_rn(gi, __fsub_rn(m.Ei, v));
                const float sum = __fadd_rn(__fadd_rn(ta, tb), tc);
                v = __fadd_rn(v, __fmul_rn(m.h, sum));
                spiked = v >= m.Vt;
            }
            if (forced == 1) spiked = fbit; else if (forced == 2) spiked = spiked || fbit;
            if (spiked) { v = m.Vr; ref = m.R; }
            ge = __fsub_rn(ge, __fmul_rn(m.ke, ge));
            gi = __fsub_rn(gi, __fmul_rn(m.ki, gi));
            a.v[i] = v; a.ge[i] = ge; a.gi[i] = gi; a.ref[i] = ref;
        } else {                                    // Brunel model A (readings R3-R5, R12)
            float v = a.v[i];
            uint32_t ref = a.ref[i];
            if (ref > 0u) {
                ref -= 1u;
                v = m.Vr;                          // input and drive discarded
            } else {
                const uint32_t x = philox_pick(j >> 2, (uint32_t)t, 0u, kTagExt, a.key0, a.key1, j & 3);
                uint32_t next = 0;
                while ((uint64_t)x >= m.ptab[next]) ++next;   // min{k : x < T_k}
                const uint32_t ne = c & 0xFFFFu, ni = c >> 16;
                v = __fadd_rn(v, __fmul_rn(m.h, __fsub_rn(m.EL, v)));
                v = __fadd_rn(v, __fmul_rn(m.JE, __uint2float_rn(ne + next)));
                v = __fadd_rn(v, __fmul_rn(m.JI, __uint2float_rn(ni)));
                spiked = v >= m.theta;
            }
            if (forced == 1) spiked = fbit; else if (forced == 2) spiked = spiked || fbit;
            if (spiked) { v = m.Vr; ref = m.R; }
            a.v[i] = v; a.ref[i] = ref;
        }
    }
    // --- warp ballot -> bitmap word (32 consecutive local indices; S % 32 == 0) ---
    const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, spiked);
    const uint32_t wi = i >> 5;
    if (lane == 0 && wi < a.W) {
        uint32_t *bm = a.G == 1 ? a.record + (t % a.record_steps) * (uint64_t)a.W : a.sendbuf;
        bm[wi] = ballot;
    }
    // --- block prefix over warp popcounts -> one atomic per CTA -> ordered append ---
    __shared__ uint32_t s_wcnt[kUpdateBlock / 32];
    __shared__ uint32_t s_base;
    if (lane == 0) s_wcnt[warp] = __popc(ballot);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < kUpdateBlock / 32; ++w) { const uint32_t cw = s_wcnt[w]; s_wcnt[w] = tot; tot += cw; }
        if (tot) atomicAdd(&a.stats[0], (unsigned long long)tot);
        s_base = (produce_list && tot) ? atomicAdd(&a.spcount[t % 3], tot) : 0u;
        if (produce_list && blockIdx.x == 0) a.spcount[(t + 1) % 3] = 0u;
    }
    __syncthreads();
    if (produce_list && spiked) {
        const uint32_t pos = s_base + s_wcnt[warp] + __popc(ballot & ((1u << lane) - 1u));
        a.splist[pos] = j;
    }
}

__device__ __forceinline__ uint2 ld_stream_v2(const uint16_t *p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

// Destination-tiled delivery.  CTA (b, c) owns tile b's counters in shared memory and
// handles spikes p = c, c+C, c+2C, ... of the step's list.  GS lanes cooperate on one
// segment, each loading 8 bytes (4 u16 offsets) per window.
template <int GS>
__global__ void __launch_bounds__(kDeliverBlock) deliver_tiled(SimArgs a, uint32_t k,
                                                               const uint32_t *__restrict__ list) {
    extern __shared__ __align__(16) uint32_t smem[];
    const uint32_t tw_pad = (a.TW + 3u) & ~3u;
    uint32_t *cnt = smem;
    uint64_t *dstart = reinterpret_cast<uint64_t *>(smem + tw_pad + (tw_pad & 1u ? 1u : 0u));
    uint32_t *dlen = reinterpret_cast<uint32_t *>(dstart + kDescChunk);
    const uint64_t t = *a.t0 + k;
    const uint32_t b = blockIdx.x / a.C, c = blockIdx.x % a.C;
    const uint32_t tid = threadIdx.x;
    for (uint32_t x = tid; x < a.TW; x += kDeliverBlock) cnt[x] = 0u;
    const uint32_t n_sp = a.spcount[t % 3];
    const uint32_t my = n_sp > c ? (n_sp - c + a.C - 1u) / a.C : 0u;
    uint32_t delivered = 0;
    const uint32_t grp = tid / GS, lig = tid % GS;
    constexpr uint32_t ngrp = kDeliverBlock / GS;
    for (uint32_t q0 = 0; q0 < my; q0 += kDescChunk) {
        const uint32_t nq = min((uint32_t)kDescChunk, my - q0);
        __syncthreads();
        for (uint32_t q = tid; q < nq; q += kDeliverBlock) {
            const uint32_t s = list[c + (q0 + q) * a.C];
            const uint32_t *bp = a.bnd + (uint64_t)s * (a.NT + 1u) + b;
            const uint32_t b0 = bp[0], b1 = bp[1];
            dstart[q] = a.row_ptr[s] + b0;
            dlen[q] = (b1 - b0) | (s >= a.n_exc ? 0x80000000u : 0u);
            delivered += b1 - b0;
        }
        __syncthreads();
        for (uint32_t q = grp; q < nq; q += ngrp) {
            const uint64_t st = dstart[q];
            const uint32_t lw = dlen[q];
            const uint64_t en = st + (lw & 0x7FFFFFFFu);
            const uint32_t qv = (lw >> 31) ? 65536u : 1u;
            for (uint64_t w = (st & ~3ull) + lig * 4u; w < en; w += GS * 4u) {
                const uint2 v = ld_stream_v2(a.ent + w);
                const uint32_t e[4] = {v.x & 0xFFFFu, v.x >> 16, v.y & 0xFFFFu, v.y >> 16};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (w + u >= st && w + u < en) atomicAdd(&cnt[e[u]], qv);
            }
        }
    }
    __syncthreads();
    // Add the tile into the input ring slot of step t + delay (exclusive owner when C = 1).
    uint32_t *dst = a.ring + ((t + a.delay) % a.D) * a.ring_stride + (uint64_t)b * a.TW;
    if (a.C == 1u) {
        for (uint32_t x = tid * 4u; x < a.TW; x += kDeliverBlock * 4u) {
            uint4 o = *reinterpret_cast<uint4 *>(dst + x);
            o.x += cnt[x]; o.y += cnt[x + 1]; o.z += cnt[x + 2]; o.w += cnt[x + 3];
            *reinterpret_cast<uint4 *>(dst + x) = o;
        }
    } else {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            const uint32_t bytes_total = a.TW * 4u;
            for (uint32_t off = 0; off < bytes_total; off += 32768u) {
                const uint32_t nb = min(32768u, bytes_total - off);
                const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(cnt) + off;
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;"
                             :: "l"(reinterpret_cast<char *>(dst) + off), "r"(saddr), "r"(nb) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }
    // delivered-event statistics: one atomic per CTA
    __shared__ uint32_t s_red[kDeliverBlock / 32];
    uint32_t d = delivered;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xFFFFFFFFu, d, o);
    if ((tid & 31) == 0) s_red[tid >> 5] = d;
    __syncthreads();
    if (tid == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < kDeliverBlock / 32; ++w) tot += s_red[w];
        if (tot) atomicAdd(&a.stats[1], tot);
    }
    if (a.C != 1u && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Paper-style baseline: warp i delivers spike (i mod |S|) to column block floor(i/|S|)
// (column-wise; here a column block is one tile segment), with global atomics.
__global__ void __launch_bounds__(256) deliver_global_atomics(SimArgs a, uint32_t k,
                                                              const uint32_t *__restrict__ list) {
    const uint64_t t = *a.t0 + k;
    const uint32_t n_sp = a.spcount[t % 3];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x / 32);
    uint32_t *slot = a.ring + ((t + a.delay) % a.D) * a.ring_stride;
    uint32_t delivered = 0;
    for (uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
         w < (uint64_t)a.NT * n_sp; w += nwarps) {
        const uint32_t b = (uint32_t)(w / n_sp), p = (uint32_t)(w % n_sp);
        const uint32_t s = list[p];
        const uint32_t *bp = a.bnd + (uint64_t)s * (a.NT + 1u) + b;
        const uint32_t b0 = bp[0], b1 = bp[1];
        const uint64_t st = a.row_ptr[s] + b0;
        const uint32_t qv = s >= a.n_exc ? 65536u : 1u;
        uint32_t *tile = slot + (uint64_t)b * a.TW;
        for (uint32_t e = lane; e < b1 - b0; e += 32) atomicAdd(tile + a.ent[st + e], qv);
        if (lane == 0) delivered += b1 - b0;
    }
    if (lane == 0 && delivered) atomicAdd(&a.stats[1], (unsigned long long)delivered);
}

// Gathered bitmaps of all ranks -> global spike list + record ring copy.
__global__ void __launch_bounds__(256) bitmap_to_list(SimArgs a, uint32_t k) {
    const uint64_t t = *a.t0 + k;
    const uint32_t idx = blockIdx.x * 256 + threadIdx.x;
    const uint32_t nw = a.G * a.W;
    const uint32_t word = idx < nw ? a.gather[idx] : 0u;
    if (idx < nw) a.record[(t % a.record_steps) * (uint64_t)nw + idx] = word;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t cnt = __popc(word), incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
    }
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_base;
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < 8; ++w) { const uint32_t cw = s_w[w]; s_w[w] = tot; tot += cw; }
        s_base = tot ? atomicAdd(&a.spcount[t % 3], tot) : 0u;
        if (blockIdx.x == 0) a.spcount[(t + 1) % 3] = 0u;
    }
    __syncthreads();
    uint32_t pos = s_base + s_w[warp] + incl - cnt;
    if (word) {
        const uint32_t r = idx / a.W, wl = idx % a.W;
        uint32_t bits = word;
        while (bits) {
            const uint32_t bit = __ffs(bits) - 1;
            bits &= bits - 1;
            a.splist[pos++] = (uint32_t)local_to_global((uint64_t)wl * 32 + bit, r, a.G, a.S);
        }
    }
}

__global__ void advance_kernel(uint64_t *t0, uint32_t steps) { *t0 += steps; }

// ------------------------------------------------------------------ launchers
cudaError_t launch_update(const SimArgs &a, uint32_t k, bool produce_list, cudaStream_t s) {
    const uint32_t threads = a.W * 32u;
    const uint32_t grid = (threads + kUpdateBlock - 1) / kUpdateBlock;
    switch (a.model) {
    case 1: update_kernel<1><<<grid, kUpdateBlock, 0, s>>>(a, k, produce_list); break;
    case 2: update_kernel<2><<<grid, kUpdateBlock, 0, s>>>(a, k, produce_list); break;
    case 4: update_kernel<4><<<grid, kUpdateBlock, 0, s>>>(a, k, produce_list); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

size_t deliver_smem_bytes(uint32_t TW) {
    const uint32_t tw_pad = (TW + 3u) & ~3u;
    return (size_t)(tw_pad + 1) * 4 + (size_t)kDescChunk * 12 + 16;
}

static uint32_t pick_group(const SimArgs &a, double mean_seg) {
    (void)a;
    if (mean_seg <= 12) return 4;
    if (mean_seg <= 28) return 8;
    if (mean_seg <= 60) return 16;
    return 32;
}

cudaError_t prepare_deliver(uint32_t TW) {
    const int bytes = (int)deliver_smem_bytes(TW);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(deliver_tiled<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))) return e;
    if ((e = cudaFuncSetAttribute(deliver_tiled<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))) return e;
    if ((e = cudaFuncSetAttribute(deliver_tiled<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes))) return e;
    return cudaFuncSetAttribute(deliver_tiled<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

cudaError_t launch_deliver(const SimArgs &a, uint32_t k, double mean_seg, int n_sm, cudaStream_t s) {
    const uint32_t *list = a.splist;
    if (a.global_atomics) {
        deliver_global_atomics<<<n_sm * 8, 256, 0, s>>>(a, k, list);
        return cudaGetLastError();
    }
    const size_t smem = deliver_smem_bytes(a.TW);
    const uint32_t grid = a.NT * a.C;
    switch (pick_group(a, mean_seg)) {
    case 4: deliver_tiled<4><<<grid, kDeliverBlock, smem, s>>>(a, k, list); break;
    case 8: deliver_tiled<8><<<grid, kDeliverBlock, smem, s>>>(a, k, list); break;
    case 16: deliver_tiled<16><<<grid, kDeliverBlock, smem, s>>>(a, k, list); break;
    default: deliver_tiled<32><<<grid, kDeliverBlock, smem, s>>>(a, k, list); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_bitmap_to_list(const SimArgs &a, uint32_t k, cudaStream_t s) {
    const uint32_t nw = a.G * a.W;
    bitmap_to_list<<<(nw + 255) / 256, 256, 0, s>>>(a, k);
    return cudaGetLastError();
}

cudaError_t launch_advance(uint64_t *t0, uint32_t steps, cudaStream_t s) {
    advance_kernel<<<1, 1, 0, s>>>(t0, steps);
    return cudaGetLastError();
}

}  // namespace spice
