// sim.cu — per-step kernels of the Spice hot path on sm_100a.
//
// One CTA owns one destination tile of TW consecutive local targets (SURVEY §8(a) a3,
// PAPER.md:198-200 "cache-aware": concurrent writes stay inside one narrow destination
// band — here the band is a shared-memory tile).
//
//   k_update<M>      neuron update of a tile for step t (a1; Listing 1):
//                    4 neurons per thread (one Philox call covers 4 consecutive IDs),
//                    4-bit nibbles OR-reduced into 32-bit bitmap words, spikes appended
//                    to the tile's own list region (no global atomics)
//   k_deliver        destination-tiled delivery of step t (a3): per-tile lists of segment
//                    descriptors of the spiking rows, expanded per warp into a ring of
//                    16-byte windows of u16 offsets, shared-memory atomicAdd of packed
//                    receptor counts, then the tile is added to the input ring slot t + delay
//   k_deliver_plastic Brunel+ (a4): potentiation, depression and delivery of a tile
//   k_fused<M,V>     deliver(t) + update(t+1) of the same tile in one CTA (G = 1): with
//                    delay 1 the tile's inputs never leave shared memory; one launch per
//                    step, the kernel boundary is the step barrier
//   k_global_atomics paper-style column-wise warps with global atomics:
//                    the A/B baseline
//   k_b2l            gathered per-rank bitmaps -> global spike list (a2, G > 1)
//
// Floating point: every operation of the neuron update is an explicit round-to-nearest
// intrinsic in the order fixed by DESIGN.md readings R3-R5 (no contraction), so results
// are bit-identical to the fp32 oracle.
#include <algorithm>

#include "spice_internal.cuh"
#include "spice_launch.h"

namespace spice {

// --------------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    return x;
}

// Exclusive scan of arr[0..n) in shared memory (n <= kBlock * 8); arr[n] = total.
__device__ __forceinline__ void block_exclusive_scan(uint32_t *arr, uint32_t n, uint32_t *s_tmp) {
    const uint32_t tid = threadIdx.x, per = (n + kBlock - 1) / kBlock;
    const uint32_t lo = min(n, tid * per), hi = min(n, lo + per);
    uint32_t sum = 0;
    for (uint32_t x = lo; x < hi; ++x) sum += arr[x];
    const uint32_t incl = warp_incl_scan(sum);
    if ((tid & 31) == 31) s_tmp[tid >> 5] = incl;
    __syncthreads();
    if (tid < 32) {
        const uint32_t v = tid < kBlock / 32 ? s_tmp[tid] : 0u;
        const uint32_t wi = warp_incl_scan(v);
        if (tid < kBlock / 32) s_tmp[tid] = wi - v;
    }
    __syncthreads();
    uint32_t run = s_tmp[tid >> 5] + incl - sum;
    for (uint32_t x = lo; x < hi; ++x) { const uint32_t c = arr[x]; arr[x] = run; run += c; }
    if (tid == kBlock - 1) arr[n] = run;
    __syncthreads();
}

// t mod m for a step counter: 32-bit remainder while t < 2^32 (the 64-bit remainder is a
// ~100-instruction subroutine every thread would run once per launch)
__device__ __forceinline__ uint64_t mod32(uint64_t t, uint32_t m) {
    return (t >> 32) ? t % m : (uint64_t)((uint32_t)t % m);
}
// Step-indexed buffers that CTAs of different steps may touch at once (spike lists, the
// Brunel+ pre state): three copies by t mod 3, so that a CTA one step ahead (the persistent
// kernels' split barrier) never writes the copy a slower CTA still reads
__device__ __forceinline__ uint32_t lslot(uint64_t t) {   // t mod 3 (2^32 = 1 mod 3: fold the halves)
    const uint64_t x = (t >> 32) + (t & 0xFFFFFFFFull);
    const uint32_t y = (uint32_t)(x >> 32) + (uint32_t)x;      // (no wrap: x < 2^33)
    return y % 3u;
}
// t mod m with the host-computed M = floor((2^64 - 1) / m) + 1: for 32-bit t the remainder
// is the high word of (M t mod 2^64) m (exact for every 32-bit t and m; Lemire, Kaser and
// Kurz 2019, "Faster remainder by direct computation") -- two multiplies instead of the
// ~20-instruction reciprocal sequence of a runtime-divisor remainder
__device__ __forceinline__ uint64_t modm(uint64_t t, uint32_t m, uint64_t M) {
    if (t >> 32) return t % m;
    return __umul64hi(M * (uint32_t)t, m);
}
#define modD(a, t) modm((t), (a).D, (a).mD)
#define modR(a, t) modm((t), (a).record_steps, (a).mR)

__device__ __forceinline__ uint4 ld_stream_v4(const uint16_t *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t philox_word(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                                const SimArgs &a, uint32_t which) {
    return word_of(philox4x32_10(make_uint4(w0, w1, w2, w3), a.key0, a.key1), which);
}

// ------------------------------------------------------------------ neuron update
// Where a tile's neuron state lives during the update: the global SoA arrays (base 0) or
// shared-memory copies of the tile slice [base, base + TW) staged by TMA bulk copies.
struct StatePtrs {
    float *v, *ge, *gi;
    uint32_t *ref, *acc;
    uint32_t base;
};
__device__ __forceinline__ StatePtrs global_state(const SimArgs &a) {
    return StatePtrs{a.v, a.ge, a.gi, a.ref, a.acc, 0u};
}
// Update the 4 consecutive owned neurons i0..i0+3 (i0 % 4 == 0) for step t with packed
// input counts c[4]; returns the spike nibble.  State arrays are padded to NT*TW.
template <int MODEL>
__device__ __forceinline__ uint32_t update4(const SimArgs &a, const StatePtrs &sp, uint64_t t, uint32_t i0,
                                            const uint32_t c[4], const long long pin[4],
                                            const uint64_t *ptab, bool acc_done, int forced) {
    const uint32_t li = i0 - sp.base;                  // index into the state arrays
    const ModelConst &m = a.mc;
    const uint32_t j0 = a.G == 1 ? i0 : (uint32_t)local_to_global(i0, a.rank, a.G, a.S);   // multiple of 4
    uint32_t valid = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) valid |= (i0 + e < a.n_own ? 1u : 0u) << e;
    uint32_t fbits = 0;                                // forced: teacher-forcing mode of step t
    if (forced) fbits = (a.force_bits[i0 >> 5] >> (i0 & 31)) & 0xFu;
    uint32_t spk = 0;
    if (MODEL == 4) {                                   // Synth (reading R12)
#ifndef SPICE_ABLATE_PHILOX
        const uint4 x = philox4x32_10(make_uint4(j0 >> 2, (uint32_t)t, 0u, kTagFire), a.key0, a.key1);
#else
        const uint4 x = make_uint4(j0 * 0x9E3779B9u, (uint32_t)t * 0x85EBCA6Bu, j0 ^ (uint32_t)t, j0 + (uint32_t)t);
#endif
        if (!acc_done) {                                // (else applied by update_tile's batched pass)
            uint4 acc = *reinterpret_cast<const uint4 *>(sp.acc + li);
            acc.x += c[0]; acc.y += c[1]; acc.z += c[2]; acc.w += c[3];
            *reinterpret_cast<uint4 *>(sp.acc + li) = acc;
        }
        spk = ((uint64_t)x.x < m.thr_fire ? 1u : 0u) | ((uint64_t)x.y < m.thr_fire ? 2u : 0u) |
              ((uint64_t)x.z < m.thr_fire ? 4u : 0u) | ((uint64_t)x.w < m.thr_fire ? 8u : 0u);
        if (forced == 1) spk = fbits; else if (forced == 2) spk |= fbits;
    } else if (MODEL == 1) {                            // Vogels-Abbott COBA (readings R3-R5)
        float4 v4 = *reinterpret_cast<const float4 *>(sp.v + li);
        float4 ge4 = *reinterpret_cast<const float4 *>(sp.ge + li);
        float4 gi4 = *reinterpret_cast<const float4 *>(sp.gi + li);
        uint4 rf4 = *reinterpret_cast<const uint4 *>(sp.ref + li);
        float *vv = &v4.x, *gev = &ge4.x, *giv = &gi4.x;
        uint32_t *rfv = &rf4.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t ne = c[e] & 0xFFFFu, ni = c[e] >> 16;
            float ge = __fadd_rn(gev[e], __fmul_rn(m.dge, __uint2float_rn(ne)));
            float gi = __fadd_rn(giv[e], __fmul_rn(m.dgi, __uint2float_rn(ni)));
            float v = vv[e];
            uint32_t ref = rfv[e];
            bool s = false;
            if (ref > 0u) {
                ref -= 1u;
                v = m.Vr;
            } else {
                const float ta = __fsub_rn(m.EL, v);
                const float tb = __fmul_rn(ge, __fsub_rn(m.Ee, v));
                const float tc = __fmul_rn(gi, __fsub_rn(m.Ei, v));
                v = __fadd_rn(v, __fmul_rn(m.h, __fadd_rn(__fadd_rn(ta, tb), tc)));
                s = v >= m.Vt;
            }
            const bool fb = (fbits >> e) & 1u;
            if (forced == 1) s = fb; else if (forced == 2) s = s || fb;
            if (s) { v = m.Vr; ref = m.R; }
            gev[e] = __fsub_rn(ge, __fmul_rn(m.ke, ge));
            giv[e] = __fsub_rn(gi, __fmul_rn(m.ki, gi));
            vv[e] = v;
            rfv[e] = ref;
            spk |= (s ? 1u : 0u) << e;
        }
        *reinterpret_cast<float4 *>(sp.v + li) = v4;
        *reinterpret_cast<float4 *>(sp.ge + li) = ge4;
        *reinterpret_cast<float4 *>(sp.gi + li) = gi4;
        *reinterpret_cast<uint4 *>(sp.ref + li) = rf4;
    } else {                                            // Brunel model A (readings R3-R5, R12)
        float4 v4 = *reinterpret_cast<const float4 *>(sp.v + li);
        uint4 rf4 = *reinterpret_cast<const uint4 *>(sp.ref + li);
        float *vv = &v4.x;
        uint32_t *rfv = &rf4.x;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (rfv[0] == 0u || rfv[1] == 0u || rfv[2] == 0u || rfv[3] == 0u)
            x = philox4x32_10(make_uint4(j0 >> 2, (uint32_t)t, 0u, kTagExt), a.key0, a.key1);
        // n_ext = min{k : x < T_k} = #{k : T_k <= x} (the table is non-decreasing and ends with
        // 2^32): a branch-free binary search, the four neurons' searches interleaved (one
        // dependent table load per halving instead of a walk of ~lambda loads per neuron)
        uint32_t nx[4] = {0u, 0u, 0u, 0u};
        for (uint32_t step = a.mc.ptab_half; step > 0; step >>= 1) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t q = nx[e] + step - 1u;
                if (q < a.mc.ptab_len && ptab[q] <= (uint64_t)word_of(x, e)) nx[e] += step;
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float v = vv[e];
            uint32_t ref = rfv[e];
            bool s = false;
            if (ref > 0u) {
                ref -= 1u;
                v = m.Vr;                              // input and drive discarded
            } else {
                const uint32_t next = nx[e];
                const uint32_t ne = c[e] & 0xFFFFu, ni = c[e] >> 16;
                v = __fadd_rn(v, __fmul_rn(m.h, __fsub_rn(m.EL, v)));
                v = __fadd_rn(v, __fmul_rn(m.JE, __uint2float_rn(ne + next)));
                v = __fadd_rn(v, __fmul_rn(m.JI, __uint2float_rn(ni)));
                if (MODEL == 3) v = __fadd_rn(v, __fmul_rn(__ll2float_rn(pin[e]), 2.3283064365386963e-10f));
                s = v >= m.theta;
            }
            const bool fb = (fbits >> e) & 1u;
            if (forced == 1) s = fb; else if (forced == 2) s = s || fb;
            if (s) { v = m.Vr; ref = m.R; }
            vv[e] = v;
            rfv[e] = ref;
            spk |= (s ? 1u : 0u) << e;
        }
        *reinterpret_cast<float4 *>(sp.v + li) = v4;
        *reinterpret_cast<uint4 *>(sp.ref + li) = rf4;
    }
    return spk & valid;
}

// Diagnostics (SPICE_PHASES=1 with a library built with -DSPICE_PHASES_BUILD=1, see
// tools/phases.py): thread 0 of every fused-kernel CTA accumulates the SM
// clock offset of phase boundary `slot` from the kernel start into ptimes[cta*16 + slot];
// slot 13 counts launches, 14/15 hold %globaltimer at start/end of the last launch.
__device__ __forceinline__ long long &phase_c0() { __shared__ long long c0; return c0; }
__device__ __forceinline__ void phase_mark(const SimArgs &a, int slot, uint32_t who = 0) {
#if !SPICE_PHASES_BUILD
    (void)a; (void)slot; (void)who;   // compiled out: even predicated-off marks cost issue slots (ncu r01u)
#else
    if (a.ptimes && threadIdx.x == who) {
        unsigned long long *p = a.ptimes + blockIdx.x * 16u;
        // (fire-and-forget reductions: a load-add-store would stall the marking thread for
        //  a global round trip and distort the next interval)
        if (slot == 0) {
            phase_c0() = clock64();
            unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            p[14] = g; atomicAdd(p + 13, 1ull);
        } else {
            atomicAdd(p + slot, (unsigned long long)(clock64() - phase_c0()));
            if (slot == 12) { unsigned long long g; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g)); p[15] = g; }
        }
    }
#endif
}

// Update every neuron of tile b for step t.  Inputs come from `cnt` (shared memory, the
// tile's counts) or, when cnt == nullptr, from input ring slot t mod D (read and cleared).
// ------------------------------------------------------------------ delivery
struct DeliverSmem {
    uint4 *wbuf;       // [warps * kStages * 32 lanes] cp.async window stages
    uint32_t *cnt;     // [TW + kDummy] tile counters (+ padding-sentinel dummies)
    uint64_t *dsm;     // [dcap] the CTA's segment descriptors (delivery phase)
    uint32_t *stage;   // [kStageWords] bnd-row staging of the update phase (aliases dsm)
    uint32_t *pref;    // [NR + 1] region prefix
    uint32_t *tmp;     // [32]
    uint32_t *prod;    // [prod_words]
};

__device__ __forceinline__ uint32_t region_of(const uint32_t *pref, uint32_t nr, uint32_t p) {
    uint32_t lo = 0, hi = nr;             // largest r with pref[r] <= p
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pref[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr uint32_t kRing = 512;                        // ring entries per warp (power of 2)
// spike IDs of the update kept in shared memory for the descriptor pass: the words of the
// delivery area past the descriptor staging (kStageWords) and before the end of the rings
constexpr uint32_t kSidCap = (kBlock / 32) * kRing - kStageWords;
// synth fast path: shared-memory area of the producer warps (spike IDs, then row staging)
constexpr uint32_t kSynthSid = 2048;

// Descriptor transposition (G = 1, padded layout): for the n spikes of region b (this
// tile's spikes), one pass loads every spike's bnd row (a warp per spike, coalesced),
// row start and out-degree, staged in smem (CH spikes at a time; CH covers a whole step's
// tile list in the common case), then writes, for every destination tile bb, the
// descriptors desc[par][bb][b][q0 .. q0+CH) with coalesced stores.  Delivery CTAs then read
// their descriptors contiguously.  Returns (to thread 0) the spikes' delivered-event count.
// Staging geometry of write_descriptors (shared with the update's early row staging).
struct DescStage { uint32_t rowlen, rs4, CH; };
__device__ __forceinline__ DescStage desc_stage(const SimArgs &a) {
    DescStage d;
    d.rowlen = a.NT + 1u;
    // staged rows keep their global 16-byte phase h = (s rowlen) mod 4 so that they are
    // copied in 16-byte chunks (the bnd array carries 4 words of tail padding)
    d.rs4 = (d.rowlen + 6u) & ~3u;
    d.CH = max(1u, (uint32_t)kStageWords / (d.rs4 + 3u));
    return d;
}
// SUB: run by the pth threads ptid = 0 .. pth - 1 of a producer warp group (named barrier 1)
// while the other warps of the CTA deliver (synth fast path); sid_cap: the capacity of sid_s.
template <bool SUB = false>
__device__ __forceinline__ uint64_t write_descriptors(const SimArgs &a, uint64_t t, uint32_t b, uint32_t n,
                                  const uint32_t *region, uint64_t *region_rows, uint32_t *stage,
                                  bool marks = false, const uint32_t *sid_s = nullptr,
                                  uint32_t ptid = threadIdx.x, uint32_t pth = kBlock, uint32_t sid_cap = kSidCap,
                                  uint32_t stage_words = kStageWords) {
    auto barrier = [&]() {
        if constexpr (SUB) asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");
        else __syncthreads();
    };
    if (sid_s && n <= sid_cap) region = sid_s;          // the spike IDs' shared-memory copy
    const uint32_t lane = ptid & 31, warp = ptid >> 5, nwp = pth / 32;
    const uint32_t dbuf = (uint32_t)mod32(t, 3);        // descriptor lists: 3 buffers by step
    // dense per-tile lists: this CTA's n descriptors go to [off, off + n) of every
    // destination tile's list of step t (one atomic on the step's counter)
    // (the reservation's latency overlaps the row loads: thread 0 publishes it after issuing
    //  its copies; the pass's closing barrier orders it before the descriptor writes)
    __shared__ uint32_t s_off;
    uint32_t off_reg = 0;
    if (ptid == 0 && n) off_reg = atomicAdd(&a.dcount[t & 3u], n);
    if (marks) phase_mark(a, 11, threadIdx.x - ptid);
    const DescStage ds = desc_stage(a);
    const uint32_t rowlen = ds.rowlen, rs4 = ds.rs4;
    const uint32_t CH = SUB ? max(1u, stage_words / (rs4 + 3u)) : ds.CH;
    uint64_t *srow = reinterpret_cast<uint64_t *>(stage + CH * rs4);
    uint32_t *sdeg = reinterpret_cast<uint32_t *>(srow + CH);
    const uint4 *bnd4 = reinterpret_cast<const uint4 *>(a.bnd);
    uint64_t dsum = 0;
    for (uint32_t q0 = 0; q0 < n; q0 += CH) {
        const uint32_t nq = min(CH, n - q0);
        barrier();
        // every load of the pass in flight at once (cp.async, no register round trips)
        for (uint32_t ql = warp; ql < nq; ql += nwp) {                    // one warp per spike row
            const uint32_t s = region[q0 + ql];
            const uint64_t g0 = (uint64_t)s * rowlen;
            const uint64_t k0 = g0 >> 2, nk = ((g0 + rowlen - 1) >> 2) - k0 + 1;
            for (uint32_t k = lane; k < nk; k += 32)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" :: "r"(smem_u32(stage + ql * rs4 + 4u * k)), "l"(bnd4 + k0 + k) : "memory");
            if (lane == 0) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_u32(srow + ql)), "l"(a.row_ptr + s) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(smem_u32(sdeg + ql)), "l"(a.deg + s) : "memory");
            }
        }
        if (ptid == 0 && q0 == 0) s_off = off_reg;
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        barrier();
        SPICE_CHECK((uint64_t)s_off + n <= a.dstride);
        if (marks) phase_mark(a, 10, threadIdx.x - ptid);
        if (warp == 0)
            for (uint32_t ql = lane; ql < nq; ql += 32) { region_rows[q0 + ql] = srow[ql]; dsum += sdeg[ql]; }
        for (uint32_t j0 = 0; j0 < nq; j0 += 32) {          // lane = spike; per-spike values hoisted
            const uint32_t ql = j0 + lane;
            if (ql < nq) {                                   // padded: rs, lo, hi multiples of 8
                const uint32_t rsw = (uint32_t)(srow[ql] >> kWinShift);
                const uint32_t ih = region[q0 + ql] >= a.n_exc ? 0x80000000u : 0u;
                const uint32_t *row = stage + ql * rs4 + (uint32_t)(((uint64_t)region[q0 + ql] * rowlen) & 3u);
                uint2 *dst = reinterpret_cast<uint2 *>(a.desc + (uint64_t)dbuf * a.NT * a.dstride + s_off + q0 + ql);
                for (uint32_t bb = warp; bb < a.NT; bb += nwp) {
                    const uint32_t lo = row[bb], hi = row[bb + 1];
                    dst[(uint64_t)bb * a.dstride] = make_uint2(rsw + (lo >> kWinShift), ((hi - lo) >> kWinShift) | ih);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xFFFFFFFFu, dsum, o);
    barrier();
    return dsum;                                       // valid in warp 0
}

// Update the owned neurons [lo, lo + width) for step t (a tile, or one CTA's slice of a
// cluster tile); b is the CTA's spike-list region / counter slot.
// cl_c < kMaxCluster: cnt is this CTA's slice of a cluster tile whose C = a.C CTAs each hold
// partial counts for it; the update adds the peers' partials (distributed shared memory).
// DESC = true: compile only the padded-layout descriptor path (the fused G = 1 kernel's
// variants), keeping the inlined code on the hot path small (instruction-fetch stalls were
// the largest stall class of the fused kernel, ncu r01u).
__device__ __forceinline__ void post_state_update(const SimArgs &a, uint64_t t, uint32_t i0, uint32_t nib);   // (Brunel+)

// SUB: run by the pth threads ptid = 0 .. pth - 1 of a warp group (named barrier 1) while
// the CTA's other warps deliver the current step (delay >= 2: the update of t + 1 does not
// depend on the delivery of t -- the timestep grouping of P:290 inside one kernel).
// Brunel drive: the Poisson inversion table in shared memory (one instance per kernel)
__device__ __forceinline__ uint64_t *ptab_smem() { __shared__ uint64_t s_ptab[kPtabSmem]; return s_ptab; }
// ... staged by the whole CTA (a step kernel's prologue: the table is constant)
__device__ __forceinline__ bool stage_ptab(const SimArgs &a) {
    if (a.mc.ptab_len > kPtabSmem) return false;
    for (uint32_t x = threadIdx.x; x < a.mc.ptab_len; x += kBlock) ptab_smem()[x] = a.mc.ptab[x];
    return true;
}

template <int MODEL, bool DESC = false, bool SUB = false>
__device__ __forceinline__ void update_tile(const SimArgs &a, uint64_t t, uint32_t b, uint32_t lo, uint32_t width,
                            const uint32_t *cnt, bool write_list, uint32_t *s_count, uint32_t *stage,
                            const StatePtrs *staged = nullptr, bool marks = false,
                            uint32_t cl_c = kMaxCluster, uint32_t *sid_s = nullptr, uint32_t *bm_s = nullptr,
                            uint32_t ptid = threadIdx.x, uint32_t pth = kBlock, uint32_t stage_words = kStageWords,
                            bool ptab_staged = false) {
    auto sync = [&]() {
        if constexpr (SUB) asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");
        else __syncthreads();
    };
    const StatePtrs sp = staged ? *staged : global_state(a);
    const uint32_t tid = ptid, lane = tid & 31;
    const uint32_t span = lo < a.W * 32u ? min(width, a.W * 32u - lo) : 0u;   // bitmap coverage
    const uint32_t par = lslot(t);
    uint32_t *region = a.sl_ids + ((uint64_t)par * a.NR + b) * a.RS;
    uint64_t *region_rows = a.sl_rows + ((uint64_t)par * a.NR + b) * a.RS;
    uint32_t *bm = a.G == 1 ? a.record + modR(a, t) * (uint64_t)a.W : a.sendbuf;
    uint32_t *ring_slot = a.ring + modD(a, t) * a.ring_stride + lo;
    // Brunel drive: the Poisson inversion table in shared memory (the walk is a chain of
    // dependent loads per neuron); ptab_staged: the kernel's prologue copied it already
    const uint64_t *ptab = a.mc.ptab;
    if ((MODEL == 2 || MODEL == 3) && a.mc.ptab_len <= kPtabSmem) {
        if (!ptab_staged) {
            for (uint32_t x = tid; x < a.mc.ptab_len; x += pth) ptab_smem()[x] = a.mc.ptab[x];
            sync();
        }
        ptab = ptab_smem();
    }
    const bool acc_done = false;
    const int forced = a.force_ctl[0] == t ? (int)a.force_ctl[1] : 0;   // once per CTA, not per neuron
    // synth accumulators (global, one RMW per neuron): the next iteration's values are loaded
    // one iteration ahead, so the loop pays the load latency once rather than per iteration
    constexpr bool ACC_PF = MODEL == 4 && SPICE_ACC_PREFETCH;
    const bool acc_pf = ACC_PF && staged == nullptr;
    uint4 acc_next = make_uint4(0u, 0u, 0u, 0u);
    if (acc_pf && 4u * tid < span && lo + 4u * tid < a.n_own)
        acc_next = *reinterpret_cast<const uint4 *>(a.acc + lo + 4u * tid);
    for (uint32_t x0 = 0; x0 < span; x0 += 4u * pth) {         // uniform trip count per CTA
        if (x0 + 4u * (tid & ~31u) >= span) continue;             // whole warp past the slice
        const uint32_t x4 = x0 + 4u * tid;
        uint32_t nib = 0;
        const bool act = x4 < span && lo + x4 < a.n_own;
        uint4 acc_cur = acc_next;
        if (acc_pf) {
            const uint32_t xn = x4 + 4u * pth;
            if (xn < span && lo + xn < a.n_own) acc_next = *reinterpret_cast<const uint4 *>(a.acc + lo + xn);
        }
        if (act) {
            uint32_t c[4];
            long long pin[4] = {0, 0, 0, 0};
            if (MODEL == 3) {
                long long *ps = a.pring + modD(a, t) * a.ring_stride + lo + x4;
#pragma unroll
                for (int e = 0; e < 4; ++e) { pin[e] = ps[e]; ps[e] = 0; }
            }
            if (cnt) {
                uint4 cv = *reinterpret_cast<const uint4 *>(cnt + x4);
#ifndef SPICE_ABLATE_PEER
                if (cl_c < kMaxCluster) {
#else
                if (false) {
#endif
                    const uint32_t la = (uint32_t)__cvta_generic_to_shared(cnt + x4);
#pragma unroll 1
                    for (uint32_t k = 1; k < a.C; ++k) {
                        uint32_t peer = cl_c + k;
                        if (peer >= a.C) peer -= a.C;
                        uint32_t ra;
                        uint4 v;
                        asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(peer));
                        asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ra));
                        cv.x += v.x; cv.y += v.y; cv.z += v.z; cv.w += v.w;
                    }
                }
                if (a.dly) {                              // longer-delay arrivals of earlier steps
                    const uint4 rv = *reinterpret_cast<const uint4 *>(ring_slot + x4);
                    *reinterpret_cast<uint4 *>(ring_slot + x4) = make_uint4(0, 0, 0, 0);
                    cv.x += rv.x; cv.y += rv.y; cv.z += rv.z; cv.w += rv.w;
                }
                c[0] = cv.x; c[1] = cv.y; c[2] = cv.z; c[3] = cv.w;
            } else {
                const uint4 cv = *reinterpret_cast<const uint4 *>(ring_slot + x4);
                *reinterpret_cast<uint4 *>(ring_slot + x4) = make_uint4(0, 0, 0, 0);
                c[0] = cv.x; c[1] = cv.y; c[2] = cv.z; c[3] = cv.w;
            }
            if (acc_pf) {                                  // (update4 then skips its own RMW)
                acc_cur.x += c[0]; acc_cur.y += c[1]; acc_cur.z += c[2]; acc_cur.w += c[3];
#ifndef SPICE_ABLATE_ACC
                *reinterpret_cast<uint4 *>(a.acc + lo + x4) = acc_cur;
#endif
            }
            nib = update4<MODEL>(a, sp, t, lo + x4, c, pin, ptab, acc_done || acc_pf, forced);
            if constexpr (MODEL == 3) post_state_update(a, t, lo + x4, nib);
        }
        // 8 lanes x 4 bits -> one 32-neuron bitmap word
        uint32_t w = nib << (4u * (lane & 7u));
        w |= __shfl_xor_sync(0xFFFFFFFFu, w, 1);
        w |= __shfl_xor_sync(0xFFFFFFFFu, w, 2);
        w |= __shfl_xor_sync(0xFFFFFFFFu, w, 4);
        if ((lane & 7u) == 0 && x4 < span) {
            if (a.peers) {                                // PEER exchange: straight into every
                const uint64_t o = ((uint64_t)(t & 1) * a.G + a.rank) * a.W + ((lo + x4) >> 5);
                for (uint32_t r = 0; r < a.G; ++r) a.peers[r][o] = w;   // rank's window (NVLink stores)
            } else {
                bm[(lo + x4) >> 5] = w;
            }
            if (bm_s) bm_s[x4 >> 5] = w;                  // (k_small: the step's bitmap in smem)
        }
        // append spikes to this tile's list region (warp-aggregated smem counter)
        const uint32_t nsp = __popc(nib);
        const uint32_t incl = warp_incl_scan(nsp);
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        if (tot) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(s_count, tot);
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            if (write_list && nib) {
                uint32_t pos = base + incl - nsp;
                const uint32_t j0 = a.G == 1 ? lo + x4 : (uint32_t)local_to_global(lo + x4, a.rank, a.G, a.S);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if ((nib >> e) & 1u) {
                        region[pos] = j0 + e;
                        if (sid_s && pos < kSidCap) sid_s[pos] = j0 + e;
                        ++pos;
                    }
            }
        }
    }
    sync();
    if (marks) phase_mark(a, 7);
    if (staged) {                                          // staged state -> global (coalesced)
        const uint32_t nw = width / 4;
        for (uint32_t x = tid; x < nw; x += pth) {
            const uint32_t g = lo + 4 * x;
            if (MODEL == 4) reinterpret_cast<uint4 *>(a.acc + g)[0] = reinterpret_cast<const uint4 *>(sp.acc)[x];
            if (MODEL != 4) reinterpret_cast<float4 *>(a.v + g)[0] = reinterpret_cast<const float4 *>(sp.v)[x];
            if (MODEL != 4) reinterpret_cast<uint4 *>(a.ref + g)[0] = reinterpret_cast<const uint4 *>(sp.ref)[x];
            if (MODEL == 1) reinterpret_cast<float4 *>(a.ge + g)[0] = reinterpret_cast<const float4 *>(sp.ge)[x];
            if (MODEL == 1) reinterpret_cast<float4 *>(a.gi + g)[0] = reinterpret_cast<const float4 *>(sp.gi)[x];
        }
        sync();
    }
    const uint32_t n_tile = *s_count;
    if (tid == 0) {
        if (write_list) a.sl_counts[par * a.NR + b] = n_tile;
        if (n_tile) atomicAdd(&a.fired_cta[b], (unsigned long long)n_tile);   // RED: no load on the path
    }
    if (!DESC && write_list && !a.desc && MODEL != 3 && a.row_ptr) {   // row starts of the spikes, all at once
        uint32_t dsum = 0;                                // (the descriptor pass loads them itself;
        for (uint32_t q = tid; q < n_tile; q += pth) {    //  Brunel+ staging loads row_ptr itself)
            const uint32_t s = region[q];
            region_rows[q] = a.row_ptr[s];
            if (a.deg) dsum += a.deg[s];
        }
        if (a.deg) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xFFFFFFFFu, dsum, o);
            if (lane == 0 && dsum) atomicAdd(&a.delivered_cta[b], (unsigned long long)dsum);
        }
        sync();
    }
    if (marks) phase_mark(a, 8);
    if (write_list && (DESC || a.desc)) {                 // padded layout: delivered events (out-degrees)
        uint64_t dsum;
        if constexpr (SUB) dsum = write_descriptors<true>(a, t, b, n_tile, region, region_rows, stage, false, sid_s,
                                                          ptid, pth, kSidCap, stage_words);
        else dsum = write_descriptors(a, t, b, n_tile, region, region_rows, stage, marks, sid_s);
        if (tid == 0 && dsum) atomicAdd(&a.delivered_cta[b], (unsigned long long)dsum);
    }
    if (marks) phase_mark(a, 9);
    sync();
    if (tid == 0) *s_count = 0;
}

template <int MODEL>
__device__ __forceinline__ void update_tile_sub(const SimArgs &a, uint64_t t, uint32_t b, uint32_t lo, uint32_t width,
                                                uint32_t *s_count, uint32_t *stage, uint32_t ptid, uint32_t pth) {
    update_tile<MODEL, false, true>(a, t, b, lo, width, nullptr, true, s_count, stage, nullptr, false, kMaxCluster,
                                    nullptr, nullptr, ptid, pth);
}

// Eight unconditional shared-memory reductions of one padded 16-byte window (sentinel
// entries land in the dummy counters past the tile).  Padded entries are byte offsets
// (tiles up to kMaxPadTile) or, WORD = true, counter indices (cluster tiles up to
// kMaxPadTileWord).
// (debug builds: every entry, padding sentinels included, addresses a counter of the tile
//  or one of its dummies)
template <bool WORD>
__device__ __forceinline__ void check_window(const uint4 v, uint32_t tw) {
#if SPICE_CHECKS
    const uint32_t lim = WORD ? tw + kDummy : (tw + kDummy) * 4u;
    const uint32_t w8[4] = {v.x, v.y, v.z, v.w};
    for (int u = 0; u < 8; ++u) SPICE_CHECK(((w8[u >> 1] >> (16 * (u & 1))) & 0xFFFFu) < lim);
#else
    (void)v; (void)tw;
#endif
}
template <bool WORD = false>
__device__ __forceinline__ void accumulate_window(uint32_t cnt_s, const uint4 v, uint32_t q) {
    uint32_t a0, a1, a2, a3, a4, a5, a6, a7;
    if (WORD) {
        a0 = cnt_s + ((v.x & 0xFFFFu) << 2); a1 = cnt_s + ((v.x >> 14) & ~3u);
        a2 = cnt_s + ((v.y & 0xFFFFu) << 2); a3 = cnt_s + ((v.y >> 14) & ~3u);
        a4 = cnt_s + ((v.z & 0xFFFFu) << 2); a5 = cnt_s + ((v.z >> 14) & ~3u);
        a6 = cnt_s + ((v.w & 0xFFFFu) << 2); a7 = cnt_s + ((v.w >> 14) & ~3u);
    } else {
        a0 = cnt_s + (v.x & 0xFFFFu); a1 = cnt_s + (v.x >> 16);
        a2 = cnt_s + (v.y & 0xFFFFu); a3 = cnt_s + (v.y >> 16);
        a4 = cnt_s + (v.z & 0xFFFFu); a5 = cnt_s + (v.z >> 16);
        a6 = cnt_s + (v.w & 0xFFFFu); a7 = cnt_s + (v.w >> 16);
    }
    asm volatile(
        "red.shared.add.u32 [%0], %8;\n\t"
        "red.shared.add.u32 [%1], %8;\n\t"
        "red.shared.add.u32 [%2], %8;\n\t"
        "red.shared.add.u32 [%3], %8;\n\t"
        "red.shared.add.u32 [%4], %8;\n\t"
        "red.shared.add.u32 [%5], %8;\n\t"
        "red.shared.add.u32 [%6], %8;\n\t"
        "red.shared.add.u32 [%7], %8;"
        :: "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7), "r"(q)
        : "memory");
}

// Ring delivery (G = 1, padded layout; default).  Consumes the segment-descriptor lists of
// write_descriptors (one 8-byte descriptor per spike x tile, cheap to produce) but streams
// windows like a window list: each warp expands its segment descriptors, 32 at a time,
// into a per-warp shared-memory ring of window entries (window index | inh << 31; each
// lane stores its own segment's windows at its exclusive-prefix position), then consumes
// the ring 64 entries per iteration with lane L taking entries L and L + 32 (consecutive
// windows of a segment sit in one load instruction and coalesce into one L1 line lookup),
// the next iteration's two window loads in flight while the current windows are reduced.
// ------------------------------------------------------- synth step, G = 1 (fast path)
// The synth drive is input-independent (reading R12: neuron j fires at step t iff
// Philox(j>>2, t, 0, 5)[j&3] < floor(a 2^32)), so the fused kernel of step t computes
// the spikes of step t + 1 on kFireWarps warps WHILE the other warps deliver step t (the
// draws are ALU work, the delivery is memory-bound), stages them as a slice bitmap and
// spike list in shared memory and starts the copies of their rows' segment bounds; at the
// end it publishes them (record bitmap, spike list, descriptors) and the update of step
// t + 1 reduces to the accumulator: acc += this step's input.  Every output (record
// bitmap, spike lists, descriptors, counters) is the one the general update writes.
// (Measured: in the prologue, before the grid dependency, the draws were on the step's
// critical path -- the CTA whose SM frees last pays them: 3.7 us of a 24.7 us step.)
__device__ __forceinline__ void synth_fire(const SimArgs &a, uint64_t t1, uint32_t b, uint32_t lo, uint32_t width,
                                           uint32_t *sfire, uint32_t *sid_s, uint32_t *s_count, uint32_t sid_cap,
                                           uint32_t tid = threadIdx.x, uint32_t nth = kBlock) {
    const uint32_t lane = tid & 31;
    const uint32_t span = lo < a.W * 32u ? min(width, a.W * 32u - lo) : 0u;
    const int forced = a.force_ctl[0] == t1 ? (int)a.force_ctl[1] : 0;
    for (uint32_t x0 = 0; x0 < span; x0 += 4u * nth) {
        if (x0 + 4u * (tid & ~31u) >= span) continue;            // whole warp past the slice
        const uint32_t x4 = x0 + 4u * tid;
        uint32_t nib = 0;
        if (x4 < span && lo + x4 < a.n_own) {
            const uint32_t j0 = lo + x4;                           // G = 1: local = global
            const uint4 x = philox4x32_10(make_uint4(j0 >> 2, (uint32_t)t1, 0u, kTagFire), a.key0, a.key1);
            const uint64_t thr = a.mc.thr_fire;
            nib = ((uint64_t)x.x < thr ? 1u : 0u) | ((uint64_t)x.y < thr ? 2u : 0u) |
                  ((uint64_t)x.z < thr ? 4u : 0u) | ((uint64_t)x.w < thr ? 8u : 0u);
            if (forced) {
                const uint32_t fb = (a.force_bits[j0 >> 5] >> (j0 & 31)) & 0xFu;
                nib = forced == 1 ? fb : (nib | fb);
            }
            uint32_t valid = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) valid |= (j0 + e < a.n_own ? 1u : 0u) << e;
            nib &= valid;
        }
        // bitmap words and list positions from four ballots (bit e of every lane's nibble):
        // no shuffles -- the fire warps run beside the delivery, whose shared-memory atomics
        // keep the MIO queue (shuffles, shared memory) busy
        uint32_t m[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) m[e] = __ballot_sync(0xFFFFFFFFu, (nib >> e) & 1u);
        if (lane < 4) {                              // word `lane` of the warp's 128 neurons:
            uint32_t w = 0;                          // lanes 8 lane .. 8 lane + 7, bit 4 L' + e
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                uint32_t x = (m[e] >> (8u * lane)) & 0xFFu;                 // spread 8 bits to 4i
                x = (x | (x << 12)) & 0x000F000Fu;
                x = (x | (x << 6)) & 0x03030303u;
                x = (x | (x << 3)) & 0x11111111u;
                w |= x << e;
            }
            const uint32_t xw = x0 + 4u * (tid & ~31u) + 32u * lane;
            if (xw < span) sfire[xw >> 5] = w;
        }
        const uint32_t lt = (1u << lane) - 1u;
        const uint32_t tot = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
        if (tot) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(s_count, tot);
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            uint32_t pos = base + __popc(m[0] & lt) + __popc(m[1] & lt) + __popc(m[2] & lt) + __popc(m[3] & lt);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if ((nib >> e) & 1u) {                   // (shared list only: the global
                    if (pos < sid_cap) sid_s[pos] = lo + x4 + e;   //  region is written by synth_publish
                    ++pos;                               //  when the list overflows, else unused)
                }
        }
    }
}

// acc += input of step t1 for the owned neurons [lo, lo + width): the tile counters (plus
// the C - 1 peers' partial counts through distributed shared memory, plus longer-delay ring
// arrivals) or, cnt == nullptr, the ring slot of t1 (read and cleared).
__device__ __forceinline__ void synth_accumulate(const SimArgs &a, uint64_t t1, uint32_t lo, uint32_t width,
                                                 const uint32_t *cnt, uint32_t cl_c,
                                                 uint32_t tid = threadIdx.x, uint32_t nth = kBlock) {
    uint32_t *ring_slot = a.ring + modD(a, t1) * a.ring_stride + lo;
    const uint32_t span = min(width, a.n_own > lo ? a.n_own - lo : 0u);
    if (cnt && !a.dly && (cl_c >= kMaxCluster || a.C == 2) && span <= 4u * nth * 4u) {
        // common case: every load of the thread's <= 4 groups in flight before any add
        uint4 acc[4], cv[4], pv[4];
        const uint32_t peer = cl_c < kMaxCluster ? cl_c ^ 1u : 0u;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const uint32_t x4 = 4u * tid + (uint32_t)it * 4u * nth;
            if (x4 < span) {
                acc[it] = *reinterpret_cast<const uint4 *>(a.acc + lo + x4);
                cv[it] = *reinterpret_cast<const uint4 *>(cnt + x4);
                pv[it] = make_uint4(0u, 0u, 0u, 0u);
                if (cl_c < kMaxCluster) {
                    uint32_t ra;
                    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"((uint32_t)__cvta_generic_to_shared(cnt + x4)), "r"(peer));
                    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(pv[it].x), "=r"(pv[it].y), "=r"(pv[it].z), "=r"(pv[it].w) : "r"(ra));
                }
            }
        }
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const uint32_t x4 = 4u * tid + (uint32_t)it * 4u * nth;
            if (x4 < span) {
                uint4 o = acc[it];
                o.x += cv[it].x + pv[it].x; o.y += cv[it].y + pv[it].y;
                o.z += cv[it].z + pv[it].z; o.w += cv[it].w + pv[it].w;
                *reinterpret_cast<uint4 *>(a.acc + lo + x4) = o;
            }
        }
        return;
    }
    for (uint32_t x4 = 4u * tid; x4 < span; x4 += 4u * nth) {
        uint4 acc = *reinterpret_cast<const uint4 *>(a.acc + lo + x4);
        uint4 cv;
        if (cnt) {
            cv = *reinterpret_cast<const uint4 *>(cnt + x4);
            if (cl_c < kMaxCluster) {
                const uint32_t la = (uint32_t)__cvta_generic_to_shared(cnt + x4);
#pragma unroll 1
                for (uint32_t k = 1; k < a.C; ++k) {
                    uint32_t peer = cl_c + k;
                    if (peer >= a.C) peer -= a.C;
                    uint32_t ra;
                    uint4 v;
                    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(peer));
                    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ra));
                    cv.x += v.x; cv.y += v.y; cv.z += v.z; cv.w += v.w;
                }
            }
            if (a.dly) {
                const uint4 rv = *reinterpret_cast<const uint4 *>(ring_slot + x4);
                *reinterpret_cast<uint4 *>(ring_slot + x4) = make_uint4(0, 0, 0, 0);
                cv.x += rv.x; cv.y += rv.y; cv.z += rv.z; cv.w += rv.w;
            }
        } else {
            cv = *reinterpret_cast<const uint4 *>(ring_slot + x4);
            *reinterpret_cast<uint4 *>(ring_slot + x4) = make_uint4(0, 0, 0, 0);
        }
        acc.x += cv.x; acc.y += cv.y; acc.z += cv.z; acc.w += cv.w;
        *reinterpret_cast<uint4 *>(a.acc + lo + x4) = acc;
    }
}

// Synth fast path, producer warps: in the prologue (the spike IDs of step t + 1 are known,
// the descriptor buffer and counter of t + 1 are free: the kernels that used them finished
// before this one could launch) reserve the step's slots in the dense per-tile lists and
// start the cp.async copies of the spiking rows' segment bounds, row starts and out-degrees;
// they land while the CTA delivers.  Only when the rows fit one staging pass (else the
// general write_descriptors runs at the end).
struct SynthStage { uint32_t rs4, CH; };
__device__ __forceinline__ SynthStage synth_stage(const SimArgs &a, uint32_t stage_words) {
    const DescStage ds = desc_stage(a);
    return SynthStage{ds.rs4, max(1u, stage_words / (ds.rs4 + 3u))};
}
__device__ __forceinline__ void synth_rows_prefetch(const SimArgs &a, uint64_t t1, uint32_t n, const uint32_t *sid_s,
                                                    uint32_t *stage, uint32_t stage_words, uint32_t ptid, uint32_t pth,
                                                    uint32_t *s_off) {
    const SynthStage ss = synth_stage(a, stage_words);
    if (n == 0 || n > ss.CH || n > kSynthSid) return;
    const uint32_t lane = ptid & 31, warp = ptid >> 5, nwp = pth / 32, rowlen = a.NT + 1u;
    uint64_t *srow = reinterpret_cast<uint64_t *>(stage + ss.CH * ss.rs4);
    uint32_t *sdeg = reinterpret_cast<uint32_t *>(srow + ss.CH);
    const uint4 *bnd4 = reinterpret_cast<const uint4 *>(a.bnd);
    for (uint32_t ql = warp; ql < n; ql += nwp) {
        const uint32_t sj = sid_s[ql];
        const uint64_t g0 = (uint64_t)sj * rowlen;
        const uint64_t k0 = g0 >> 2, nk = ((g0 + rowlen - 1) >> 2) - k0 + 1;
        for (uint32_t kk = lane; kk < nk; kk += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" :: "r"(smem_u32(stage + ql * ss.rs4 + 4u * kk)), "l"(bnd4 + k0 + kk) : "memory");
        if (lane == 0) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_u32(srow + ql)), "l"(a.row_ptr + sj) : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(smem_u32(sdeg + ql)), "l"(a.deg + sj) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // the list reservation last: its round trip stalls only the reserving warp, after its copies
    if (ptid == pth - 32) *s_off = atomicAdd(&a.dcount[t1 & 3u], n);
}
// ... and at the end of the step: wait for the copies, write the descriptors.  Returns the
// spikes' delivered-event count (valid in producer warp 0).
__device__ __forceinline__ uint64_t synth_descriptors(const SimArgs &a, uint64_t t1, uint32_t n, const uint32_t *sid_s,
                                                      uint64_t *region_rows, uint32_t *stage, uint32_t stage_words,
                                                      uint32_t ptid, uint32_t pth, uint32_t off) {
    const SynthStage ss = synth_stage(a, stage_words);
    const uint32_t lane = ptid & 31, warp = ptid >> 5, nwp = pth / 32, rowlen = a.NT + 1u;
    uint64_t *srow = reinterpret_cast<uint64_t *>(stage + ss.CH * ss.rs4);
    uint32_t *sdeg = reinterpret_cast<uint32_t *>(srow + ss.CH);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");
    phase_mark(a, 6, threadIdx.x - ptid);            // (diagnostics: rows staged)
    uint64_t dsum = 0;
    if (warp == 0)                                   // (the list's row starts are not needed on
        for (uint32_t ql = lane; ql < n; ql += 32) dsum += sdeg[ql];   //  the descriptor path)
    (void)region_rows;
    const uint32_t dbuf = (uint32_t)mod32(t1, 3);
    SPICE_CHECK((uint64_t)off + n <= a.dstride);
    for (uint32_t j0 = 0; j0 < n; j0 += 32) {
        const uint32_t ql = j0 + lane;
        if (ql < n) {
            const uint32_t rsw = (uint32_t)(srow[ql] >> kWinShift);
            const uint32_t sj = sid_s[ql];
            const uint32_t ih = sj >= a.n_exc ? 0x80000000u : 0u;
            const uint32_t *row = stage + ql * ss.rs4 + (uint32_t)(((uint64_t)sj * rowlen) & 3u);
            uint2 *dst = reinterpret_cast<uint2 *>(a.desc + (uint64_t)dbuf * a.NT * a.dstride + off + ql);
            for (uint32_t bb = warp; bb < a.NT; bb += nwp) {
                const uint32_t lo = row[bb], hi = row[bb + 1];
                dst[(uint64_t)bb * a.dstride] = make_uint2(rsw + (lo >> kWinShift), ((hi - lo) >> kWinShift) | ih);
            }
        }
    }
    phase_mark(a, 7, threadIdx.x - ptid);            // (diagnostics: descriptors issued)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_xor_sync(0xFFFFFFFFu, dsum, o);
    return dsum;
}

#ifndef SPICE_FIRE_WARPS
#define SPICE_FIRE_WARPS 9
#endif
constexpr uint32_t kFireWarps = SPICE_FIRE_WARPS;   // synth: warps drawing + publishing step t + 1 during delivery

// Publication of step t + 1 by the fire warps (ptid < pth), right after they drew its
// spikes -- still during the delivery of step t: record bitmap, spike list and count, and
// the descriptors of its spiking rows (into descriptor buffer (t + 1) mod 3, which no
// kernel reads before the delivery of t + 1; the list slots were reserved by
// synth_rows_prefetch).  The end of the step is then only the accumulator update.
__device__ __forceinline__ void synth_publish(const SimArgs &a, uint64_t t, uint32_t b, uint32_t lo,
                                             const uint32_t *s_fire, const uint32_t *sid_s, uint32_t n,
                                             uint32_t *stage, uint32_t stage_words, uint32_t s_off,
                                             uint32_t ptid, uint32_t pth) {
    const uint64_t t1 = t + 1;
    const uint32_t par1 = lslot(t1);
    uint32_t *bm = a.record + modR(a, t1) * (uint64_t)a.W;
    const uint32_t nwd = (min(a.TWs, a.W * 32u > lo ? a.W * 32u - lo : 0u) + 31u) / 32u;
    uint32_t *region = a.sl_ids + ((uint64_t)par1 * a.NR + b) * a.RS;
    uint64_t *region_rows = a.sl_rows + ((uint64_t)par1 * a.NR + b) * a.RS;
    for (uint32_t x = ptid; x < nwd; x += pth) bm[(lo >> 5) + x] = s_fire[x];
    if (n > kSynthSid) {                             // (more spikes than the shared list holds:
        __shared__ uint32_t s_pos;                   //  synth_fire listed only the first ones)
        if (ptid == 0) s_pos = 0;
        asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");
        for (uint32_t x = ptid; x < nwd; x += pth) {
            uint32_t w = s_fire[x];
            uint32_t p = w ? atomicAdd(&s_pos, __popc(w)) : 0u;
            while (w) { region[p++] = lo + 32u * x + (uint32_t)(__ffs(w) - 1); w &= w - 1u; }
        }
    }
    if (ptid == 0) {
        a.sl_counts[par1 * a.NR + b] = n;
        if (n) atomicAdd(&a.fired_cta[b], (unsigned long long)n);
    }
    asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");   // (region complete)
    phase_mark(a, 5, threadIdx.x - ptid);            // (diagnostics: bitmap + list published)
    const bool staged = n > 0 && n <= synth_stage(a, stage_words).CH && n <= kSynthSid;   // (synth_rows_prefetch)
    const uint64_t dsum = staged ? synth_descriptors(a, t1, n, sid_s, region_rows, stage, stage_words, ptid, pth, s_off)
                                 : write_descriptors<true>(a, t1, b, n, region, region_rows, stage, true, sid_s,
                                                           ptid, pth, kSynthSid, stage_words);
    if (ptid == 0 && dsum) atomicAdd(&a.delivered_cta[b], (unsigned long long)dsum);
}

struct Win { uint4 a, b; };                          // one delivery window (kWin entries; b: kWin = 16)

// Mixed per-synapse delays (reading R19): 8 entries of a window with their delay bytes;
// minimum-delay events go to the tile counters (shared memory), longer ones straight into
// ring slot (t + d) mod D (global red: they are read by the update of step t + d).
template <bool WORD>
__device__ __forceinline__ void accumulate_window_dly(const SimArgs &a, uint32_t cnt_s, const uint4 v, const uint2 dd,
                                                      uint32_t q, uint32_t tD, uint64_t tile_base) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const uint32_t raw = (w[u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
        const uint32_t d = ((u < 4 ? dd.x : dd.y) >> (8 * (u & 3))) & 0xFFu;
        if (d == a.delay) {
            asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(cnt_s + (WORD ? raw << 2 : raw)), "r"(q) : "memory");
        } else {
            uint32_t sl = tD + d;
            if (sl >= a.D) sl -= a.D;
            atomicAdd(a.ring + (uint64_t)sl * a.ring_stride + tile_base + (WORD ? raw : raw >> 2), q);
        }
    }
}

// The step's descriptor count of tile list t (thread 0 may pass it preloaded) and the
// reset of the counter step t + 2's producers use; block-wide.
__device__ __forceinline__ uint32_t delivery_count(const SimArgs &a, uint64_t t, uint32_t b, uint32_t c,
                                                   uint32_t pre_total) {
    __shared__ uint32_t s_total;
    if (threadIdx.x == 0) {
        s_total = pre_total != 0xFFFFFFFFu ? pre_total : a.dcount[t & 3u];
        if (b == 0 && c == 0)                       // next user: step t + 3's producers (two
            a.dcount[(t + 3) & 3u] = 0u;            // kernel boundaries / grid barriers later)
    }
    __syncthreads();
    return s_total;
}

// The per-warp part of ring delivery: warp `warp` of NW delivering warps takes its share
// of the tile list's n_sp visits (no block-wide barriers inside).
template <bool WORD, bool DLY = false>
__device__ __forceinline__ void deliver_ring_core(const SimArgs &a, uint64_t t, uint32_t b, uint32_t c,
                                                  uint32_t *cnt, uint32_t *ring_base, uint32_t n_sp,
                                                  uint32_t warp, uint32_t NW) {
    constexpr uint32_t NONE = 0xFFFFFFFFu;
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
    const uint32_t my = n_sp > c ? (n_sp - c + a.C - 1u) / a.C : 0u;
    const uint32_t v0 = (uint32_t)((uint64_t)my * warp / NW), v1 = (uint32_t)((uint64_t)my * (warp + 1) / NW);
    const uint64_t *dlist = a.desc + ((uint64_t)mod32(t, 3) * a.NT + b) * a.dstride + c;   // visit v -> dlist[v * C]
    uint32_t *ring = ring_base + warp * kRing;
    SPICE_CHECK((uint64_t)my * a.C <= a.dstride);     // (the step's list fits its buffer)
    auto dload = [&](uint32_t vb) -> uint64_t {
        const uint32_t v = vb + lane;
        return v < v1 ? dlist[(uint64_t)v * a.C] : 0ull;
    };
    uint32_t gnext = v0;
    uint64_t dn = dload(v0);
    uint32_t w0 = 0, nw = 0, inh = 0, pre = 0, T = 0, c0 = 0;   // current group, c0 = expanded
    uint32_t head = 0, tail = 0;                                // ring cursors (warp-uniform)
    auto fill = [&](uint32_t want) {                            // expand until >= want queued
        while (tail - head < want) {
            if (c0 >= T) {
                if (gnext >= v1) break;
                const uint64_t d = dn;
                gnext += 32;
                dn = dload(gnext);
                nw = (uint32_t)(d >> 32) & 0x7FFFFFFFu;
                w0 = (uint32_t)d;
                inh = (uint32_t)(d >> 63) << 31;
                const uint32_t incl = warp_incl_scan(nw);
                pre = incl - nw;
                T = __shfl_sync(FULL, incl, 31);
                c0 = 0;
                continue;
            }
            const uint32_t take = min(T - c0, kRing - (tail - head));
            const uint32_t klo = c0 > pre ? c0 - pre : 0u;
            const uint32_t khi = min(pre + nw, c0 + take);
            for (uint32_t k = klo; pre + k < khi; ++k)
                ring[(tail + pre + k - c0) & (kRing - 1)] = (w0 + k) | inh;
            tail += take;
            c0 += take;
        }
        __syncwarp();
    };
    auto entry = [&](uint32_t x) -> uint32_t { return x < tail ? ring[x & (kRing - 1)] : NONE; };
    auto load_win = [&](uint32_t e) -> Win {
        Win w;
        if (e == NONE) { w.a = make_uint4(0, 0, 0, 0); if constexpr (kWin == 16) w.b = w.a; return w; }
        SPICE_CHECK((uint64_t)kWin * ((e & 0x7FFFFFFFu) + 1u) <= a.nnz);
        const uint16_t *p = a.ent + (uint64_t)kWin * (e & 0x7FFFFFFFu);
        w.a = ld_stream_v4(p);
        if constexpr (kWin == 16) w.b = ld_stream_v4(p + 8);
        return w;
    };
    auto load_dly = [&](uint32_t e) -> uint4 {
        if (!DLY || e == NONE) return make_uint4(0, 0, 0, 0);
        const uint8_t *p = a.dly + (uint64_t)kWin * (e & 0x7FFFFFFFu);
        if constexpr (kWin == 16) return *reinterpret_cast<const uint4 *>(p);
        const uint2 d = *reinterpret_cast<const uint2 *>(p);
        return make_uint4(d.x, d.y, 0u, 0u);
    };
    const uint32_t tD = DLY ? (uint32_t)modD(a, t) : 0u;
    const uint64_t tile_base = (uint64_t)b * a.TW;
    constexpr uint32_t RW = SPICE_RW;                  // windows per lane per iteration
    fill(32u * RW);
    uint32_t e[RW];
    Win v[RW];
    uint4 dd[RW];
#pragma unroll
    for (uint32_t r = 0; r < RW; ++r) { e[r] = entry(head + 32u * r + lane); v[r] = load_win(e[r]); dd[r] = load_dly(e[r]); }
    head = min(head + 32u * RW, tail);
    while (__any_sync(FULL, e[0] != NONE)) {
        __syncwarp();
        fill(32u * RW);
        uint32_t x[RW];
        Win nv[RW];
        uint4 nd[RW];
#pragma unroll
        for (uint32_t r = 0; r < RW; ++r) { x[r] = entry(head + 32u * r + lane); nv[r] = load_win(x[r]); nd[r] = load_dly(x[r]); }
        head = min(head + 32u * RW, tail);
#pragma unroll
        for (uint32_t r = 0; r < RW; ++r)
            if (e[r] != NONE) {
                const uint32_t q = (e[r] >> 31) ? 65536u : 1u;
                if (DLY) {
                    accumulate_window_dly<WORD>(a, cnt_s, v[r].a, make_uint2(dd[r].x, dd[r].y), q, tD, tile_base);
                    if constexpr (kWin == 16)
                        accumulate_window_dly<WORD>(a, cnt_s, v[r].b, make_uint2(dd[r].z, dd[r].w), q, tD, tile_base);
                } else {
                    check_window<WORD>(v[r].a, a.TW);
                    accumulate_window<WORD>(cnt_s, v[r].a, q);
                    if constexpr (kWin == 16) accumulate_window<WORD>(cnt_s, v[r].b, q);
                }
            }
#pragma unroll
        for (uint32_t r = 0; r < RW; ++r) { e[r] = x[r]; v[r] = nv[r]; dd[r] = nd[r]; }
    }
}

template <bool WORD, bool DLY = false>
__device__ __forceinline__ void deliver_tile_ring(const SimArgs &a, uint64_t t, uint32_t b, uint32_t c,
                                                  uint32_t *cnt, uint32_t *ring_base, bool marks = false,
                                                  uint32_t pre_total = 0xFFFFFFFFu) {
    const uint32_t n_sp = delivery_count(a, t, b, c, pre_total);
    if (marks) phase_mark(a, 2);
    deliver_ring_core<WORD, DLY>(a, t, b, c, cnt, ring_base, n_sp, threadIdx.x >> 5, kBlock / 32);
    if (marks) phase_mark(a, 4);
    __syncthreads();
    if (marks) phase_mark(a, 5);
}

// ------------------------------------------------------------- Brunel+ STDP
// Reading R13 with event-driven traces: every neuron keeps the step ts of its last spike and
// the trace values just after it (pre: cx = X(ts) + 1 for all N sources, post: cy for the
// owned targets), a trace is read as c P[t - ts].  The eager rule -- (i) every post spike at
// t_p potentiates w += A+ X_pre(t_p) (clamp w_max), (ii) every pre spike at t depresses
// w -= A- Y_post(t) (clamp 0), (iii) w is delivered -- is evaluated LAZILY on the synapse
// stream (north star: "STDP weight updates run on the same synapse stream"): a row is
// processed when its source spikes (potentiation by the post spikes since the row's last
// processing, then depression and delivery) and, so that the post-spike history stays
// bounded, at a fixed flush step every kFlush steps (potentiation only).  Between two
// processings of a row nothing else touches its weights, so every weight sees exactly the
// eager sequence of fp32 operations: GPU == oracle bit for bit.  Post-spike history per
// owned neuron: its last three spike steps (in the post state) and a 2048-step bit ring.
// Every synapse touched by CTA b has its target in tile b: no two CTAs write one weight.
constexpr uint32_t kTraceLen = 8192;      // closed-form trace table (== ORC_TRACE_LEN)
constexpr uint32_t kFlush = 1024;         // row flush period (steps)
constexpr uint32_t kHistWords = 64;       // post-spike bit ring: 2048 steps per neuron
constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ const uint32_t *step_bitmap(const SimArgs &a, uint64_t t) {
    return a.record + modR(a, t) * (uint64_t)a.G * a.W + (uint64_t)a.rank * a.W;
}

__device__ __forceinline__ bool plastic_src(const SimArgs &a, uint32_t s) {
    for (uint32_t q = 0; q < a.npl; ++q)
        if (s >= a.pl[q][0] && s < a.pl[q][1]) return true;
    return false;
}

// Global spike bit of source j in the gathered bitmaps of step t (Listing 1 inverse).
__device__ __forceinline__ bool spiked_global(const SimArgs &a, const uint32_t *gbm, uint32_t j) {
    if (a.G == 1) return (gbm[j >> 5] >> (j & 31)) & 1u;
    const uint32_t r = (j / a.S) % a.G, il = (j / a.S / a.G) * a.S + j % a.S;
    return (gbm[(uint64_t)r * a.W + (il >> 5)] >> (il & 31)) & 1u;
}

// c P[t - ts]: one rounded product (0 before the first spike and past the table)
__device__ __forceinline__ float trace_val(float c, uint32_t ts, uint64_t t, const float *tab) {
    if (ts == kNone) return 0.0f;
    const uint64_t k = t - ts;
    return k < kTraceLen ? __fmul_rn(c, tab[k]) : 0.0f;
}

// The step of row j's last processing before step t: its last spike (< t) or its last
// flush step (< t, steps congruent to j mod kFlush); -1 before any.
__device__ __forceinline__ int64_t row_tproc(uint32_t j, uint64_t t, uint32_t ts_j) {
    int64_t tp = ts_j == kNone ? -1 : (int64_t)ts_j;
    const uint64_t ph = j % kFlush;
    if (t >= 1 && t - 1 >= ph) {
        const int64_t f = (int64_t)(t - 1) - (int64_t)((t - 1 - ph) % kFlush);
        if (f > tp) tp = f;
    }
    return tp;
}

// One potentiation at post spike step tp with the row's pre state (ts_j, cx_j).
// (tabp: the X table, a shared-memory copy on the delivery path)
__device__ __forceinline__ float potentiate_at(const SimArgs &a, const float *tabp, float w, uint64_t tp,
                                               uint32_t ts_j, float cx_j) {
    const float x = trace_val(cx_j, ts_j, tp, tabp);
    const float nw = __fadd_rn(w, __fmul_rn(a.mc.Ap, x));
    return nw < a.mc.wmax ? nw : a.mc.wmax;
}

// Lazy potentiation of one synapse: the post neuron's spikes in (tproc, t], in time order.
// pl = its last three spike steps up to and including t (most recent first, kNone = none);
// older ones come from its bit ring `mask` (only when all three are inside the window).
__device__ __forceinline__ float potentiate_lazy(const SimArgs &a, const float *tabp, float w, int64_t tproc,
                                                 uint32_t ts_j, float cx_j,
                                                 uint32_t p1, uint32_t p2, uint32_t p3, const uint32_t *mask) {
    if (ts_j == kNone || p1 == kNone || (int64_t)p1 <= tproc) return w;     // X = 0 / no post spike
#ifndef SPICE_ABLATE_MASK
    if (p3 != kNone && (int64_t)p3 > tproc) {
#else
    if (false) {
#endif
        for (uint64_t s = (uint64_t)(tproc + 1); s < p3;) {                  // spikes before p3
            const uint32_t wi = (uint32_t)((s >> 5) % kHistWords);
            const uint32_t b0 = (uint32_t)(s & 31u);
            const uint64_t wend = (s | 31u) + 1;                             // first step of the next word
            const uint32_t nb = (uint32_t)((wend < p3 ? wend : (uint64_t)p3) - s);   // bits b0 .. b0 + nb - 1
            uint32_t bits = mask[wi] >> b0;
            if (nb < 32) bits &= (1u << nb) - 1u;
            while (bits) {
                const uint32_t k = __ffs(bits) - 1;
                bits &= bits - 1u;
                w = potentiate_at(a, tabp, w, s + k, ts_j, cx_j);
            }
            s = wend;
        }
    }
    if (p3 != kNone && (int64_t)p3 > tproc) w = potentiate_at(a, tabp, w, p3, ts_j, cx_j);
    if (p2 != kNone && (int64_t)p2 > tproc) w = potentiate_at(a, tabp, w, p2, ts_j, cx_j);
    return potentiate_at(a, tabp, w, p1, ts_j, cx_j);
}

// Pre state of every global source for step t + 1 (CTA slices of [0, N)): a source that
// spiked at t restarts its trace, cx = X(t) + 1 (the oracle's event-driven update).
__device__ __forceinline__ void pre_state_pass(const SimArgs &a, uint64_t t, const float *tabp,
                                               uint32_t ptid = threadIdx.x, uint32_t pth = kBlock) {
    const uint32_t *gbm = a.record + modR(a, t) * (uint64_t)a.G * a.W;
    const uint32_t *ots = a.pre_ts + lslot(t) * (uint64_t)a.N;
    const float *oc = a.pre_c + lslot(t) * (uint64_t)a.N;
    uint32_t *nts = a.pre_ts + lslot(t + 1) * (uint64_t)a.N;
    float *nc = a.pre_c + lslot(t + 1) * (uint64_t)a.N;
    const uint32_t per = (a.N + gridDim.x - 1) / gridDim.x;
    const uint32_t j0 = blockIdx.x * per, j1 = min(a.N, j0 + per);
    for (uint32_t j = j0 + ptid; j < j1; j += pth) {
        uint32_t ts = ots[j];
        float c = oc[j];
        if (spiked_global(a, gbm, j)) {
            c = __fadd_rn(trace_val(c, ts, t, tabp), 1.0f);
            ts = (uint32_t)t;
        }
        nts[j] = ts;
        nc[j] = c;
    }
}

// Post state of the owned neurons [i0, i0 + 4) at their update of step t (spike nibble):
// last three spike steps and cy, double-buffered by step parity; the bit ring word of t is
// rewritten at every 32-step boundary and or-ed on a spike.
__device__ __forceinline__ void post_state_update(const SimArgs &a, uint64_t t, uint32_t i0, uint32_t nib) {
    const uint4 *o = reinterpret_cast<const uint4 *>(a.post) + (t & 1) * a.ring_stride + i0;
    uint4 *n = reinterpret_cast<uint4 *>(a.post) + ((t + 1) & 1) * a.ring_stride + i0;
    const uint32_t wi = (uint32_t)((t >> 5) % kHistWords), bit = (uint32_t)(t & 31u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (i0 + e >= a.n_own) break;
        uint4 st = o[e];
        const bool s = (nib >> e) & 1u;
        if (s) {
            const float y = trace_val(__uint_as_float(st.w), st.x, t, a.tab_m);
            st = make_uint4((uint32_t)t, st.x, st.y, __float_as_uint(__fadd_rn(y, 1.0f)));
        }
        n[e] = st;
        uint32_t *m = a.post_mask + (uint64_t)(i0 + e) * kHistWords + wi;
        if (bit == 0) *m = s ? 1u : 0u;
        else if (s) *m |= 1u << bit;
    }
}

__device__ __forceinline__ void plastic_deliver(const SimArgs &a, uint32_t *cnt, uint32_t *plo, uint32_t *phi,
                                                const float *ys, uint32_t e, uint32_t off, uint32_t fl, float wv,
                                                uint32_t tD, uint64_t tile_base) {
    uint64_t gslot = ~0ull;                          // longer per-synapse delay: ring slot t + d
    if (a.dly) {
        const uint32_t d = a.dly[e];
        if (d != a.delay) {
            uint32_t sl = tD + d;
            if (sl >= a.D) sl -= a.D;
            gslot = (uint64_t)sl * a.ring_stride + tile_base + off;
        }
    }
    if (wv >= 0.0f) {
        float nw = __fsub_rn(wv, __fmul_rn(a.mc.Am, ys[off]));     // (ii)
        nw = nw > 0.0f ? nw : 0.0f;
        a.w[e] = nw;
        // (iii) rint(w 2^32): w 2^32 is exact in fp32 (a power-of-two scaling), so the fp32
        // round-to-nearest-even conversion equals the fp64 one
        const uint64_t q = (uint64_t)__float2ll_rn(nw * 4294967296.0f);
        if (gslot != ~0ull) {
            atomicAdd(reinterpret_cast<unsigned long long *>(a.pring + gslot), (unsigned long long)q);
            return;
        }
        if (a.pl_split) {                            // fire-and-forget: no returned value
            atomicAdd(&plo[off], (uint32_t)q & 0xFFFFu);
            atomicAdd(&phi[off], (uint32_t)(q >> 16));
            return;
        }
        const uint32_t lo = (uint32_t)q, hi = (uint32_t)(q >> 32);
        const uint32_t old = atomicAdd(&plo[off], lo);
        const uint32_t carry = old + lo < old ? 1u : 0u;
        if (hi + carry) atomicAdd(&phi[off], hi + carry);
    } else {
        if (gslot != ~0ull) atomicAdd(a.ring + gslot, (fl & 1u) ? 65536u : 1u);
        else atomicAdd(&cnt[off], (fl & 1u) ? 65536u : 1u);
    }
}

struct PlasticSmem {
    uint32_t *cnt, *plo, *phi;     // [TW] counters, fixed-point low / high words
    float *ys;                     // [TW] Y(t) of the tile's neurons
    uint32_t *p1, *p2, *p3;        // [TW] their last three spike steps up to t
    uint32_t *pref, *tmp, *stage;
    float *tabp;                   // [kTraceLen] the X trace table (constant: loaded before the
                                   // dependent-launch wait)
    uint32_t *cst;                 // [kPlChunks + 1] first segment of each 32-event chunk
};

// (i)-(iii) of step t for tile b, one flattened event space over all threads: the
// (segment, entry) pairs of the step's spiking rows and of its flush rows into tile b.
// Consecutive events of a segment are consecutive threads (entry and weight loads coalesce).
// Plastic synapses (weight >= 0; static ones hold the sentinel -1): lazy potentiation, then
// on spike rows depression, store and delivery as fixed point rint(w 2^32) summed exactly in
// two u32 shared words (low word with carry detection: native 32-bit shared atomics); on
// flush rows the potentiated weight is stored.  Static synapses of spike rows add their
// packed receptor count.
constexpr uint32_t kPlSeg = 1800;                     // segments staged per pass (6 words each)
// flush-row list capacity (the stage's last 64 words are the overlapped update's scratch)
constexpr uint32_t kPlFlush = kStageWords - 6 * kPlSeg - 2 - 64;
#ifndef SPICE_PL_U
#define SPICE_PL_U 2
#endif
constexpr uint32_t kPlU = SPICE_PL_U;                 // events in flight per thread
constexpr uint32_t kPlChunks = 4096;                  // chunk-start table: passes of <= 2^17 events

// upd_count != nullptr (fused kernel, delay >= 2, one staging pass): the last kUpdWarps warps
// run the update of step t + 1 meanwhile (it reads input slot t + 1, complete since delay >= 2,
// and post state parity t + 1, already staged) and *upd_done is set.
#ifndef SPICE_PL_UPD_WARPS
#define SPICE_PL_UPD_WARPS 4
#endif
constexpr uint32_t kUpdWarps = SPICE_PL_UPD_WARPS;   // Brunel+: update warps beside the event warps
#ifndef SPICE_OVL_UPD_WARPS
#define SPICE_OVL_UPD_WARPS 12
#endif
constexpr uint32_t kOvlUpdWarps = SPICE_OVL_UPD_WARPS;   // Vogels / Brunel delay >= 2: update warps beside the delivery
template <int MODEL>
__device__ __forceinline__ void update_tile_sub(const SimArgs &a, uint64_t t, uint32_t b, uint32_t lo, uint32_t width,
                                                uint32_t *s_count, uint32_t *stage, uint32_t ptid, uint32_t pth);
__device__ __forceinline__ void grid_arrive_add(const SimArgs &a, uint32_t i, uint32_t payload);   // (below)
// arrive != kNone (persistent kernel): once the overlapped update of t + 1 and the pre state
// for t + 1 are written, the update warps arrive at grid barrier `arrive` ("t + 1 published")
__device__ __forceinline__ uint32_t deliver_tile_plastic(const SimArgs &a, uint64_t t, uint32_t b,
                                                         const PlasticSmem &sm, bool marks = false,
                                                         uint32_t *upd_count = nullptr, bool *upd_done = nullptr,
                                                         uint32_t arrive = 0xFFFFFFFFu) {
    const uint32_t tid = threadIdx.x;
    const uint32_t par = lslot(t);
    uint32_t *pref = sm.pref, *tmp = sm.tmp, *stage = sm.stage;
    const uint32_t *bm = step_bitmap(a, t);
    const uint32_t *gbm = a.record + modR(a, t) * (uint64_t)a.G * a.W;
    const uint32_t *pts = a.pre_ts + lslot(t) * (uint64_t)a.N;
    const float *pc = a.pre_c + lslot(t) * (uint64_t)a.N;
    const uint64_t tile_base = (uint64_t)b * a.TW;
    for (uint32_t r = tid; r < a.NR; r += kBlock) pref[r] = a.sl_counts[par * a.NR + r];
    // the tile's post neurons before step t's spikes (post state parity t) plus their spike at t
    const uint4 *post = reinterpret_cast<const uint4 *>(a.post) + (t & 1) * a.ring_stride + tile_base;
    for (uint32_t x = tid; x < a.TW; x += kBlock) {
        float y = 0.0f;
        uint32_t q1 = kNone, q2 = kNone, q3 = kNone;
        if (tile_base + x < a.n_own) {
            const uint4 st = post[x];
            y = trace_val(__uint_as_float(st.w), st.x, t, a.tab_m);
            const uint32_t i = (uint32_t)tile_base + x;
            if ((bm[i >> 5] >> (i & 31)) & 1u) { q1 = (uint32_t)t; q2 = st.x; q3 = st.y; }
            else { q1 = st.x; q2 = st.y; q3 = st.z; }
        }
        sm.ys[x] = y; sm.p1[x] = q1; sm.p2[x] = q2; sm.p3[x] = q3;
    }
    // flush rows of step t: plastic sources j = t mod kFlush + k kFlush that do not spike at t
    __shared__ uint32_t s_nfl;
    if (tid == 0) s_nfl = 0;
    uint32_t *flist = stage + 6 * kPlSeg + 2;
    __syncthreads();
    {
        const uint32_t ph = (uint32_t)(t % kFlush);
        const uint32_t ncand = ph < a.N ? (a.N - ph + kFlush - 1) / kFlush : 0u;
        for (uint32_t k = tid; k < ncand; k += kBlock) {
            const uint32_t j = ph + k * kFlush;
            if (plastic_src(a, j) && !spiked_global(a, gbm, j)) {
                const uint32_t pos = atomicAdd(&s_nfl, 1u);
                if (pos < kPlFlush) flist[pos] = j;
            }
        }
    }
    block_exclusive_scan(pref, a.NR, tmp);       // (its barriers also publish flist)
    if (marks) phase_mark(a, 2);
    const uint32_t n_sp = pref[a.NR];
    const uint32_t n_fl = min(s_nfl, kPlFlush);
    const uint32_t nseg = n_sp + n_fl;
    const uint64_t lbase = (uint64_t)par * a.NR * a.RS;
    const uint32_t tD = a.dly ? (uint32_t)modD(a, t) : 0u;
    uint32_t *sst = stage, *slen = stage + kPlSeg, *sfl = stage + 2 * kPlSeg + 1;
    float *sx = reinterpret_cast<float *>(stage + 3 * kPlSeg + 1);
    uint32_t *sts = stage + 4 * kPlSeg + 1;
    int32_t *stp = reinterpret_cast<int32_t *>(stage + 5 * kPlSeg + 1);
    uint32_t delivered = 0;
    for (uint32_t q0 = 0; q0 < nseg; q0 += kPlSeg) {
        const uint32_t nq = min(kPlSeg, nseg - q0);
        __syncthreads();                          // previous pass done with the staging
        for (uint32_t q = tid; q < nq; q += kBlock) {
            const uint32_t p = q0 + q;
            uint32_t s;
            uint64_t rs;
            uint32_t fl;
            if (p < n_sp) {                       // spike row
                const uint32_t r = region_of(pref, a.NR, p);
                const uint64_t slot = lbase + (uint64_t)r * a.RS + (p - pref[r]);
                s = a.sl_ids[slot];
                fl = 0u;
            } else {                              // flush row
                s = flist[p - n_sp];
                fl = 4u;
            }
            rs = a.row_ptr[s];
            const uint32_t *bp = a.bnd + (uint64_t)s * (a.NT + 1u) + b;
            const uint32_t lo = bp[0], hi = bp[1];
            const bool pls = plastic_src(a, s);
            sst[q] = (uint32_t)(rs + lo);
            slen[q] = hi - lo;
            sfl[q] = fl | (s >= a.n_exc ? 1u : 0u) | (pls ? 2u : 0u);
            const uint32_t ts_j = pls ? pts[s] : kNone;
            sts[q] = ts_j;
            sx[q] = pls ? pc[s] : 0.0f;
            stp[q] = (int32_t)row_tproc(s, t, ts_j);
        }
        __syncthreads();
        block_exclusive_scan(slen, nq, tmp);      // slen -> event prefix
        const uint32_t ne = slen[nq];
        // first segment of every 32-event chunk (one search per chunk instead of per event;
        // an event walks forward from its chunk's start over the few boundaries inside it)
        const bool chunked = ne <= 32u * kPlChunks;
        if (chunked) {
            for (uint32_t c = tid; c < (ne + 31u) / 32u; c += kBlock) {
                const uint32_t f = c * 32u;
                uint32_t lo = 0, h = nq;
                while (h - lo > 1) { const uint32_t m = (lo + h) >> 1; if (slen[m] <= f) lo = m; else h = m; }
                sm.cst[c] = lo;
            }
            __syncthreads();
        }
        if (marks) phase_mark(a, 3);
        // (fused, delay >= 2, single pass) the update of t + 1 on the last kUpdWarps warps
        const bool ovl = upd_count && a.delay >= 2 && nseg <= kPlSeg;
        uint32_t etid = tid, eth = kBlock;
        if (ovl) {
            eth = kBlock - kUpdWarps * 32;
            if (tid >= eth) {
                update_tile_sub<3>(a, t + 1, b, b * a.TW, a.TW, upd_count, sm.stage + kStageWords - 64,
                                   tid - eth, kUpdWarps * 32);
                // then the pre state for t + 1 (independent of the delivery: it writes the
                // other parity and reads step t's spikes)
                pre_state_pass(a, t, sm.tabp, tid - eth, kUpdWarps * 32);
                *upd_done = true;
                if (arrive != kNone) {
                    asm volatile("bar.sync 1, %0;" :: "r"(kUpdWarps * 32) : "memory");
                    if (tid == eth)
                        grid_arrive_add(a, arrive, 0u);
                }
                if (marks) phase_mark(a, 8, eth);
                continue;                         // (nseg <= kPlSeg: this was the only pass)
            }
        }
        for (uint32_t f0 = etid; f0 < ne; f0 += eth * kPlU) {
            uint32_t e[kPlU], off[kPlU], l[kPlU];
            float wv[kPlU];
#pragma unroll
            for (uint32_t u = 0; u < kPlU; ++u) {     // indices (shared memory) + loads
                const uint32_t f = f0 + u * eth;
                l[u] = kNone;
                if (f < ne) {
                    uint32_t lo;                      // largest q with slen[q] <= f (slen[nq] = ne > f)
                    if (chunked) {
                        lo = sm.cst[f >> 5];
                        while (slen[lo + 1] <= f) ++lo;
                    } else {
                        lo = 0;
                        uint32_t h = nq;
                        while (h - lo > 1) { const uint32_t m = (lo + h) >> 1; if (slen[m] <= f) lo = m; else h = m; }
                    }
                    l[u] = lo;
                    e[u] = sst[lo] + (f - slen[lo]);
                    SPICE_CHECK(e[u] < a.nnz);
                    off[u] = a.ent[e[u]];
                    SPICE_CHECK(off[u] < a.TW);
                    wv[u] = (sfl[lo] & 2u) ? a.w[e[u]] : -1.0f;
                }
            }
#pragma unroll
            for (uint32_t u = 0; u < kPlU; ++u) {
                if (l[u] == kNone) continue;
                const uint32_t fl = sfl[l[u]];
                float w = wv[u];
#ifndef SPICE_ABLATE_POT
                if (w >= 0.0f)                        // (i), lazily: post spikes since the last processing
#else
                if (false)
#endif
                    w = potentiate_lazy(a, sm.tabp, w, stp[l[u]], sts[l[u]], sx[l[u]], sm.p1[off[u]], sm.p2[off[u]],
                                        sm.p3[off[u]], a.post_mask + (tile_base + off[u]) * kHistWords);
                if (fl & 4u) {                        // flush row: potentiation only
                    if (w >= 0.0f && w != wv[u]) a.w[e[u]] = w;
                } else {
#ifndef SPICE_ABLATE_DEL
                    plastic_deliver(a, sm.cnt, sm.plo, sm.phi, sm.ys, e[u], off[u], fl, w, tD, tile_base);
#else
                    if (w == 12345.0f) a.w[e[u]] = w;
#endif
                }
            }
        }
        if (marks) phase_mark(a, 7);
        // delivered events: the spike rows' entries of this pass
        if (tid == 0) {
            const uint32_t sp_end = n_sp > q0 ? min(nq, n_sp - q0) : 0u;
            delivered += slen[sp_end];
        }
    }
    __syncthreads();
    if (marks) phase_mark(a, 4);
    if (!(upd_done && *upd_done)) pre_state_pass(a, t, sm.tabp);
    if (marks) phase_mark(a, 5);
    return delivered;
}

// Weights as the eager rule has them after the steps done (t_now = steps completed): the
// stored weight plus the row's pending potentiations (post spikes since its last
// processing), for the entries of rows [row_lo, row_hi) in storage order; static synapses
// read 0.  The stored state is left untouched (the lazy schedule stays the same).
__global__ void __launch_bounds__(256) k_settle_weights(SimArgs a, uint64_t t_now, uint32_t row_lo, uint32_t row_hi,
                                                        float *out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * 8;
    const uint32_t *pts = a.pre_ts + lslot(t_now) * (uint64_t)a.N;
    const float *pc = a.pre_c + lslot(t_now) * (uint64_t)a.N;
    const uint4 *post = reinterpret_cast<const uint4 *>(a.post) + (t_now & 1) * a.ring_stride;
    const uint64_t base0 = a.row_ptr[row_lo];
    for (uint64_t q = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); q < (uint64_t)(row_hi - row_lo) * a.NT; q += nwarps) {
        const uint32_t s = row_lo + (uint32_t)(q / a.NT), b = (uint32_t)(q % a.NT);
        const uint32_t *bp = a.bnd + (uint64_t)s * (a.NT + 1) + b;
        const uint64_t st = a.row_ptr[s] + bp[0];
        const uint32_t len = bp[1] - bp[0];
        const bool pls = plastic_src(a, s);
        const uint32_t ts_j = pls ? pts[s] : kNone;
        const float cx = pls ? pc[s] : 0.0f;
        const int64_t tproc = row_tproc(s, t_now, ts_j);
        for (uint32_t e = lane; e < len; e += 32) {
            float w = a.w[st + e];
            if (w >= 0.0f) {
                const uint32_t il = b * a.TW + a.ent[st + e];
                const uint4 ps = post[il];
                w = potentiate_lazy(a, a.tab_p, w, tproc, ts_j, cx, ps.x, ps.y, ps.z, a.post_mask + (uint64_t)il * kHistWords);
            } else {
                w = 0.0f;
            }
            out[st + e - base0] = w;
        }
    }
}
cudaError_t launch_settle_weights(const SimArgs &a, uint64_t t_now, uint32_t row_lo, uint32_t row_hi, float *out,
                                  cudaStream_t s) {
    const uint64_t work = (uint64_t)(row_hi - row_lo) * a.NT;
    const uint32_t grid = (uint32_t)std::min<uint64_t>((work + 7) / 8, 148ull * 16);
    if (grid) k_settle_weights<<<grid, 256, 0, s>>>(a, t_now, row_lo, row_hi, out);
    return cudaGetLastError();
}

// Padded-layout delivery of tile b (CTA c of C): byte-offset or counter-index entries.
__device__ __forceinline__ void deliver_padded(const SimArgs &a, uint64_t t, uint32_t b, uint32_t c,
                                               uint32_t *cnt, uint32_t *big, bool marks = false,
                                               uint32_t pre_total = 0xFFFFFFFFu) {
    if (a.dly) {
        if (a.eshift) deliver_tile_ring<false, true>(a, t, b, c, cnt, big, marks, pre_total);
        else deliver_tile_ring<true, true>(a, t, b, c, cnt, big, marks, pre_total);
    } else {
        if (a.eshift) deliver_tile_ring<false>(a, t, b, c, cnt, big, marks, pre_total);
        else deliver_tile_ring<true>(a, t, b, c, cnt, big, marks, pre_total);
    }
}

__device__ __forceinline__ void store_delivered(const SimArgs &a, uint32_t slot, uint32_t d, uint32_t *s_tmp) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xFFFFFFFFu, d, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_tmp[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < kBlock / 32; ++w) tot += s_tmp[w];
        if (tot) atomicAdd(&a.delivered_cta[slot], tot);
    }
}

// Delivery shared memory: cnt [TW + kDummy] | big [max(kStageWords, rings)] | pref | tmp
// | prod [a.prod_words] (synth fast path: spike IDs + descriptor staging of the producer warps)
__host__ __device__ constexpr uint32_t big_words() {
    return (uint32_t)kStageWords > (kBlock / 32) * kRing ? (uint32_t)kStageWords : (kBlock / 32) * kRing;
}
__device__ __forceinline__ DeliverSmem carve(const SimArgs &a, uint32_t *smem) {
    DeliverSmem sm;
    const uint32_t tw4 = (a.TW + 3u) & ~3u;
    sm.cnt = smem;
    smem += tw4 + kDummy;
    sm.stage = smem;
    smem += big_words();
    sm.pref = smem;
    sm.tmp = sm.pref + ((a.NR + 1 + 3) & ~3u);
    sm.prod = sm.tmp + 36;                              // 16-byte aligned (tmp is 32 + 4 words)
    return sm;
}

size_t tile_smem_bytes(uint32_t TW, uint32_t NR, uint32_t prod_words) {
    const uint32_t tw4 = (TW + 3u) & ~3u;
    return ((size_t)tw4 + kDummy + big_words() + ((NR + 1 + 3) & ~3u) + 32 + 4 + prod_words) * 4;
}

// Brunel+ tile kernels: counters, plastic fixed-point low / high words, post traces y
// ([TW] each), region prefix, scan tmp, staging.
size_t plastic_smem_bytes(uint32_t TW, uint32_t NR) {
    const uint32_t tw4 = (TW + 3u) & ~3u;
    return ((size_t)7 * tw4 + ((NR + 1 + 3) & ~3u) + 32 + kStageWords + kTraceLen + kPlChunks + 4) * 4 + 16;
}
__device__ __forceinline__ PlasticSmem carve_plastic(const SimArgs &a, uint32_t *smem) {
    PlasticSmem sm;
    const uint32_t tw4 = (a.TW + 3u) & ~3u;
    sm.cnt = smem;
    sm.plo = smem + tw4;
    sm.phi = smem + 2 * tw4;
    sm.ys = reinterpret_cast<float *>(smem + 3 * tw4);
    sm.p1 = smem + 4 * tw4;
    sm.p2 = smem + 5 * tw4;
    sm.p3 = smem + 6 * tw4;
    sm.pref = smem + 7 * tw4;
    sm.tmp = sm.pref + ((a.NR + 1 + 3) & ~3u);
    sm.stage = sm.tmp + 32;
    sm.tabp = reinterpret_cast<float *>(sm.stage + kStageWords);
    sm.cst = sm.stage + kStageWords + kTraceLen;
    return sm;
}
__device__ __forceinline__ void load_trace_table(const SimArgs &a, const PlasticSmem &sm) {
    const float4 *src = reinterpret_cast<const float4 *>(a.tab_p);
    float4 *dst = reinterpret_cast<float4 *>(sm.tabp);
    for (uint32_t x = threadIdx.x; x < kTraceLen / 4; x += kBlock) dst[x] = src[x];
}
// the tile's delivered step: counters -> ring slot t + delay, fixed-point sums -> plastic ring
__device__ __forceinline__ void plastic_flush(const SimArgs &a, uint64_t t, uint32_t b, const PlasticSmem &sm) {
    const uint64_t base = modD(a, t + a.delay) * a.ring_stride + (uint64_t)b * a.TW;
    // slot t + delay was consumed (zeroed) by the update of step t + delay - D < t; only
    // longer per-synapse delays of earlier steps add into it, else this is its sole writer
    const uint32_t sh = a.pl_split ? 16u : 32u;
    if (a.dly) {
        for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) {
            a.ring[base + x] += sm.cnt[x];
            a.pring[base + x] += (long long)(((uint64_t)sm.phi[x] << sh) + sm.plo[x]);
        }
    } else {
        for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) {
            a.ring[base + x] = sm.cnt[x];
            a.pring[base + x] = (long long)(((uint64_t)sm.phi[x] << sh) + sm.plo[x]);
        }
    }
}

// ------------------------------------------------------------------ kernels
template <int MODEL>
__global__ void __launch_bounds__(kBlock) k_update(SimArgs a, uint32_t k) {
    extern __shared__ __align__(16) uint32_t stage[];
    __shared__ uint32_t s_count;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    update_tile<MODEL>(a, *a.t0 + k, blockIdx.x, blockIdx.x * a.TWs, a.TWs, nullptr, a.G == 1, &s_count, stage);
}

// Delivery of step t alone (padded layout): the first/last step of a graph replay, the
// unfused sequence and G > 1 external exchange.
__global__ void __launch_bounds__(kBlock) k_deliver(SimArgs a, uint32_t k) {
    extern __shared__ __align__(16) uint32_t smem[];
    DeliverSmem sm = carve(a, smem);
    const uint64_t t = *a.t0 + k;
    const uint32_t b = blockIdx.x / a.C, c = blockIdx.x % a.C;
    for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) sm.cnt[x] = 0u;
    __syncthreads();
    deliver_padded(a, t, b, c, sm.cnt, sm.stage);
    const uint32_t d = 0;                                // (counted from out-degrees by the producers)
    uint32_t *dst = a.ring + modD(a, t + a.delay) * a.ring_stride + (uint64_t)b * a.TW;
    if (a.C == 1u) {
        for (uint32_t x = threadIdx.x * 4u; x < a.TW; x += kBlock * 4u) {
            uint4 o = *reinterpret_cast<uint4 *>(dst + x);
            o.x += sm.cnt[x]; o.y += sm.cnt[x + 1]; o.z += sm.cnt[x + 2]; o.w += sm.cnt[x + 3];
            *reinterpret_cast<uint4 *>(dst + x) = o;
        }
    } else {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t bytes_total = a.TW * 4u;
            for (uint32_t off = 0; off < bytes_total; off += 32768u) {
                const uint32_t nb = min(32768u, bytes_total - off);
                const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(sm.cnt) + off;
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;"
                             :: "l"(reinterpret_cast<char *>(dst) + off), "r"(saddr), "r"(nb) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    store_delivered(a, blockIdx.x, d, sm.tmp);
    if (a.C != 1u && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(kBlock) k_deliver_plastic(SimArgs a, uint32_t k) {
    extern __shared__ __align__(16) uint32_t smem[];
    PlasticSmem sm = carve_plastic(a, smem);
    const uint64_t t = *a.t0 + k;
    const uint32_t b = blockIdx.x;
    for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) { sm.cnt[x] = 0u; sm.plo[x] = 0u; sm.phi[x] = 0u; }
    load_trace_table(a, sm);
    __syncthreads();
    const uint32_t d = deliver_tile_plastic(a, t, b, sm);
    plastic_flush(a, t, b, sm);
    store_delivered(a, b, d, sm.tmp);
}

// Cluster tiles (C > 1): after every CTA of the cluster has accumulated its share of the
// tile's visits into its own full-tile counters, CTA c sums slice c of all C counter arrays
// (16-byte distributed-shared-memory loads, peers staggered) into its own slice.  The
// closing arrive is matched by cluster_wait() before exit: no CTA leaves (releasing its
// shared memory) while a peer may still read it.
__device__ __forceinline__ void cluster_reduce_slice(const SimArgs &a, uint32_t *cnt, uint32_t c) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t *mine = cnt + c * a.TWs;
    const uint32_t base = smem_u32(mine);
    for (uint32_t i = threadIdx.x * 4u; i < a.TWs; i += kBlock * 4u) {
        uint4 acc = *reinterpret_cast<const uint4 *>(mine + i);
#pragma unroll
        for (uint32_t k = 1; k < kMaxCluster; ++k) {
            if (k < a.C) {
                uint32_t peer = c + k;
                if (peer >= a.C) peer -= a.C;
                uint32_t ra;
                uint4 v;
                asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + 4u * i), "r"(peer));
                asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ra));
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
        }
        *reinterpret_cast<uint4 *>(mine + i) = acc;
    }
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Fused kernel: for MODEL != 3 the second parameter V selects the padded entry format
// (bit 0 = 1: counter indices, cluster tiles; 0: byte offsets) and bit 1 the mixed
// per-synapse delay variant; Brunel+ has one variant (V = 0).
template <int MODEL, int V>
__global__ void __launch_bounds__(kBlock) k_fused(SimArgs a, uint32_t k) {
    if constexpr (MODEL == 3) {                             // Brunel+ (delay >= 1 via the rings)
        extern __shared__ __align__(16) uint32_t smem[];
        PlasticSmem sm = carve_plastic(a, smem);
        __shared__ uint32_t s_count3;
        const uint64_t t = *a.t0 + k;
        const uint32_t b = blockIdx.x;
        phase_mark(a, 0);
        if (threadIdx.x == 0) s_count3 = 0;
        for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) { sm.cnt[x] = 0u; sm.plo[x] = 0u; sm.phi[x] = 0u; }
        load_trace_table(a, sm);                            // (constant: before the dependent-launch wait)
        __shared__ bool s_upd;
        if (threadIdx.x == 0) s_upd = false;
        asm volatile("griddepcontrol.wait;" ::: "memory");          // (programmatic dependent launch)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        __syncthreads();
        const uint32_t d = deliver_tile_plastic(a, t, b, sm, true, &s_count3, &s_upd);
        plastic_flush(a, t, b, sm);
        store_delivered(a, b, d, sm.tmp);
        __syncthreads();
        phase_mark(a, 6);
        if (!s_upd)
            update_tile<MODEL>(a, t + 1, b, b * a.TW, a.TW, nullptr, true, &s_count3, sm.stage, nullptr, true);
        phase_mark(a, 12);
    } else {                                                 // padded layout (G = 1)
        extern __shared__ __align__(16) uint32_t smem[];
        DeliverSmem sm = carve(a, smem);
        __shared__ uint32_t s_count;
        const uint64_t t = *a.t0 + k;
        const uint32_t b = blockIdx.x;
        if (threadIdx.x == 0) s_count = 0;
        // tile bt = blockIdx.x / C; with C > 1 this CTA is rank c of the tile's cluster
        const uint32_t bt = b / a.C, c = b % a.C;
        phase_mark(a, 0);
        // Programmatic dependent launch: the next step's kernel may be scheduled once every
        // CTA of this one has passed its own grid dependency (launch_dependents after
        // griddepcontrol.wait below, so at most two step kernels ever overlap); it zeroes its
        // counters and computes what needs no input while this one finishes, then waits
        // (griddepcontrol.wait) for this grid's completion
        // (G > 1: the update of t+1 only writes the send bitmap; the lists and descriptors of
        //  the gathered spikes come from bitmap->list)
        if (threadIdx.x == 0) {   // this slice's neuron state (+ input slot t+1) -> L2 while delivering
            const uint32_t lo0 = b * a.TWs, nb = a.TWs * 4u;
            const void *arr[5] = {MODEL == 4 ? (const void *)(a.acc + lo0) : (const void *)(a.v + lo0),
                                  MODEL == 4 ? nullptr : (const void *)(a.ref + lo0),
                                  MODEL == 1 ? (const void *)(a.ge + lo0) : nullptr,
                                  MODEL == 1 ? (const void *)(a.gi + lo0) : nullptr,
                                  a.delay > 1 ? (const void *)(a.ring + modD(a, t + 1) * a.ring_stride + lo0) : nullptr};
#pragma unroll
            for (int q = 0; q < 5; ++q)
                if (arr[q]) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(arr[q]), "r"(nb) : "memory");
        }
        for (uint32_t x = threadIdx.x * 4u; x < a.TW; x += kBlock * 4u)      // TW is a multiple of 32
            *reinterpret_cast<uint4 *>(sm.cnt + x) = make_uint4(0u, 0u, 0u, 0u);
        const uint32_t lo = b * a.TWs;
        // synth, G = 1: the spikes of step t + 1, computed during the delivery of t (synth_fire)
        constexpr uint32_t kFireWords = 1536;
        __shared__ uint32_t s_fire[MODEL == 4 ? kFireWords : 1];
        const bool syn = MODEL == 4 && a.G == 1 && a.TWs <= 32u * kFireWords && a.prod_words > kSynthSid;
        uint32_t *sid_s = syn ? sm.prod : sm.stage + kStageWords;
        __shared__ uint32_t s_off;
        // delay >= 2, one CTA per tile: the update of t + 1 runs on the last kUpdWarps warps
        // while the others deliver t (its input slot t + 1 is complete; P:290 timestep grouping)
        const bool ovl = !syn && a.delay >= 2 && a.C == 1;
        // Brunel: the drive's inversion table is constant -- into shared memory before the
        // grid dependency instead of at the start of the update (one round trip off its path)
        const bool pstaged = MODEL == 2 && stage_ptab(a);
        phase_mark(a, 10);                                   // (diagnostics: counters zeroed)
        asm volatile("griddepcontrol.wait;" ::: "memory");          // the previous step is complete
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        // thread 0: the step's descriptor count
        const uint32_t pre_total = threadIdx.x == 0 ? a.dcount[t & 3u] : 0xFFFFFFFFu;
        __syncthreads();
        phase_mark(a, 1);
        if (syn) {
            // synth: the spikes of step t + 1 (input-independent Philox draws, ~2.7 us of ALU
            // work per CTA) on the last kFireWarps warps while the others deliver t -- off the
            // step's critical path (in the prologue, the CTA that starts last paid them)
            constexpr uint32_t NWD = kBlock / 32 - kFireWarps;
            const uint32_t n_sp = delivery_count(a, t, bt, c, pre_total);
            const uint32_t warp = threadIdx.x >> 5;
            if (warp < NWD) {
                deliver_ring_core<(V & 1) != 0, (V & 2) != 0>(a, t, bt, c, sm.cnt, sm.stage, n_sp, warp, NWD);
            } else {
                const uint32_t ptid = threadIdx.x - NWD * 32, pth = kFireWarps * 32;
                synth_fire(a, t + 1, b, lo, a.TWs, s_fire, sid_s, &s_count, kSynthSid, ptid, pth);
                asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");
                phase_mark(a, 11, NWD * 32);                 // (diagnostics: spikes of t + 1)
                synth_rows_prefetch(a, t + 1, s_count, sid_s, sm.prod + kSynthSid, a.prod_words - kSynthSid,
                                    ptid, pth, &s_off);
                asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");   // (s_off)
                synth_publish(a, t, b, lo, s_fire, sid_s, s_count, sm.prod + kSynthSid, a.prod_words - kSynthSid,
                              s_off, ptid, pth);
                phase_mark(a, 9, NWD * 32);                  // (diagnostics: step t + 1 published)
            }
            phase_mark(a, 4);
            __syncthreads();
            phase_mark(a, 5);
        } else if (ovl) {
            constexpr uint32_t NWD = kBlock / 32 - kOvlUpdWarps;
            const uint32_t n_sp = delivery_count(a, t, bt, c, pre_total);
            const uint32_t warp = threadIdx.x >> 5;
            if (warp < NWD) {
                deliver_ring_core<(V & 1) != 0, (V & 2) != 0>(a, t, bt, c, sm.cnt, sm.stage, n_sp, warp, NWD);
            } else {
                update_tile<MODEL, true, true>(a, t + 1, b, b * a.TWs, a.TWs, nullptr, a.G == 1, &s_count,
                                               sm.stage + NWD * kRing, nullptr, false, kMaxCluster, nullptr, nullptr,
                                               threadIdx.x - NWD * 32, kOvlUpdWarps * 32, kOvlUpdWarps * kRing, pstaged);
            }
            __syncthreads();
        } else {
            deliver_tile_ring<(V & 1) != 0, (V & 2) != 0>(a, t, bt, c, sm.cnt, sm.stage, true, pre_total);
        }
        uint32_t *cnt = sm.cnt + c * a.TWs;                  // this CTA's slice
        constexpr bool DESC = true;
        if (a.delay == 1) {
            // C > 1: the update sums the C partial slices itself (peers read after one cluster
            // barrier; a second one at exit keeps every CTA's counters alive until then)
            if (a.C > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            phase_mark(a, 6);
            if (syn) {
                synth_accumulate(a, t + 1, lo, a.TWs, cnt, a.C > 1 ? c : kMaxCluster);
                phase_mark(a, 7);
                __syncthreads();
            }
            else
                update_tile<MODEL, DESC>(a, t + 1, b, lo, a.TWs, cnt, a.G == 1, &s_count, sm.stage, nullptr, true,
                                         a.C > 1 ? c : kMaxCluster, sm.stage + kStageWords, nullptr, threadIdx.x, kBlock,
                                         kStageWords, pstaged);
            // (an arrive right after the update loop, waited at exit, measured 0.5 us slower)
            if (a.C > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            if (a.C > 1) cluster_reduce_slice(a, sm.cnt, c);   // slice summed in place
            phase_mark(a, 6);
            uint32_t *dst = a.ring + modD(a, t + a.delay) * a.ring_stride + lo;
            for (uint32_t x = threadIdx.x * 4u; x < a.TWs; x += kBlock * 4u) {
                uint4 o = *reinterpret_cast<const uint4 *>(cnt + x);
                if (V & 2) {                                  // the slot may hold longer-delay arrivals
                    const uint4 r = *reinterpret_cast<const uint4 *>(dst + x);
                    o.x += r.x; o.y += r.y; o.z += r.z; o.w += r.w;
                }
                *reinterpret_cast<uint4 *>(dst + x) = o;
            }
            if (syn) {
                __syncthreads();                             // (the slot's ring writes above)
                synth_accumulate(a, t + 1, lo, a.TWs, nullptr, kMaxCluster);
                __syncthreads();
            } else if (ovl) {
                // (the update of t + 1 ran during the delivery)
            } else {
                update_tile<MODEL, DESC>(a, t + 1, b, lo, a.TWs, nullptr, a.G == 1, &s_count, sm.stage, nullptr, true,
                                         kMaxCluster, sm.stage + kStageWords, nullptr, threadIdx.x, kBlock, kStageWords,
                                         pstaged);
            }
            if (a.C > 1) cluster_wait();                     // partners done reading this CTA's counters
        }
        phase_mark(a, 12);
    }
}

// ------------------------------------------------- synth, persistent (G = 1, delay 1)
// In-kernel grid barrier (all CTAs co-resident: cooperative launch).  Barrier i of a launch
// counts arrivals in slot i mod 4 (one thread of every CTA: a gpu-scope release add, then
// an acquire spin until all gridDim.x arrived); CTA 0 clears slot (i + 2) mod 4 once past
// barrier i (its last users passed barrier i - 2 before anyone could arrive at i - 1),
// k_advance clears all four after the launch.  A barrier not complete within ~10 s (a CTA
// that never got scheduled) sets gbar[8] and every CTA falls through the remaining
// barriers: the host reports an error instead of hanging the GPU.
// (slot i: a 64-bit word at gbar + 2 (i mod 4) -- arrivals in the low half, a payload the
//  arrivals add in the high half: the synth kernel's descriptor count of the next step)
__device__ __forceinline__ unsigned long long *gbar_slot(const SimArgs &a, uint32_t i) {
    return reinterpret_cast<unsigned long long *>(a.gbar) + (i & 3u);
}
__device__ __forceinline__ void grid_arrive_add(const SimArgs &a, uint32_t i, uint32_t payload) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;"
                 :: "l"(gbar_slot(a, i)), "l"(((unsigned long long)payload << 32) | 1ull) : "memory");
}
// Thread 0 waits; returns the payload sum (valid in thread 0).
__device__ __forceinline__ uint32_t grid_wait(const SimArgs &a, uint32_t i) {
    uint32_t payload = 0;
    if (threadIdx.x == 0) {
        const unsigned long long *slot = gbar_slot(a, i);
        unsigned long long t_start;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        for (uint32_t spin = 0;; ++spin) {
            unsigned long long v;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
            if ((uint32_t)v >= gridDim.x) { payload = (uint32_t)(v >> 32); break; }
            if ((spin & 255u) == 255u) {
                if (*(volatile uint32_t *)(a.gbar + 8)) break;
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (now - t_start > 10000000000ull) { atomicExch(a.gbar + 8, 1u); break; }
            }
        }
        __threadfence();                              // (also drops stale L1 lines of this SM)
        if (blockIdx.x == 0) *gbar_slot(a, i + 2u) = 0ull;
    }
    __syncthreads();
    return payload;
}

// nsteps consecutive synth steps k .. k + nsteps - 1 in ONE launch (each: deliver t + the
// update of t + 1).  The synth update of t + 1 is acc += input(t + 1) and the drive does not
// depend on the input (reading R12), so the tile counters are not cleared between
// steps: they keep the running sum of the launch's inputs in shared memory (u32, wrapping
// exactly like acc) and are folded into acc once, at the end of the launch -- the per-step
// counter clearing, cluster reduction and accumulator pass (~4.5 us of a 21.5 us step in
// the one-kernel-per-step form) disappear, as does the kernel boundary.  Per step: the
// delivery warps deliver t while the fire warps draw, list and publish the spikes of t + 1
// (descriptor buffer (t + 1) mod 3) and then arrive at the step's grid barrier ("all CTAs
// published t + 1"), which every CTA waits for before step t + 1: a CTA's delivery of t
// overlaps the other CTAs' barrier traffic.  Why that is enough: the delivery of t + 1 reads
// only the descriptors of t + 1 and the CTA's own counters; descriptor buffer (t + 2) mod 3,
// written in step t + 1, was last read by the deliveries of t - 1, which every CTA finished
// before it could publish t + 1.  Outputs per step (record bitmap,
// spike lists, descriptors, fired / delivered counts) are those of k_fused; acc equals
// k_fused's after the launch.
template <int V>
__global__ void __launch_bounds__(kBlock) k_synth_run(SimArgs a, uint32_t k, uint32_t nsteps) {
    extern __shared__ __align__(16) uint32_t smem[];
    DeliverSmem sm = carve(a, smem);
    __shared__ uint32_t s_count, s_off;
    constexpr uint32_t kFireWords = 1536;
    __shared__ uint32_t s_fire[kFireWords];
    const uint32_t b = blockIdx.x, bt = b / a.C, c = b % a.C, lo = b * a.TWs;
    uint32_t *sid_s = sm.prod;
    constexpr uint32_t NWD = kBlock / 32 - kFireWarps;
    const uint32_t warp = threadIdx.x >> 5;
    for (uint32_t x = threadIdx.x * 4u; x < a.TW; x += kBlock * 4u)      // TW is a multiple of 32
        *reinterpret_cast<uint4 *>(sm.cnt + x) = make_uint4(0u, 0u, 0u, 0u);
    asm volatile("griddepcontrol.wait;" ::: "memory");          // the replay's first update is complete
    for (uint32_t i = 0; i < nsteps; ++i) {
        const uint64_t t = *a.t0 + k + i;
        // the step's descriptor count: the barrier word's payload (no extra round trip), or,
        // for the launch's first step (published by k_update), the step counter
        const uint32_t wsum = i ? grid_wait(a, i - 1) : 0u;
        phase_mark(a, 0);
        const uint32_t pre_total = threadIdx.x == 0 ? (i ? wsum : a.dcount[t & 3u]) : 0xFFFFFFFFu;
        if (threadIdx.x == 0) s_count = 0;
        const uint32_t n_sp = delivery_count(a, t, bt, c, pre_total);   // (block-wide)
        phase_mark(a, 1);
        if (warp < NWD) {
            deliver_ring_core<(V & 1) != 0, false>(a, t, bt, c, sm.cnt, sm.stage, n_sp, warp, NWD);
        } else {
            const uint32_t ptid = threadIdx.x - NWD * 32, pth = kFireWarps * 32;
            synth_fire(a, t + 1, b, lo, a.TWs, s_fire, sid_s, &s_count, kSynthSid, ptid, pth);
            asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");
            phase_mark(a, 11, NWD * 32);
            synth_rows_prefetch(a, t + 1, s_count, sid_s, sm.prod + kSynthSid, a.prod_words - kSynthSid,
                                ptid, pth, &s_off);
            phase_mark(a, 2, NWD * 32);
            asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");   // (s_off)
            phase_mark(a, 3, NWD * 32);
            synth_publish(a, t, b, lo, s_fire, sid_s, s_count, sm.prod + kSynthSid, a.prod_words - kSynthSid,
                          s_off, ptid, pth);
            // barrier i = "every CTA has published step t + 1": the fire warps arrive right
            // away; this CTA's delivery warps finish step t meanwhile (the next delivery needs
            // only the descriptors of t + 1 and this CTA's own counters, never cleared here)
            asm volatile("bar.sync 1, %0;" :: "r"(pth) : "memory");
            phase_mark(a, 8, NWD * 32);
            if (ptid == 0 && i + 1 < nsteps)            // (+ this CTA's descriptors of t + 1)
                grid_arrive_add(a, i, s_count);
            phase_mark(a, 9, NWD * 32);
        }
        phase_mark(a, 4);
        __syncthreads();
        phase_mark(a, 12);
    }
    // fold the launch's input sums into acc (C > 1: this CTA's slice of all C partial tiles)
    if (a.C > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    synth_accumulate(a, *a.t0 + k + nsteps, lo, a.TWs, sm.cnt + c * a.TWs, a.C > 1 ? c : kMaxCluster);
    if (a.C > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ------------------------------------------------ Brunel+, persistent (G = 1)
// The steps of a replay in one launch: per step the delivery of t (lazy STDP on the synapse
// stream) with the update of t + 1 and the pre-state pass on 8 warps beside it (k_fused<3>);
// the barrier is "every CTA has published t + 1" (its spikes, lists and pre state): the
// update warps arrive as soon as they are done, the delivery of t finishes meanwhile.  The
// next delivery reads the spike lists and pre state of t + 1 (copies (t + 1) mod 3) and this
// CTA's own tile state; the copies a CTA one step ahead writes, (t + 2) mod 3, are not the
// ones a slower CTA still reads (t mod 3).  A step whose segments need more than one staging
// pass runs the update after the delivery (k_fused's order) and arrives at its end.
__global__ void __launch_bounds__(kBlock) k_plastic_run(SimArgs a, uint32_t k, uint32_t nsteps) {
    extern __shared__ __align__(16) uint32_t smem[];
    PlasticSmem sm = carve_plastic(a, smem);
    __shared__ uint32_t s_count3;
    __shared__ bool s_upd;
    const uint32_t b = blockIdx.x;
    load_trace_table(a, sm);                                // (constant: before the dependent-launch wait)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (uint32_t i = 0; i < nsteps; ++i) {
        const uint64_t t = *a.t0 + k + i;
        if (i) grid_wait(a, i - 1);
        phase_mark(a, 0);
        if (threadIdx.x == 0) { s_count3 = 0; s_upd = false; }
        for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) { sm.cnt[x] = 0u; sm.plo[x] = 0u; sm.phi[x] = 0u; }
        __syncthreads();
        phase_mark(a, 1);
        const uint32_t arrive = i + 1 < nsteps ? i : kNone;
        const uint32_t d = deliver_tile_plastic(a, t, b, sm, true, &s_count3, &s_upd, arrive);
        plastic_flush(a, t, b, sm);
        store_delivered(a, b, d, sm.tmp);
        __syncthreads();
        phase_mark(a, 6);
        if (!s_upd) {
            update_tile<3>(a, t + 1, b, b * a.TW, a.TW, nullptr, true, &s_count3, sm.stage, nullptr, true);
            if (arrive != kNone && threadIdx.x == 0)
                grid_arrive_add(a, arrive, 0u);
        }
        phase_mark(a, 12);
    }
}

// Small networks (G = 1, delay 1, one tile of all owned neurons, fits shared memory): one
// CTA runs nsteps whole steps per launch.  Neuron state and the input counters live in
// shared memory for the launch; a step is update(t) (the shared update code: bitmap into
// the record ring, states written through to global) -> delivery of the step's spikes,
// found in the bitmap, warp per spike, lanes over the row's 16-byte windows, into the
// zeroed counters.  At the launch boundaries the inputs move through ring slots t0 % D /
// (t0 + nsteps) % D, so every other kernel sequence (unfused, profile, external) stays
// interchangeable.  Replaces 32 grid-wide kernel boundaries per graph by one.
__host__ __device__ inline size_t small_smem_words(uint32_t TW, uint32_t model, bool rows) {
    const uint32_t sw = model == 4 ? 1u : (model == 1 ? 4u : 2u);    // state words per neuron
    // counters, state, the step's bitmap, [per-source first window, end window, out-degree]
    return (size_t)TW + kDummy + (size_t)sw * TW + TW / 32 + (rows ? 3ull * TW : 0ull);
}
constexpr size_t kSmallSmemMax = 227 * 1024 - 2048;
__host__ __device__ inline bool small_rows(uint32_t TW, uint32_t model) {
    return small_smem_words(TW, model, true) * 4 + 16 <= kSmallSmemMax;
}
size_t small_smem_bytes(uint32_t TW, uint32_t model) {
    return small_smem_words(TW, model, small_rows(TW, model)) * 4 + 16;
}

template <int MODEL>
__global__ void __launch_bounds__(kBlock) k_small(SimArgs a, uint32_t k0, uint32_t nsteps) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ uint32_t s_count;
    __shared__ unsigned long long s_deliv;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t TW = a.TW;                               // multiple of 32, covers n_own
    uint32_t *cnt = smem;
    uint32_t *st = smem + TW + kDummy;                      // 16-byte aligned (TW, kDummy % 4 == 0)
    StatePtrs sp{nullptr, nullptr, nullptr, nullptr, nullptr, 0u};
    if (MODEL == 4) { sp.acc = st; }
    else if (MODEL == 1) { sp.v = reinterpret_cast<float *>(st); sp.ge = reinterpret_cast<float *>(st + TW);
                           sp.gi = reinterpret_cast<float *>(st + 2 * TW); sp.ref = st + 3 * TW; }
    else { sp.v = reinterpret_cast<float *>(st); sp.ref = st + TW; }
    uint32_t *bm_s = st + (MODEL == 4 ? 1u : (MODEL == 1 ? 4u : 2u)) * TW;
    const bool rows = small_rows(TW, MODEL);               // (uniform)
    uint32_t *rw0 = bm_s + TW / 32, *rw1 = rw0 + TW, *rdg = rw1 + TW;
    if (rows)                                               // sources' windows, staged once
        for (uint32_t x = tid; x < a.n_own; x += kBlock) {
            const uint64_t rs = a.row_ptr[x];
            rw0[x] = (uint32_t)((rs + a.bnd[2u * x]) >> kWinShift);
            rw1[x] = (uint32_t)((rs + a.bnd[2u * x + 1u]) >> kWinShift);
            rdg[x] = a.deg[x];
        }
    const uint64_t t0 = *a.t0 + k0;
    uint32_t *slot0 = a.ring + modD(a, t0) * a.ring_stride;
    for (uint32_t x = tid * 4u; x < TW; x += kBlock * 4u) {    // stage state + step t0's inputs
        if (MODEL == 4) *reinterpret_cast<uint4 *>(sp.acc + x) = *reinterpret_cast<const uint4 *>(a.acc + x);
        if (MODEL != 4) *reinterpret_cast<float4 *>(sp.v + x) = *reinterpret_cast<const float4 *>(a.v + x);
        if (MODEL != 4) *reinterpret_cast<uint4 *>(sp.ref + x) = *reinterpret_cast<const uint4 *>(a.ref + x);
        if (MODEL == 1) *reinterpret_cast<float4 *>(sp.ge + x) = *reinterpret_cast<const float4 *>(a.ge + x);
        if (MODEL == 1) *reinterpret_cast<float4 *>(sp.gi + x) = *reinterpret_cast<const float4 *>(a.gi + x);
        *reinterpret_cast<uint4 *>(cnt + x) = *reinterpret_cast<const uint4 *>(slot0 + x);
        *reinterpret_cast<uint4 *>(slot0 + x) = make_uint4(0u, 0u, 0u, 0u);
    }
    if (tid == 0) { s_count = 0; s_deliv = 0; }
    __syncthreads();
    const uint32_t cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
    const uint4 *ent4 = reinterpret_cast<const uint4 *>(a.ent);
    uint64_t deliv = 0;
    for (uint32_t q = 0; q < nsteps; ++q) {
        const uint64_t t = t0 + q;
        update_tile<MODEL>(a, t, 0, 0, TW, cnt, false, &s_count, nullptr, &sp, false, kMaxCluster,
                           nullptr, bm_s);                   // ends with a barrier
        for (uint32_t x = tid * 4u; x < TW; x += kBlock * 4u)
            *reinterpret_cast<uint4 *>(cnt + x) = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
        for (uint32_t wi = warp; wi < a.W; wi += kBlock / 32) {
            uint32_t word = bm_s[wi];
            while (word) {                                   // warp-uniform
                const uint32_t sidx = wi * 32u + (uint32_t)__ffs(word) - 1u;
                word &= word - 1u;
                uint32_t w0, w1;
                if (rows) { w0 = rw0[sidx]; w1 = rw1[sidx]; }
                else {
                    const uint64_t rs = a.row_ptr[sidx];
                    w0 = (uint32_t)((rs + a.bnd[2u * sidx]) >> kWinShift); w1 = (uint32_t)((rs + a.bnd[2u * sidx + 1u]) >> kWinShift);
                }
                const uint32_t qv = sidx >= a.n_exc ? 65536u : 1u;
                for (uint32_t w = w0 + lane; w < w1; w += 32) {
                    for (uint32_t h = 0; h < kWin / 8; ++h) {
                        const uint4 v0 = ent4[(kWin / 8) * w + h];
                        if (a.eshift) accumulate_window<false>(cnt_s, v0, qv);
                        else accumulate_window<true>(cnt_s, v0, qv);
                    }
                }
                if (lane == 0) deliv += rows ? rdg[sidx] : a.deg[sidx];
            }
        }
        __syncthreads();
    }
    // step t0 + nsteps's inputs -> its ring slot (added: the slot is otherwise empty)
    uint32_t *slot1 = a.ring + modD(a, t0 + nsteps) * a.ring_stride;
    for (uint32_t x = tid * 4u; x < TW; x += kBlock * 4u) {
        uint4 o = *reinterpret_cast<uint4 *>(slot1 + x);
        o.x += cnt[x]; o.y += cnt[x + 1]; o.z += cnt[x + 2]; o.w += cnt[x + 3];
        *reinterpret_cast<uint4 *>(slot1 + x) = o;
    }
    if (lane == 0 && deliv) atomicAdd(&s_deliv, (unsigned long long)deliv);
    __syncthreads();
    if (tid == 0 && s_deliv) atomicAdd(&a.delivered_cta[0], s_deliv);
}

cudaError_t launch_small(const SimArgs &a, uint32_t k0, uint32_t nsteps, cudaStream_t s) {
    const size_t bytes = small_smem_bytes(a.TW, a.model);
    switch (a.model) {
    case 1: k_small<1><<<1, kBlock, bytes, s>>>(a, k0, nsteps); break;
    case 2: k_small<2><<<1, kBlock, bytes, s>>>(a, k0, nsteps); break;
    case 4: k_small<4><<<1, kBlock, bytes, s>>>(a, k0, nsteps); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// Procedural connectivity ("only store the parameters used to
// create the network and then generate adjacency data on the fly" [Knight2021]): no rows are
// stored; the CTA of tile b regenerates, for every spike s of step t, its row segment into
// the tile from the same Philox predicate the generator uses (FIXED_PROB rules: edge s -> j
// iff Philox(s, j>>2, rule, 1)[j&3] < floor(p 2^32), reading R9), one Philox call per spike and
// 4-target block, flattened over all threads, and accumulates the hits' packed receptor
// counts in shared memory (per-synapse delays: minimum delay there, longer delays into ring
// slot t + d).  Memory: O(neurons) instead of O(synapses); the work is one Philox call per
// 4 candidate pairs instead of 2 bytes per synapse.
__global__ void __launch_bounds__(kBlock) k_deliver_proc(SimArgs a, uint32_t k) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *cnt = smem;                                   // [TW]
    uint32_t *pref = smem + ((a.TW + 3u) & ~3u), *tmp = pref + ((a.NR + 1 + 3) & ~3u);
    const uint64_t t = *a.t0 + k;
    const uint32_t par = lslot(t), b = blockIdx.x;
    for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) cnt[x] = 0u;
    for (uint32_t r = threadIdx.x; r < a.NR; r += kBlock) pref[r] = a.sl_counts[par * a.NR + r];
    __syncthreads();
    block_exclusive_scan(pref, a.NR, tmp);
    const uint32_t n_sp = pref[a.NR];
    const uint32_t lo = b * a.TW, width = min(a.TW, a.n_own - lo), nblk = (width + 3u) / 4u;
    const uint64_t lbase = (uint64_t)par * a.NR * a.RS;
    const uint32_t tD = (uint32_t)modD(a, t);
    uint32_t hits = 0;
    const uint64_t total = (uint64_t)n_sp * nblk;
    for (uint64_t f = threadIdx.x; f < total; f += kBlock) {
        const uint32_t p = (uint32_t)(f / nblk), q4 = (uint32_t)(f % nblk);
        const uint32_t r = region_of(pref, a.NR, p);
        const uint32_t s = a.sl_ids[lbase + (uint64_t)r * a.RS + (p - pref[r])];
        const uint32_t i0 = lo + 4u * q4;                   // 4 consecutive owned targets
        const uint32_t j0 = a.G == 1 ? i0 : (uint32_t)local_to_global(i0, a.rank, a.G, a.S);
        const uint32_t qv = s >= a.n_exc ? 65536u : 1u;
        for (uint32_t rr = 0; rr < a.nproc; ++rr) {
            const uint32_t *R = a.proc[rr];                 // src_b, src_e, dst_b, dst_e, thr lo, thr hi, index, dmin | dmax << 16
            if (s < R[0] || s >= R[1] || j0 + 3u < R[2] || j0 >= R[3]) continue;
            const uint64_t thr = ((uint64_t)R[5] << 32) | R[4];
            const uint4 x = philox4x32_10(make_uint4(s, j0 >> 2, R[6], kTagConn), a.key0, a.key1);
#pragma unroll
            for (uint32_t e = 0; e < 4; ++e) {
                const uint32_t j = j0 + e;
                if (i0 + e >= lo + width || j < R[2] || j >= R[3] || (uint64_t)word_of(x, e) >= thr) continue;
                ++hits;
                const uint32_t off = i0 + e - lo;
                const uint32_t dlo = R[7] & 0xFFFFu, dhi = R[7] >> 16;
                uint32_t d = dlo;
                if (dhi > dlo) {                            // per-synapse delay (reading R19)
                    const uint4 y = philox4x32_10(make_uint4(s, j >> 2, R[6], kTagDelay), a.key0, a.key1);
                    d += (uint32_t)(((uint64_t)word_of(y, j & 3) * (dhi - dlo + 1)) >> 32);
                }
                if (d == a.delay) atomicAdd(&cnt[off], qv);
                else {
                    uint32_t sl = tD + d;
                    if (sl >= a.D) sl -= a.D;
                    atomicAdd(a.ring + (uint64_t)sl * a.ring_stride + lo + off, qv);
                }
            }
        }
    }
    __syncthreads();
    uint32_t *dst = a.ring + modD(a, t + a.delay) * a.ring_stride + lo;
    for (uint32_t x = threadIdx.x; x < a.TW; x += kBlock) dst[x] += cnt[x];
    store_delivered(a, b, hits, tmp);
}

// Synapses of this rank under the procedural rules (count only; nothing is stored), and the
// per-target excitatory / inhibitory in-degrees tc[2 i], tc[2 i + 1] (packing check).
__global__ void k_count_proc(SimArgs a, unsigned long long *out, uint32_t *tc) {
    unsigned long long c = 0;
    const uint64_t nblk = (a.n_own + 3u) / 4u;
    const uint64_t total = (uint64_t)a.N * nblk;
    for (uint64_t f = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total; f += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)(f / nblk), i0 = 4u * (uint32_t)(f % nblk);
        const uint32_t j0 = a.G == 1 ? i0 : (uint32_t)local_to_global(i0, a.rank, a.G, a.S);
        for (uint32_t rr = 0; rr < a.nproc; ++rr) {
            const uint32_t *R = a.proc[rr];
            if (s < R[0] || s >= R[1] || j0 + 3u < R[2] || j0 >= R[3]) continue;
            const uint64_t thr = ((uint64_t)R[5] << 32) | R[4];
            const uint4 x = philox4x32_10(make_uint4(s, j0 >> 2, R[6], kTagConn), a.key0, a.key1);
            for (uint32_t e = 0; e < 4; ++e) {
                const uint32_t j = j0 + e;
                if (i0 + e < a.n_own && j >= R[2] && j < R[3] && (uint64_t)word_of(x, e) < thr) {
                    ++c;
                    atomicAdd(&tc[2u * (i0 + e) + (s >= a.n_exc ? 1u : 0u)], 1u);
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
cudaError_t launch_count_proc(const SimArgs &a, unsigned long long *out, uint32_t *tc, cudaStream_t s) {
    k_count_proc<<<148 * 8, 256, 0, s>>>(a, out, tc);
    return cudaGetLastError();
}

// Paper-style baseline: warp w delivers spike (w mod |S|) to tile (w / |S|), column-wise
// (P:200), with one global atomic per event.
__global__ void __launch_bounds__(kBlock) k_global_atomics(SimArgs a, uint32_t k) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *pref = smem, *tmp = smem + ((a.NR + 1 + 3) & ~3u);
    const uint64_t t = *a.t0 + k;
    const uint32_t par = lslot(t);
    for (uint32_t r = threadIdx.x; r < a.NR; r += kBlock) pref[r] = a.sl_counts[par * a.NR + r];
    __syncthreads();
    block_exclusive_scan(pref, a.NR, tmp);
    const uint32_t n_sp = pref[a.NR];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (kBlock / 32);
    uint32_t *slot = a.ring + modD(a, t + a.delay) * a.ring_stride;
    const uint64_t lbase = (uint64_t)par * a.NR * a.RS;
    uint32_t delivered = 0;
    for (uint64_t w = (uint64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); w < (uint64_t)a.NT * n_sp; w += nwarps) {
        const uint32_t b = (uint32_t)(w / n_sp), p = (uint32_t)(w % n_sp);
        const uint32_t r = region_of(pref, a.NR, p);
        const uint64_t sl = lbase + (uint64_t)r * a.RS + (p - pref[r]);
        const uint32_t s = a.sl_ids[sl];
        const uint32_t *bp = a.bnd + (uint64_t)s * (a.NT + 1u) + b;
        const uint64_t st = a.sl_rows[sl] + bp[0];
        const uint32_t len = bp[1] - bp[0];
        const uint32_t qv = s >= a.n_exc ? 65536u : 1u;
        uint32_t *tile = slot + (uint64_t)b * a.TW;
        for (uint32_t e = lane; e < len; e += 32) {
            const uint32_t x = (uint32_t)a.ent[st + e] >> a.eshift;
            if (x >= a.TW) continue;                     // skip padding sentinels
            if (a.dly && a.dly[st + e] != a.delay)       // longer per-synapse delay (reading R19)
                atomicAdd(a.ring + modD(a, t + a.dly[st + e]) * a.ring_stride + (uint64_t)b * a.TW + x, qv);
            else
                atomicAdd(tile + x, qv);
        }
        if (lane == 0 && !a.deg) delivered += len;
    }
    store_delivered(a, blockIdx.x % (a.NT * a.C), delivered, tmp);
}

// Gathered bitmaps of all ranks -> global spike list regions + record ring copy.
__global__ void __launch_bounds__(kBlock) k_b2l(SimArgs a, uint32_t k) {
    __shared__ uint32_t s_count;
    const uint64_t t = *a.t0 + k;
    const uint32_t par = (uint32_t)(t & 1);
    const uint32_t nw = a.G * a.W, r = blockIdx.x;
    if (threadIdx.x == 0) s_count = 0;
    __syncthreads();
    const uint32_t ls = lslot(t);                         // (list copy; par: the PEER window parity)
    uint32_t *region = a.sl_ids + ((uint64_t)ls * a.NR + r) * a.RS;
    uint64_t *region_rows = a.sl_rows + ((uint64_t)ls * a.NR + r) * a.RS;
    const uint32_t bw = a.RS / 32;                      // bitmap words of this region
    for (uint32_t q0 = 0; q0 < bw; q0 += kBlock) {
        const uint32_t idx = r * bw + q0 + threadIdx.x;
        const bool in = q0 + threadIdx.x < bw && idx < nw;
        uint32_t word = in ? a.gather[(a.peers ? (uint64_t)par * nw : 0ull) + idx] : 0u;
        if (word) {               // bits past the rank's owned neurons (global ID >= N) are ignored
            const uint64_t j0 = local_to_global((uint64_t)(idx % a.W) * 32, idx / a.W, a.G, a.S);
            word = j0 >= a.N ? 0u : (a.N - j0 >= 32 ? word : word & ((1u << (a.N - j0)) - 1u));
        }
        if (in) a.record[modR(a, t) * (uint64_t)nw + idx] = word;
        const uint32_t cnt = __popc(word), incl = warp_incl_scan(cnt);
        const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
        uint32_t base = 0;
        if ((threadIdx.x & 31) == 0 && tot) base = atomicAdd(&s_count, tot);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        uint32_t pos = base + incl - cnt;
        if (word) {
            const uint32_t rk = idx / a.W, wl = idx % a.W;
            uint32_t bits = word;
            while (bits) {
                const uint32_t bit = __ffs(bits) - 1;
                bits &= bits - 1;
                const uint32_t j = (uint32_t)local_to_global((uint64_t)wl * 32 + bit, rk, a.G, a.S);
                region[pos] = j;
                if (a.row_ptr) region_rows[pos] = a.row_ptr[j];   // (procedural networks store no rows)
                ++pos;
            }
        }
    }
    __syncthreads();
    const uint32_t n = s_count;
    if (threadIdx.x == 0) a.sl_counts[ls * a.NR + r] = n;
    if (a.desc) {
        // padded layout (G > 1): the region's spikes -> transposed segment descriptors of
        // every local tile, as the G = 1 update writes them for its own spikes; the
        // delivered events on this rank (out-degrees onto local targets) are counted here
        extern __shared__ __align__(16) uint32_t stage[];
        const uint64_t dsum = write_descriptors(a, t, r, n, region, region_rows, stage);
        if (threadIdx.x == 0 && dsum) atomicAdd(&a.delivered_cta[r % (a.NT * a.C)], (unsigned long long)dsum);
    }
}

__global__ void k_advance(uint64_t *t0, uint32_t steps, uint32_t *gbar) {
    *t0 += steps;
    if (gbar)                                        // (persistent launches: four 64-bit slots)
        for (int q = 0; q < 8; ++q) gbar[q] = 0u;
}

// PEER exchange (device-initiated): after the kernel that
// stored this rank's bitmap of step t into every rank's receive window, one thread
// publishes "step t arrived" in every window's flag of this rank (system-scope release;
// the kernel boundary has completed the bitmap stores).  The receiving side's k_peer_wait
// spins (acquire) until all G flags show step t, so the spike union of step t is in its
// window before bitmap->list reads it.  A peer that does not arrive within ~20 s sets
// xerr instead of hanging the GPU (the host reports it as an exchange error).
__device__ __forceinline__ unsigned long long *peer_flags(const SimArgs &a, uint32_t *win) {
    return reinterpret_cast<unsigned long long *>(win + 2ull * a.G * a.W);
}
__global__ void k_peer_signal(SimArgs a, uint32_t k) {
    const uint64_t t = *a.t0 + k;
    asm volatile("fence.sc.sys;" ::: "memory");
    for (uint32_t r = 0; r < a.G; ++r) {
        unsigned long long *f = peer_flags(a, a.peers[r]) + a.rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(f), "l"((unsigned long long)(t + 1)) : "memory");
    }
}
__global__ void k_peer_wait(SimArgs a, uint32_t k) {
    const uint64_t t = *a.t0 + k;
    unsigned long long *f = peer_flags(a, a.gather);
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    for (uint32_t r = 0; r < a.G; ++r) {
        while (true) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f + r) : "memory");
            if (v >= t + 1) break;
            unsigned long long now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (now - t_start > 20000000000ull) { *a.xerr = 1u + r; return; }
            __nanosleep(200);
        }
    }
    asm volatile("fence.sc.sys;" ::: "memory");
}
cudaError_t launch_peer_signal(const SimArgs &a, uint32_t k, cudaStream_t s) {
    k_peer_signal<<<1, 1, 0, s>>>(a, k);
    return cudaGetLastError();
}
cudaError_t launch_peer_wait(const SimArgs &a, uint32_t k, cudaStream_t s) {
    k_peer_wait<<<1, 1, 0, s>>>(a, k);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ launchers
template <typename K>
static cudaError_t allow_smem(K kern, size_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

cudaError_t prepare_kernels(const SimArgs &a) {
    const size_t bytes = tile_smem_bytes(a.TW, a.NR, a.prod_words);
    const size_t ub = (size_t)kStageWords * 4;
    cudaError_t e = cudaSuccess;
#define ALLOW(kern, b) if (!e) e = allow_smem(kern, b)
    ALLOW(k_update<1>, ub); ALLOW(k_update<2>, ub); ALLOW(k_update<3>, ub); ALLOW(k_update<4>, ub);
    ALLOW(k_deliver, bytes);
    ALLOW((k_fused<1, 0>), bytes); ALLOW((k_fused<1, 1>), bytes); ALLOW((k_fused<1, 2>), bytes); ALLOW((k_fused<1, 3>), bytes);
    ALLOW((k_fused<2, 0>), bytes); ALLOW((k_fused<2, 1>), bytes); ALLOW((k_fused<2, 2>), bytes); ALLOW((k_fused<2, 3>), bytes);
    ALLOW((k_fused<4, 0>), bytes); ALLOW((k_fused<4, 1>), bytes); ALLOW((k_fused<4, 2>), bytes); ALLOW((k_fused<4, 3>), bytes);
    ALLOW(k_global_atomics, tile_smem_bytes(0, a.NR, 0));
    {
        const size_t sb = small_smem_bytes(a.TW, a.model);
        if (sb <= kSmallSmemMax) {
            ALLOW(k_small<1>, sb); ALLOW(k_small<2>, sb); ALLOW(k_small<4>, sb);
        }
    }
    ALLOW(k_b2l, ub);
    if (a.nproc) ALLOW(k_deliver_proc, (((a.TW + 3u) & ~3u) + ((a.NR + 1 + 3) & ~3u) + 36) * 4);
    if (a.model == 3) {
        const size_t pb = plastic_smem_bytes(a.TW, a.NR);
        ALLOW(k_deliver_plastic, pb);
        ALLOW((k_fused<3, 0>), pb);
    }
#undef ALLOW
    return e;
}

cudaError_t launch_update(const SimArgs &a, uint32_t k, cudaStream_t s) {
    const size_t ub = (size_t)kStageWords * 4;
    switch (a.model) {
    case 1: k_update<1><<<a.NT * a.C, kBlock, ub, s>>>(a, k); break;
    case 2: k_update<2><<<a.NT * a.C, kBlock, ub, s>>>(a, k); break;
    case 3: k_update<3><<<a.NT * a.C, kBlock, ub, s>>>(a, k); break;
    case 4: k_update<4><<<a.NT * a.C, kBlock, ub, s>>>(a, k); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_deliver(const SimArgs &a, uint32_t k, bool global_atomics, int n_sm, cudaStream_t s) {
    if (global_atomics) {
        const size_t bytes = tile_smem_bytes(0, a.NR, 0);
        k_global_atomics<<<min((uint32_t)(n_sm * 4), a.NT * a.C), kBlock, bytes, s>>>(a, k);
        return cudaGetLastError();
    }
    if (a.model == 3) {
        const size_t pb = plastic_smem_bytes(a.TW, a.NR);
        k_deliver_plastic<<<a.NT, kBlock, pb, s>>>(a, k);
        return cudaGetLastError();
    }
    if (a.nproc) {                                         // procedural connectivity
        k_deliver_proc<<<a.NT, kBlock, (((a.TW + 3u) & ~3u) + ((a.NR + 1 + 3) & ~3u) + 36) * 4, s>>>(a, k);
        return cudaGetLastError();
    }
    if (!a.desc) return cudaErrorInvalidValue;             // padded layout only
    k_deliver<<<a.NT * a.C, kBlock, tile_smem_bytes(a.TW, a.NR, a.prod_words), s>>>(a, k);
    return cudaGetLastError();
}

// The fused step kernel: C > 1 launches the C CTAs of a tile as one thread-block cluster;
// every launch may start early (programmatic dependent launch, see k_fused).
template <typename K>
static void launch_step_kernel(K kern, const SimArgs &a, uint32_t k, size_t bytes, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.NT * a.C);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = a.C;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = a.C > 1 ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kern, a, k);
}

template <int M, int V>
static void fused_v(const SimArgs &a, uint32_t k, size_t bytes, cudaStream_t s) {
    launch_step_kernel(k_fused<M, V>, a, k, bytes, s);
}

template <int M>
static void fused_m(const SimArgs &a, uint32_t k, size_t bytes, cudaStream_t s) {
    if constexpr (M == 3) {                               // Brunel+ (C = 1)
        launch_step_kernel(k_fused<M, 0>, a, k, bytes, s);
    } else {
        if (a.dly) {                                       // mixed per-synapse delays
            if (a.eshift) fused_v<M, 2>(a, k, bytes, s);
            else fused_v<M, 3>(a, k, bytes, s);
        } else {
            if (a.eshift) fused_v<M, 0>(a, k, bytes, s);   // byte-offset entries
            else fused_v<M, 1>(a, k, bytes, s);            // counter-index entries
        }
    }
}

cudaError_t launch_fused(const SimArgs &a, uint32_t k, cudaStream_t s) {
    if (a.model != 3 && !a.desc) return cudaErrorInvalidValue;
    const size_t bytes = tile_smem_bytes(a.TW, a.NR, a.prod_words);
    switch (a.model) {
    case 1: fused_m<1>(a, k, bytes, s); break;
    case 2: fused_m<2>(a, k, bytes, s); break;
    case 3: fused_m<3>(a, k, plastic_smem_bytes(a.TW, a.NR), s); break;
    case 4: fused_m<4>(a, k, bytes, s); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// The persistent step kernel (k_synth_run): cooperative launch (every CTA
// co-resident, which their grid barrier needs; the launch fails instead of deadlocking).
static size_t run_smem(const SimArgs &a) {
    return a.model == 3 ? plastic_smem_bytes(a.TW, a.NR) : tile_smem_bytes(a.TW, a.NR, a.prod_words);
}
static cudaLaunchConfig_t run_config(const SimArgs &a, cudaStream_t s, cudaLaunchAttribute *at, bool coop) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.NT * a.C);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = run_smem(a);
    cfg.stream = s;
    uint32_t na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
    ++na;
    if (a.C > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = a.C;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cfg;
}

// The persistent kernel of this configuration (nullptr: none), G = 1: synth with delay 1
// (padded layout), Brunel+.
typedef void (*RunKernel)(SimArgs, uint32_t, uint32_t);
static RunKernel run_kernel(const SimArgs &a) {
    if (a.G != 1) return nullptr;
    if (a.model == 3 && a.C == 1) return k_plastic_run;  // Brunel+ (delay >= 1 via the rings)
    if (!a.desc) return nullptr;
    if (a.model == 4) {
        if (a.delay != 1 || a.dly || a.prod_words <= kSynthSid || a.TWs > 32u * 1536u || a.C > kMaxCluster)
            return nullptr;
        return a.eshift ? k_synth_run<0> : k_synth_run<1>;
    }
    // (Vogels / Brunel with delay >= 2 in the same persistent form -- update warps publishing
    //  t + 1 while the others deliver t -- measured 9.6-9.9 vs 9.4 us/step for Brunel 100K:
    //  there the update of t + 1, not the kernel boundary, is the critical path; not kept)
    return nullptr;
}

// Thread-block clusters of C one-CTA-per-SM step kernels that can be resident at once (the
// GPC layout decides: 148 CTAs in 2-clusters but 132 in 4-clusters on a B200).
uint32_t max_active_clusters(uint32_t C) {
    const size_t bytes = 200 * 1024;                      // (forces one CTA per SM)
    if (cudaFuncSetAttribute(k_fused<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * 64);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, k_fused<4, 1>, &cfg) != cudaSuccess) { cudaGetLastError(); return 0; }
    return (uint32_t)ncl;
}

bool run_supported(const SimArgs &a, int n_sm) {
    const RunKernel kern = run_kernel(a);
    if (!kern) return false;
    const size_t bytes = run_smem(a);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    uint64_t resident = 0;
    if (a.C > 1) {
        cudaLaunchAttribute at[3];
        cudaLaunchConfig_t cfg = run_config(a, nullptr, at, false);
        cfg.attrs = at + 1;                               // (cluster dimension only)
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) { cudaGetLastError(); return false; }
        resident = (uint64_t)ncl * a.C;
    } else {
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kBlock, bytes) != cudaSuccess) { cudaGetLastError(); return false; }
        resident = (uint64_t)per * n_sm;
    }
    return resident >= (uint64_t)a.NT * a.C;
}

cudaError_t launch_run(const SimArgs &a, uint32_t k, uint32_t nsteps, cudaStream_t s) {
    if (nsteps == 0) return cudaSuccess;
    const RunKernel kern = run_kernel(a);
    if (!a.gbar || !kern) return cudaErrorInvalidValue;
    // cooperative: the launch fails unless every CTA can be co-resident (co-residency was also
    // checked at creation).  SPICE_NO_COOP=1 drops the attribute for profilers that cannot
    // replay cooperative cluster launches (ncu 2025.2 reports them as empty grids); the grid
    // barrier's timeout flag still guards against a CTA that never gets an SM.
    static const bool coop = getenv("SPICE_NO_COOP") == nullptr;
    cudaLaunchAttribute at[3];
    cudaLaunchConfig_t cfg = run_config(a, s, at, coop);
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, k, nsteps);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_bitmap_to_list(const SimArgs &a, uint32_t k, cudaStream_t s) {
    k_b2l<<<a.NR, kBlock, a.desc ? (size_t)kStageWords * 4 : 0, s>>>(a, k);
    return cudaGetLastError();
}

// ------------------------------------------------------------- read-out compaction
// Recorded steps [t_begin, t_begin + nsteps) of the bitmap ring (words = G W per step) ->
// per-step global spike IDs, ascending, packed step after step (spice_spikes_prefetch: only
// the IDs cross the host link, not the bitmaps).  Global word gw (IDs 32 gw .. 32 gw + 31)
// lies in global slice gw / (S / 32) = (local slice) G + rank (the partition).
__device__ __forceinline__ uint32_t global_word(const uint32_t *bm, uint32_t gw, uint32_t G, uint32_t W,
                                                uint32_t spw, uint32_t N) {
    const uint32_t sl = gw / spw, rk = sl % G, lw = (sl / G) * spw + gw % spw;
    uint32_t w = lw < W ? bm[(uint64_t)rk * W + lw] : 0u;
    const uint32_t rem = N - 32u * gw;                       // (gw < ceil(N / 32))
    if (rem < 32u) w &= (1u << rem) - 1u;
    return w;
}
// CTA q: the spike count of step t_begin + q -> counts[q]
__global__ void __launch_bounds__(1024) k_compact_count(const uint32_t *record, uint32_t R, uint64_t words,
                                                        uint64_t t_begin, uint32_t G, uint32_t W, uint32_t S,
                                                        uint32_t N, uint32_t *counts) {
    __shared__ uint32_t s_part[32];
    const uint32_t *bm = record + ((t_begin + blockIdx.x) % R) * words;
    const uint32_t GW = (N + 31u) / 32u, spw = S / 32u;
    uint32_t c = 0;
    for (uint32_t gw = threadIdx.x; gw < GW; gw += blockDim.x) c += __popc(global_word(bm, gw, G, W, spw, N));
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if ((threadIdx.x & 31u) == 0) s_part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t v = threadIdx.x < blockDim.x / 32 ? s_part[threadIdx.x] : 0u;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (threadIdx.x == 0) counts[blockIdx.x] = v;
    }
}
// CTA q: the IDs of step t_begin + q at ids[sum of counts[0 .. q)], ascending; warp w takes a
// contiguous run of global words (its base: a scan of the warps' counts)
__global__ void __launch_bounds__(1024) k_compact_ids(const uint32_t *record, uint32_t R, uint64_t words,
                                                      uint64_t t_begin, uint32_t G, uint32_t W, uint32_t S,
                                                      uint32_t N, const uint32_t *counts, uint32_t *ids) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint64_t s_base;
    const uint32_t *bm = record + ((t_begin + blockIdx.x) % R) * words;
    const uint32_t GW = (N + 31u) / 32u, spw = S / 32u;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarps = blockDim.x / 32;
    const uint32_t chunk = (GW + nwarps * 32u - 1) / (nwarps * 32u) * 32u;
    const uint32_t g0 = min(GW, warp * chunk), g1 = min(GW, g0 + chunk);
    if (threadIdx.x == 0) {
        uint64_t b = 0;
        for (uint32_t q = 0; q < blockIdx.x; ++q) b += counts[q];
        s_base = b;
    }
    uint32_t c = 0;
    for (uint32_t gw = g0 + lane; gw < g1; gw += 32u) c += __popc(global_word(bm, gw, G, W, spw, N));
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    if (lane == 0) s_warp[warp] = c;
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = lane < nwarps ? s_warp[lane] : 0u;
        const uint32_t incl = warp_incl_scan(v);
        s_warp[lane] = incl - v;
    }
    __syncthreads();
    uint32_t *out = ids + s_base + s_warp[warp];
    uint32_t run = 0;
    for (uint32_t i = g0; i < g1; i += 32u) {                 // (warp-uniform trips)
        const uint32_t gw = i + lane;
        uint32_t w = gw < g1 ? global_word(bm, gw, G, W, spw, N) : 0u;
        const uint32_t cnt = __popc(w), incl = warp_incl_scan(cnt);
        uint32_t pos = run + incl - cnt;
        while (w) {
            const uint32_t bit = __ffs(w) - 1;
            w &= w - 1;
            out[pos++] = 32u * gw + bit;
        }
        run += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
}
cudaError_t launch_compact(const uint32_t *record, uint32_t R, uint64_t words, uint64_t t_begin, uint32_t nsteps,
                           uint32_t G, uint32_t W, uint32_t S, uint32_t N, uint32_t *counts, uint32_t *ids,
                           cudaStream_t s) {
    if (!nsteps) return cudaSuccess;
    k_compact_count<<<nsteps, 1024, 0, s>>>(record, R, words, t_begin, G, W, S, N, counts);
    k_compact_ids<<<nsteps, 1024, 0, s>>>(record, R, words, t_begin, G, W, S, N, counts, ids);
    return cudaGetLastError();
}

cudaError_t launch_advance(uint64_t *t0, uint32_t steps, cudaStream_t s, uint32_t *gbar) {
    k_advance<<<1, 1, 0, s>>>(t0, steps, gbar);
    return cudaGetLastError();
}

}  // namespace spice
