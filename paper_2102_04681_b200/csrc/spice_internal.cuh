// spice_internal.cuh — shared definitions of the B200 Spice library (not part of the ABI).
//
// Product code: nothing here is shared with oracle/ (the CPU oracle is written
// separately in plain C).  Both follow the same paper passages and DESIGN.md readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spice {

// Philox counter word 3 stream tags (reading R9).
enum : uint32_t { kTagConn = 1, kTagIndeg = 2, kTagInit = 3, kTagExt = 4, kTagFire = 5, kTagDelay = 6 };

#ifndef SPICE_KBLOCK
#define SPICE_KBLOCK 1024
#endif
#ifndef SPICE_PHASES_BUILD
#define SPICE_PHASES_BUILD 0    // in-kernel phase clocks (tools/phases.py builds a variant)
#endif
#ifndef SPICE_ACC_PREFETCH
#define SPICE_ACC_PREFETCH 1    // synth update: accumulators loaded one loop iteration ahead
#endif
#ifndef SPICE_PROD_WARPS
#define SPICE_PROD_WARPS 2      // synth fast path: producer warps beside the delivering warps
#endif
#ifndef SPICE_RW
#define SPICE_RW (SPICE_WIN_SHIFT == 3 ? 2 : 1)   // ring delivery: windows per lane per iteration
#endif
constexpr int kBlock = SPICE_KBLOCK;  // threads per tile CTA (update / deliver / fused)
constexpr int kStageWords = 12288;     // bnd rows staged per descriptor-transposition pass
constexpr uint32_t kMaxTileWidth = 49152;   // u32 counters per tile <= 192 KiB smem
constexpr uint32_t kMaxRegions = 4096;      // spike-list regions per step
constexpr uint32_t kB2LWords = 256;         // minimum bitmap words per bitmap->list region
constexpr int kEntPad = 64;           // u16 padding before/after the entry array
// Padded layout: every (row, tile) segment is a whole number of delivery windows of
// kWin u16 entries, starting at a window boundary.  16-byte windows (kWinShift = 3)
// measured faster than sector-sized 32-byte windows (kWinShift = 4: +12 % padding
// atomics, synth delivery 12.3 -> 14.5 us, DESIGN.md delivery log).
#ifndef SPICE_WIN_SHIFT
#define SPICE_WIN_SHIFT 3
#endif
constexpr uint32_t kWinShift = SPICE_WIN_SHIFT;
constexpr uint32_t kWin = 1u << kWinShift;
constexpr uint32_t kDummy = 64;       // dummy counters past the tile (padding sentinels)
constexpr uint32_t kPtabSmem = 128;   // Poisson inversion table entries staged in smem
constexpr uint32_t kMaxPadTile = 16320;   // padded layout, byte-offset entries: (TW + kDummy) * 4 fits a u16
constexpr uint32_t kMaxPadTileWord = 65472;   // padded layout, word-offset entries: TW + kDummy fits a u16
constexpr uint32_t kMaxCluster = 8;       // CTAs per tile cluster (portable cluster size)

// Device-side bounds checks of the hot kernels' indices (debug builds only: -DSPICE_CHECKS=1,
// tools/checked_run.py; compute-sanitizer is not available on the GPU pool).  A violated
// check traps: the launch fails with an illegal-instruction error naming no data.
#if SPICE_CHECKS
#define SPICE_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define SPICE_CHECK(cond) do { } while (0)
#endif

// Philox4x32-10 (Salmon et al., SC'11).  Multipliers 0xD2511F53 / 0xCD9E8D57, Weyl
// key increments 0x9E3779B9 / 0xBB67AE85; 10 rounds.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ uint32_t word_of(const uint4 &v, uint32_t w) {
    return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
}

// Static strided partition (§III-F, Listing 1; reading R1).
__host__ __device__ __forceinline__ uint64_t local_to_global(uint64_t i, uint32_t g, uint32_t G,
                                                             uint32_t S) {
    return (i / S * G + g) * S + i % S;
}

// Model constants, all derived on the host in double and rounded once to float.
struct ModelConst {
    float h, EL, Vt, Vr, Ee, Ei, ke, ki, dge, dgi;   // Vogels
    float theta, JE, JI;                              // Brunel (V_L in EL, V_r in Vr)
    uint32_t R;                                       // refractory steps
    uint64_t thr_fire;                                // synth: floor(a 2^32) (2^32 = always)
    const uint64_t *ptab;                             // Brunel: Poisson inversion table
    uint32_t ptab_len;
    uint32_t ptab_half;                               // half the power of two >= ptab_len
    float ap, am, Ap, Am, wmax;                       // Brunel+ STDP (reading R13)
};

constexpr int kMaxPlasticRules = 4;

// Everything a step kernel needs, passed by value.
//
// Connectivity (destination-tiled, source-major CSR): owned targets (local indices) are
// cut into NT tiles of TW; row s = ent[row_ptr[s] .. row_ptr[s+1]) is the concatenation of
// its tile segments, segment (s, b) = row_ptr[s] + [bnd[s*(NT+1)+b], bnd[s*(NT+1)+b+1]);
// entries are u16 offsets inside the tile, ascending within a segment.  Rows stay
// contiguous so that neighbouring tiles' segments share DRAM sectors through L2.
//
// Spike lists: per step parity p, NR regions of RS slots; region r holds counts[p*NR+r]
// spikes: global source IDs at ids[(p*NR + r)*RS ...] and their row starts at rows[...]
// (order inside a step is irrelevant to the integer accumulation, reading R10; the
// bitmap record is the canonical output).
struct SimArgs {
    uint32_t model, N, n_exc, delay, D, rank, G, S;
    uint32_t n_own;          // owned neurons of this rank
    uint32_t W;              // bitmap words per rank
    uint32_t TW, NT, C;      // tile width, tile count, CTAs per tile
    uint32_t TWs;            // targets per CTA slice = TW / C: CTA x updates the owned
                             // neurons [x TWs, (x+1) TWs) and owns spike-list region x.
                             // With C > 1 (G = 1) the C CTAs of a tile form a thread-block
                             // cluster: each accumulates its share of the tile's visits into
                             // a full-tile shared counter array, then reduces its slice
                             // across the cluster through distributed shared memory
    uint64_t ring_stride;    // NT * TW
    uint32_t record_steps;
    uint64_t mD, mR;         // fast remainders mod D / record_steps: floor((2^64 - 1) / m) + 1
    uint32_t pdl;            // 1: fused step kernels use programmatic dependent launch
    uint64_t nnz;            // stored entries (incl. padding sentinels): bounds of ent / w / dly
    uint32_t persist;        // 1: the steps of a replay in one persistent launch (k_synth_run)
    uint32_t *gbar;          // [10] its grid-barrier slots (barrier i of a launch: 64-bit word
                             // i mod 4, arrivals low / payload high; zero between launches)
                             // and a timeout flag at [8]
    uint32_t pl_split;       // Brunel+: plastic fixed point q summed as (q mod 2^16) and
                             // (q >> 16) in two u32 words (no carry round trip; abi.cu proves
                             // neither sum can wrap), else low word + carry into the high word
    uint32_t prod_words;     // synth fast path (G = 1): producer-warp shared-memory words
    uint32_t key0, key1;
    uint32_t NR, RS;         // spike-list regions
    unsigned long long *ptimes;   // diagnostics (SPICE_PHASES=1): per CTA [16] phase clocks
    ModelConst mc;
    // connectivity
    const uint64_t *row_ptr; // [N+1]
    const uint32_t *bnd;     // [N * (NT+1)]
    const uint16_t *ent;
    const uint32_t *deg;     // padded layout (G = 1, not Brunel+): every segment is padded to
                             // a multiple of 8 entries with sentinels >= TW (dummy counters
                             // TW .. TW+63); deg[s] = true out-degree (delivered-event count)
    uint32_t eshift;         // entries hold (tile offset << eshift); 2 (byte offsets) when padded
    // state
    float *v, *ge, *gi;
    uint32_t *ref, *acc;
    uint32_t *ring;          // D * ring_stride packed receptor counts
    const uint8_t *dly;      // mixed per-synapse delays (reading R19): delay of every stored
                             // entry, aligned with ent; nullptr = every synapse has `delay`.
                             // `delay` is then the minimum delay (the shared-memory path);
                             // longer-delay events go to ring slot t + d with global atomics
    // spikes
    uint32_t *sl_ids;        // 3 * NR * RS (copy t mod 3)
    uint64_t *sl_rows;       // 3 * NR * RS row starts of the listed spikes
    uint32_t *sl_counts;     // 2 * NR
    // G = 1 (padded layout): per-step segment descriptors, written transposed by the
    // updating CTAs into one dense list per destination tile: desc[((t mod 3)*NT + b)*dstride + i]
    // = first 16-byte window (bits 0-31) | window count (32-62) | inh (63) of the i-th
    // spike of the step restricted to tile b (list order = producer arrival order)
    uint64_t *desc;
    uint64_t dstride;        // descriptor slots per (parity, tile) list (>= owned neurons)
    uint32_t *dcount;        // [4] descriptors per list of step t at dcount[t % 4]
    uint32_t *record;        // record_steps * G * W words
    uint32_t *sendbuf;       // W words (G > 1, NCCL exchange)
    uint32_t *gather;        // G * W words (G > 1); PEER exchange: this rank's receive window,
                             // 2 step-parity halves of G * W words, then G u64 arrival flags
    uint32_t *const *peers;  // PEER exchange: device array of the G ranks' receive windows
                             // (this rank's own at index rank; CUDA IPC mappings of the others)
    uint32_t *xerr;          // PEER exchange: set when a peer's flag did not arrive in time
    unsigned long long *fired_cta;      // [NT]   per-CTA counters (no shared atomics)
    unsigned long long *delivered_cta;  // [NT*C]
    // Brunel+ (model 3): per-synapse weights aligned with ent, fixed-point plastic input
    // ring, pre traces x for all N sources (double-buffered by step parity), post traces
    // y for owned neurons, and per-target in-synapse index (absolute entry, source).
    float *w;
    long long *pring;        // D * ring_stride, rint(w 2^32) sums
    // event-driven STDP state (reading R13), double-buffered by step parity:
    uint32_t *pre_ts;        // [3][N] step of every source's last spike (~0 = none), copy t mod 3
    float *pre_c;            // [3][N] its pre trace just after that spike, X(ts) + 1
    uint32_t *post;          // [2][ring_stride] uint4 per owned neuron: last three spike
                             // steps (most recent first) and cy = Y(ts) + 1 (float bits)
    uint32_t *post_mask;     // [ring_stride][64] post-spike bit ring (2048 steps)
    const float *tab_p, *tab_m;   // [8192] exp(-k dt / tau+-), rounded once
    uint32_t nproc;          // procedural connectivity (NEXT-4): rules regenerated per spike
    uint32_t proc[16][8];    // src_b, src_e, dst_b, dst_e, thr lo, thr hi, rule index, dmin | dmax << 16
    uint32_t npl;                                  // plastic boxes (src x dst ranges)
    uint32_t pl[kMaxPlasticRules][4];
    const uint64_t *t0;      // step index of the first step of this graph replay
    const uint32_t *force_bits;  // W words over local indices
    const uint64_t *force_ctl;   // [0] forced step (~0 = none), [1] mode
};

}  // namespace spice
