// spice_internal.cuh — shared definitions of the B200 Spice library (not part of the ABI).
//
// Product code: nothing here is shared with oracle/ (the CPU oracle is written
// separately in plain C).  Both follow the same paper passages and DESIGN.md readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spice {

// Philox counter word 3 stream tags (reading R9).
enum : uint32_t { kTagConn = 1, kTagIndeg = 2, kTagInit = 3, kTagExt = 4, kTagFire = 5 };

constexpr int kUpdateBlock = 256;     // threads per update CTA (8 warps -> 8 bitmap words)
constexpr int kDeliverBlock = 512;    // threads per delivery CTA
constexpr int kDescChunk = 1024;      // segment descriptors staged in smem per pass
constexpr uint32_t kMaxTileWidth = 49152;   // u32 counters per tile <= 192 KiB smem
constexpr int kEntPad = 64;           // u16 padding before/after the entry array

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
};

// Everything a step kernel needs, passed by value.
struct SimArgs {
    uint32_t model, N, n_exc, delay, D, rank, G, S;
    uint32_t n_own;          // owned neurons of this rank
    uint32_t W;              // bitmap words per rank
    uint32_t TW, NT, C;      // tile width, tile count, CTAs per tile
    uint64_t ring_stride;    // NT * TW
    uint32_t record_steps;
    uint32_t key0, key1;
    uint32_t global_atomics; // delivery variant
    ModelConst mc;
    // device buffers
    const uint64_t *row_ptr; // [N+1] row starts (global source rows)
    const uint32_t *bnd;     // [N * (NT+1)] segment starts within the row
    const uint16_t *ent;     // tile-local target offsets
    float *v, *ge, *gi;
    uint32_t *ref, *acc;
    uint32_t *ring;          // D * ring_stride packed receptor counts
    uint32_t *splist;        // spike list (global IDs), capacity N
    uint32_t *spcount;       // [3] per-step list lengths (rotating)
    uint32_t *record;        // record_steps * G * W words
    uint32_t *sendbuf;       // W words (G > 1)
    uint32_t *gather;        // G * W words (G > 1)
    unsigned long long *stats;   // [0] fired, [1] delivered
    const uint64_t *t0;      // step index of the first step of this graph replay
    const uint32_t *force_bits;  // W words over local indices
    const uint64_t *force_ctl;   // [0] forced step (~0 = none), [1] mode
};

}  // namespace spice
