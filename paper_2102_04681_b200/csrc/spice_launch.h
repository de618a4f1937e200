// spice_launch.h — host launchers shared by the library's translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "spice_internal.cuh"

namespace spice {

// ---- step kernels (sim.cu) ----
size_t tile_smem_bytes(uint32_t tile_width, uint32_t n_regions, uint32_t prod_words);
constexpr uint32_t kSynthProdWordsHost = 8192;   // (== kSynthProdWords in sim.cu)
size_t plastic_smem_bytes(uint32_t tile_width, uint32_t n_regions);
cudaError_t prepare_kernels(const SimArgs &a);
cudaError_t launch_update(const SimArgs &a, uint32_t k, cudaStream_t s);
cudaError_t launch_deliver(const SimArgs &a, uint32_t k, bool global_atomics, int n_sm, cudaStream_t s);
cudaError_t launch_fused(const SimArgs &a, uint32_t k, cudaStream_t s);
cudaError_t launch_bitmap_to_list(const SimArgs &a, uint32_t k, cudaStream_t s);
// *t0 += steps; gbar != nullptr: clear the persistent kernel's grid-barrier slots
cudaError_t launch_advance(uint64_t *t0, uint32_t steps, cudaStream_t s, uint32_t *gbar = nullptr);
// Persistent steps (G = 1, synth with delay 1): k .. k + nsteps - 1 in one cooperative
// launch (a.gbar: grid-barrier slots);
// supported = the configuration has such a kernel and its whole grid can be co-resident.
bool run_supported(const SimArgs &a, int n_sm);
// Clusters of C one-CTA-per-SM step kernels resident at once (0 if unknown).
uint32_t max_active_clusters(uint32_t C);
cudaError_t launch_run(const SimArgs &a, uint32_t k, uint32_t nsteps, cudaStream_t s);
// Recorded bitmaps of nsteps steps -> counts[nsteps] and the packed ascending global IDs.
cudaError_t launch_compact(const uint32_t *record, uint32_t R, uint64_t words, uint64_t t_begin, uint32_t nsteps,
                           uint32_t G, uint32_t W, uint32_t S, uint32_t N, uint32_t *counts, uint32_t *ids,
                           cudaStream_t s);
cudaError_t launch_count_proc(const SimArgs &a, unsigned long long *out, uint32_t *tc, cudaStream_t s);
cudaError_t launch_settle_weights(const SimArgs &a, uint64_t t_now, uint32_t row_lo, uint32_t row_hi, float *out,
                                  cudaStream_t s);
cudaError_t launch_peer_signal(const SimArgs &a, uint32_t k, cudaStream_t s);
cudaError_t launch_peer_wait(const SimArgs &a, uint32_t k, cudaStream_t s);
size_t small_smem_bytes(uint32_t tile_width, uint32_t model);
cudaError_t launch_small(const SimArgs &a, uint32_t k0, uint32_t nsteps, cudaStream_t s);

// ---- generator (gen.cu) ----
struct GenRule {
    uint32_t src_begin, src_end, dst_begin, dst_end, kind, k, index;
    uint64_t thr;   // floor(p 2^32), 2^32 = always
};
struct GenGeom {
    uint32_t N, n_own, rank, G, S, TW, NT;
    uint32_t key0, key1;
    uint32_t pad8;       // pad every (row, tile) segment to a multiple of 8 entries
    uint32_t eshift;     // entries store (tile offset << eshift): 2 = byte offsets (padded layout)
};
// Count segment lengths cnt[s*(NT+1)+b] (+=) for one rule.
cudaError_t gen_count(const GenGeom &g, const GenRule &r, uint32_t *cnt, cudaStream_t s);
// cnt -> bnd (exclusive prefix within each row, in place; element NT = row length) and
// row_ptr (exclusive prefix over rows).  Returns nnz through *nnz (synchronises).
// Padded layout (g.pad8): bnd/row_ptr over padded lengths, true row lengths into deg[N].
cudaError_t gen_scan(const GenGeom &g, uint32_t *cnt_bnd, uint64_t *row_ptr, uint64_t *nnz,
                     uint32_t *deg, cudaStream_t s);
// Sentinel offsets in the padding of every segment (cursor = true segment lengths).
cudaError_t gen_pad_segments(const GenGeom &g, const uint64_t *row_ptr, const uint32_t *bnd,
                             const uint32_t *cursor, uint16_t *ent, cudaStream_t s);
// Sum of n u32 values (synchronises).
cudaError_t gen_sum_u32(const uint32_t *x, uint64_t n, uint64_t *out_host, cudaStream_t s);
// Fill the entries of one rule; cursor[s*(NT+1)+b] counts entries already written.
cudaError_t gen_fill(const GenGeom &g, const GenRule &r, const uint64_t *row_ptr,
                     const uint32_t *bnd, uint32_t *cursor, uint16_t *ent, cudaStream_t s);
// Sort every (row, tile) segment ascending.
cudaError_t gen_sort_segments(const GenGeom &g, const uint64_t *row_ptr, const uint32_t *bnd,
                              uint16_t *ent, cudaStream_t s);
// In-place exclusive scan of n u64 values; data[n] receives the total.
cudaError_t gen_scan_u64(uint64_t *data, uint64_t n, cudaStream_t s);
// Brunel+: plastic boxes (src x dst ranges of plastic rules).
struct PlasticBoxes {
    uint32_t n;
    uint32_t box[kMaxPlasticRules][4];
};
// Weights: w0 on plastic synapses, the sentinel -1 on static ones.
cudaError_t gen_plastic_weights(const GenGeom &g, const PlasticBoxes &pb, const uint64_t *row_ptr,
                                const uint32_t *bnd, const uint16_t *ent, float *w, float w0, cudaStream_t s);
// Per-synapse delays (reading R19): every stored entry (padding sentinels: dmin) gets the
// delay of its (source, target) pair under the rule that contains it.
struct DelayRules {
    uint32_t n;
    uint32_t box[16][4];          // src_begin, src_end, dst_begin, dst_end
    uint32_t lo[16], hi[16], index[16];
};
cudaError_t gen_delays(const GenGeom &g, const DelayRules &dr, uint32_t dmin, const uint64_t *row_ptr,
                       const uint32_t *bnd, const uint16_t *ent, uint8_t *dly, cudaStream_t s);
// Initial state (reading R15).
cudaError_t gen_init_uniform(const GenGeom &g, uint32_t field, float lo, float hi, float *out,
                             cudaStream_t s);

}  // namespace spice
