/*
 * spice.h — C ABI of the B200-native Spice hot path (arXiv 2102.04681).
 *
 * One network slice per process and GPU ("each GPU is responsible for delivering all
 * spikes to its neurons via its synapses", §III-D).  The calls below are
 * the four north-star entry points (create / step / read_spikes / free) plus parity
 * and debug hooks used by the tests.  Plain C types only; no torch types.
 *
 * Conventions (all functions):
 *   - Return a spice_status; never throw, exit or abort.  On failure
 *     spice_last_error() (thread-local) holds a message naming the rank and step.
 *   - After SPICE_ECUDA or SPICE_ENCCL the handle is poisoned: every call except
 *     spice_free returns SPICE_ESTATE.
 *   - The library owns every device allocation it makes; callers own host buffers.
 *   - "global ID" = neuron index in [0, n_neurons); "local index" = position of an
 *     owned neuron in Listing 1 order: j = (i/S*G + g)*S + i%S.
 *   - All calls on one handle must come from one host thread.
 */
#ifndef SPICE_H
#define SPICE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPICE_ABI_VERSION 2u

#if defined(__GNUC__)
#define SPICE_API __attribute__((visibility("default")))
#else
#define SPICE_API
#endif

typedef struct spice_net spice_net;   /* opaque; owned by the library */

typedef enum {
    SPICE_OK = 0,
    SPICE_EINVAL = 1,   /* invalid configuration or argument */
    SPICE_ENOMEM = 2,   /* device or host allocation failed (message names the buffer) */
    SPICE_ECUDA = 3,    /* CUDA runtime error; handle poisoned */
    SPICE_ENCCL = 4,    /* NCCL error; handle poisoned */
    SPICE_ERANGE = 5,   /* requested steps are outside the spike record ring */
    SPICE_ETRUNC = 6,   /* output buffer too small; *total holds the size needed */
    SPICE_ESTATE = 7    /* handle poisoned or call not valid in the current state */
} spice_status;

/* Neuron models (§IV: Vogels, Brunel, Brunel+, Synth). */
enum { SPICE_VOGELS = 1, SPICE_BRUNEL = 2, SPICE_BRUNEL_PLUS = 3, SPICE_SYNTH = 4 };

/* Connectivity rule kinds.  FIXED_PROB is the paper's descriptor entry
 * {range1, range2, p} (§III-B): edge s->j iff
 * Philox4x32-10(ctr = (s, j>>2, rule index, 1), key = seed)[j&3] < floor(p 2^32).
 * FIXED_INDEGREE (the BASELINE synth rule): target j draws k sources
 * src_begin + floor(r64 |src| / 2^64), r64 from Philox(ctr = (j, k>>1, rule, 2)). */
enum { SPICE_FIXED_PROB = 0, SPICE_FIXED_INDEGREE = 1 };

/* Flags */
#define SPICE_FLAG_EXTERNAL_EXCHANGE 0x1u  /* G > 1 without NCCL: the caller moves bitmaps
                                              between spice_exchange_begin / _end */
#define SPICE_FLAG_GLOBAL_ATOMICS    0x2u  /* deliver with the paper-style column-wise
                                              warps and global atomics (A/B baseline) */
#define SPICE_FLAG_UNFUSED           0x4u  /* G = 1: separate update and delivery kernels
                                              instead of the fused deliver(t)+update(t+1) */
#define SPICE_FLAG_PROCEDURAL        0x10u /* procedural connectivity (PAPER.md:506
                                              [Knight2021]): no adjacency is stored, each tile
                                              regenerates its row segments of every spike from
                                              the FIXED_PROB Philox predicate; Vogels / Brunel /
                                              Synth-with-FIXED_PROB rules only */
#define SPICE_FLAG_USER_STREAM       0x8u  /* enqueue on spice_config.stream (may be the
                                              legacy default stream 0) instead of a
                                              library-owned non-blocking stream */

/* Spike exchange between the G ranks (§III-D/E: "the only data that need
 * to be exchanged between GPUs are spikes"; every rank must hold the union of all ranks'
 * spikes of step t before it delivers them, Fig. 2). */
enum { SPICE_EXCHANGE_NCCL = 0,   /* ncclAllGather of fixed-size bitmaps inside the step graph */
       SPICE_EXCHANGE_PEER = 1 }; /* device-initiated: the update kernel stores its bitmap words
                                     straight into every peer's receive window (CUDA IPC
                                     mapped memory over NVLink/NVSwitch, or the same GPU),
                                     and one release flag per rank and step; see
                                     spice_peer_handle / spice_peer_connect */

typedef struct {
    uint32_t src_begin, src_end;   /* range1, half-open global IDs */
    uint32_t dst_begin, dst_end;   /* range2, half-open global IDs */
    uint32_t kind;                 /* SPICE_FIXED_PROB | SPICE_FIXED_INDEGREE */
    uint32_t k;                    /* in-degree for FIXED_INDEGREE */
    uint32_t plastic;              /* 1: STDP synapses (Brunel+ E->E only) */
    uint16_t delay_min, delay_max; /* per-synapse delays (reading R19): synapse
                                      s->j of the rule has delay dmin + floor(x (dmax-dmin+1)
                                      / 2^32), x = Philox(ctr = (s, j>>2, rule, 6))[j&3];
                                      delay_min = 0: the network's delay_steps */
    double   p;                    /* probability for FIXED_PROB */
} spice_rule;

/* Model constant vectors (model_params), in order:
 *  VOGELS     [tau_m, E_L, V_t, V_r, t_ref, E_e, E_i, tau_e, tau_i, dg_e, dg_i,
 *              v_lo, v_hi, ge_lo, ge_hi, gi_lo, gi_hi]                   (17)
 *  BRUNEL     [tau_m, V_L, theta, V_r, t_ref, J_E, g, lambda_ext, v_lo, v_hi]  (10)
 *  BRUNEL_PLUS BRUNEL + [tau_plus, tau_minus, A_plus, A_minus, w_max, w0]    (16)
 *  SYNTH      []  (uses `activity`)
 * Times in ms, potentials in mV, conductances in units of g_L. */
typedef struct {
    uint32_t abi_version;          /* SPICE_ABI_VERSION */
    uint32_t model;
    uint32_t n_neurons;            /* N */
    uint32_t n_exc;                /* [0, n_exc) excitatory; n_exc == N: one population */
    const spice_rule *rules;       /* copied during create */
    uint32_t n_rules;
    uint32_t delay_steps;          /* uniform synaptic delay >= 1 */
    double   dt_ms;
    uint64_t seed;                 /* Philox key = (seed lo, seed hi) */
    double   activity;             /* SYNTH per-step firing probability */
    const double *model_params;    /* copied during create */
    uint32_t n_model_params;
    uint32_t rank, world_size;     /* this slice g and the GPU count G */
    uint32_t slice_width;          /* S, multiple of 32; 0 = spice_default_slice_width */
    int32_t  device;               /* CUDA device ordinal */
    const void *nccl_unique_id;    /* 128-byte ncclUniqueId from rank 0; required when
                                      world_size > 1 unless EXTERNAL_EXCHANGE */
    uint32_t record_steps;         /* spike record ring length in steps (>= 1) */
    uint32_t flags;                /* SPICE_FLAG_* */
    uint32_t tile_width;           /* targets per delivery tile (multiple of 32,
                                      <= 49152); 0 = auto */
    uint32_t ctas_per_tile;        /* CTAs sharing one tile (>= 1); 0 = auto */
    uint32_t exchange;             /* SPICE_EXCHANGE_NCCL | SPICE_EXCHANGE_PEER (G > 1) */
    void    *stream;               /* cudaStream_t, used with SPICE_FLAG_USER_STREAM */
    /* Device allocator for every buffer the library holds (e.g. the torch caching
     * allocator); NULL = cudaMalloc/cudaFree.  dev_alloc returns NULL on failure (then
     * SPICE_ENOMEM).  Buffers are returned through dev_free by spice_free. */
    void *(*dev_alloc)(size_t bytes, void *ctx);
    void  (*dev_free)(void *ptr, void *ctx);
    void    *alloc_ctx;
} spice_config;

/* Create this rank's slice (§III-B: the descriptor {range1, range2, p}
 * is "uploaded to the GPU where it is expanded"; §III-D: rank g expands
 * {range1, range2 ∩ owned(g), p}; §III-F P:376 + Listing 1: owned(g) = the
 * equal-width slices j with floor(j/S) mod G = g).  Allocates neuron state (SoA),
 * the delay ring of input slots, spike lists, the record ring and the step
 * graphs.  cfg and everything it points to is copied; the caller keeps ownership.
 * Collective over the world when world_size > 1 with SPICE_EXCHANGE_NCCL (communicator
 * init).  Errors: EINVAL (N = 0, p outside [0,1], ranges outside [0,N), delay 0, rules of
 * one source with overlapping destination ranges, packed receptor counts that could
 * overflow, ...), ENOMEM (message names the buffer), ECUDA, ENCCL.  *out is NULL on
 * failure. */
SPICE_API spice_status spice_create_network(const spice_config *cfg, spice_net **out);

/* Enqueue n_steps lock-step simulation steps on the library stream and return.  Step t
 * (reading R2): every owned neuron is updated, reading and clearing input slot
 * t mod D (P:161 onUpdate, "invoked by the framework on every simulation step"); the
 * spiking IDs form S_t ("inserted into one of delay many spike arrays"); G > 1: S_t
 * is exchanged so every rank holds the union; S_t is delivered row by row into
 * slot (t + delay) mod D ("delivered to all neighbors in said row"); Brunel+ applies
 * STDP on the same synapse stream (reading R13).  n_steps is decomposed into
 * replays of captured step graphs of 2^k steps (k <= 8); inside a replay every step but
 * the first is one fused kernel (delivery of t + update of t + 1) -- for synth (delay 1)
 * and Brunel+ at G = 1 all of them run in ONE persistent cooperative launch with an
 * in-kernel grid barrier per step (set SPICE_NO_PERSIST=1 at create time for one kernel
 * per step).  No host round trip; n_steps = 0 is a no-op.  ESTATE on a poisoned or
 * external-exchange handle; a grid barrier that does not complete within 10 s (a CTA
 * never scheduled) is reported as ECUDA by the next synchronising call instead of hanging. */
SPICE_API spice_status spice_step(spice_net *net, uint64_t n_steps);

/* Copy the spikes of steps [t_begin, t_end) to the host (synchronises the stream): the
 * spike arrays S_t of P:161, as the union over all ranks (Fig. 2; reading R11:
 * ascending global IDs, at most one spike per neuron and step).  ids (caller-owned,
 * cap entries) receives global IDs, ascending within each step, the same list on every
 * rank; offsets (t_end - t_begin + 1 entries, may be NULL) receives per-step starts.
 * ERANGE if a step is not in the record ring (older than record_steps or not yet
 * simulated); ETRUNC if cap is too small (then *total = spikes needed, nothing else
 * written). */
SPICE_API spice_status spice_read_spikes(spice_net *net, uint64_t t_begin, uint64_t t_end,
                               uint32_t *ids, uint64_t cap, uint64_t *offsets,
                               uint64_t *total);

/* Release everything the handle owns (device buffers through dev_free when given, the
 * graphs, the library stream, the NCCL communicator or peer mappings).  NULL-safe; valid
 * on a poisoned handle.  Collective when an NCCL communicator exists. */
SPICE_API spice_status spice_free(spice_net *net);

/* Double-buffered spike read-out for streaming runs (same data and ordering as
 * spice_read_spikes).  prefetch enqueues, on the library stream after the steps already
 * enqueued, the compaction of the recorded bitmaps of steps [t_begin, t_end) into per-step
 * ascending global IDs on the device (two kernels) and an asynchronous copy of the counts
 * and of the IDs (up to 1.25x the slot's previous total) into library-owned pinned host slot
 * `slot` (0 or 1), and returns without waiting; collect waits for that slot's copy only (an
 * event, not a stream sync, so later enqueued steps keep running), fetches any IDs beyond
 * the guess on a private copy stream, and fills ids / offsets as spice_read_spikes does
 * (ETRUNC with *total set when cap is too small; the slot stays full).  Device buffers of
 * (t_end - t_begin) x n_neurons IDs per slot are allocated on first use.  Chunks of fewer
 * than 2^16 bitmap words are copied as bitmaps and decoded on the host.  ERANGE as
 * spice_read_spikes (t_end may exceed the steps enqueued so far by 0); ESTATE when collect
 * names an empty slot. */
SPICE_API spice_status spice_spikes_prefetch(spice_net *net, uint64_t t_begin, uint64_t t_end,
                                             uint32_t slot);
SPICE_API spice_status spice_spikes_collect(spice_net *net, uint32_t slot, uint32_t *ids,
                                            uint64_t cap, uint64_t *offsets, uint64_t *total);

/* ---------------------------- parity / debug hooks --------------------------- */

/* Rows [row_begin, row_end) (global source IDs) of this rank's adjacency list: the
 * rank's half of every row split at its slice pivots (§III-D), as global target
 * IDs ascending within each row ("Each row's entries are sorted"; padding sentinels
 * removed).  tgt_global is caller-owned (cap entries); row_offsets has
 * row_end - row_begin + 1 entries.  Synchronises.  EINVAL for rows outside [0, N);
 * ETRUNC semantics as in spice_read_spikes. */
SPICE_API spice_status spice_read_connectivity(spice_net *net, uint32_t row_begin, uint32_t row_end,
                                     uint32_t *tgt_global, uint64_t cap,
                                     uint64_t *row_offsets, uint64_t *total);

/* Per-synapse delays in steps (reading R19) of this rank's synapses in the order of
 * spice_read_connectivity for rows [row_begin, row_end).  ETRUNC as above. */
SPICE_API spice_status spice_read_delays(spice_net *net, uint32_t row_begin, uint32_t row_end,
                                         uint8_t *delays, uint64_t cap, uint64_t *total);

/* Neuron state (the SoA neuron pool of P:151 §III-A) of the owned neurons in local order
 * (Listing 1; n must equal the owned count, host buffer caller-owned):
 * 0 v (f32), 1 ge (f32), 2 gi (f32), 3 refractory counter (u32), 4 synth accumulator
 * (u32), 5 pre trace x (f32; the trace of the owned neuron's own spikes, reading R13),
 * 6 post trace y (f32).  Both calls synchronise the stream and act on the state after the
 * steps enqueued so far.  EINVAL for a field the model lacks or a wrong n. */
enum { SPICE_FIELD_V = 0, SPICE_FIELD_GE = 1, SPICE_FIELD_GI = 2, SPICE_FIELD_REF = 3,
       SPICE_FIELD_ACC = 4, SPICE_FIELD_XTR = 5, SPICE_FIELD_YTR = 6 };
SPICE_API spice_status spice_read_state(spice_net *net, uint32_t field, void *host_out, uint64_t n);
SPICE_API spice_status spice_write_state(spice_net *net, uint32_t field, const void *host_in, uint64_t n);

/* The spike-array slot of the delay ring ("selecting the appropriate spike
 * array based on the current simulation step and delay") that the update of step
 * (t_now + rel) reads, rel in [0, delay], for the owned neurons in local order (n = owned
 * count): packed receptor counts (reading R10: exc in bits 0-15, inh in bits 16-31; one
 * population: all 32 bits) and, for Brunel+, plastic fixed-point sums rint(w 2^32)
 * (plastic may be NULL).  Synchronises.  EINVAL for rel > delay or a wrong n. */
SPICE_API spice_status spice_read_input(spice_net *net, uint32_t rel, uint32_t *counts,
                              int64_t *plastic, uint64_t n);

/* Plastic weights (the synapse pool mapped 1:1 onto the adjacency list) of this
 * rank's synapses in the order of spice_read_connectivity for rows [row_begin, row_end);
 * non-plastic synapses read as 0.  Brunel+ only (EINVAL otherwise).  ETRUNC as above. */
SPICE_API spice_status spice_read_weights(spice_net *net, uint32_t row_begin, uint32_t row_end,
                                float *w, uint64_t cap, uint64_t *total);

/* Teacher forcing of the next step (the north star's "per-step synaptic input under
 * teacher-forced identical spikes" parity criterion): mode 1 replaces its spike set by the
 * owned neurons among ids (global IDs), mode 2 adds them to the natural set; a forced
 * spike resets the neuron like a natural one (reading R5).  Synchronises.  EINVAL for an
 * id >= N or another mode. */
SPICE_API spice_status spice_force_spikes(spice_net *net, const uint32_t *ids, uint64_t n, int mode);

/* Counters since create (synchronises): steps done, spikes emitted by owned neurons,
 * synaptic events delivered to owned neurons (one per (spike, synapse) pair, P:200;
 * the numerator of the BASELINE metric "synaptic events/sec"). */
SPICE_API spice_status spice_stats(spice_net *net, uint64_t *steps, uint64_t *fired,
                         uint64_t *delivered);

/* The cudaStream_t the library enqueues on (for CUDA-event timing by the caller). */
SPICE_API void *spice_stream(spice_net *net);

/* Synchronise the library stream. */
SPICE_API spice_status spice_sync(spice_net *net);

/* Sizes of this slice: owned neurons, synapses, delivery tiles, device bytes held. */
SPICE_API spice_status spice_info(spice_net *net, uint64_t *n_owned, uint64_t *n_synapses,
                        uint32_t *n_tiles, uint32_t *tile_width, uint32_t *ctas_per_tile,
                        uint64_t *device_bytes);

/* Setup cost (§IV "Setup Time": "our actual setup kernel generates
 * networks at ~200M synapses/ms").  gen_ms: device time of the generator kernels of
 * this slice (count, scan, fill, pad, sort; CUDA events on the library stream, without
 * allocations or host round trips).  create_ms: host wall time of spice_create_network
 * (allocation, generation, state init, graph capture).  Either pointer may be NULL. */
SPICE_API spice_status spice_setup_times(spice_net *net, double *gen_ms, double *create_ms);

/* Run n_steps steps with each kernel launched individually and bracketed by CUDA events
 * on the library stream; writes the average device time per launch in ms:
 * [0] neuron update kernel, [1] delivery kernel, [2] fused deliver(t)+update(t+1) kernel
 * (G = 1; 0 otherwise), [3] exchange (NCCL all-gather + bitmap->list; G > 1), and, when
 * cap >= 5, [4] the fused kernel inside a captured graph of 32 back-to-back launches, or
 * one persistent launch of 32 steps, per step (the configuration spice_step runs; G = 1,
 * 0 otherwise), timed over n_steps / 32 replays.
 * *n_kernels = entries written (cap >= 4).  Advances the network.  Synchronises. */
SPICE_API spice_status spice_profile(spice_net *net, uint64_t n_steps, double *ms_per_kernel,
                                     uint32_t cap, uint32_t *n_kernels);

/* Diagnostics.  With SPICE_PHASES=1 in the environment at create time, thread 0 of every
 * fused-kernel CTA accumulates, per launch, the SM-clock offset of each phase boundary
 * from the kernel start: out[cta*16 + slot] for slots 1..12 (1 counters zeroed, 2 region
 * prefix, 3 descriptors staged, 4 warp 0 done delivering, 5 delivery barrier, 6 delivered
 * stat, 7 update loop, 8 spike rows, 9 descriptors written, 12 end); slot 13 = launches,
 * 14/15 = %globaltimer (ns) at start/end of the last launch.  *count = NT*C*16 (0 when
 * disabled).  Synchronises. */
SPICE_API spice_status spice_debug_phases(spice_net *net, uint64_t *out, uint64_t cap, uint64_t *count);

/* Number of kernels the library launches per simulated step (evidence for benches). */
SPICE_API uint32_t spice_kernels_per_step(spice_net *net);
/* Exact number of this library's kernel launches enqueued by spice_step(net, n_steps)
 * (NCCL's own kernels excluded); small networks run a whole graph chunk in one launch. */
SPICE_API uint64_t spice_launches(spice_net *net, uint64_t n_steps);

/* Thread-local message of the last failing call ("" if none). */
SPICE_API const char *spice_last_error(void);

/* ------------------------- multi-GPU plumbing -------------------------------- */

/* Fill 128 bytes with a fresh ncclUniqueId (rank 0 only; broadcast it yourself).  The
 * NCCL exchange replaces the paper's host-driven hierarchical cudaMemcpy synchronisation
 * (§III-E, Fig. 2) by one all-gather of fixed-size bitmaps per step. */
SPICE_API spice_status spice_nccl_unique_id(void *out128);

/* External exchange (SPICE_FLAG_EXTERNAL_EXCHANGE; used for single-GPU "virtual rank"
 * tests of the exchange step): begin enqueues the neuron update of the next
 * step, leaving this rank's spike
 * bitmap (words_per_rank u32 words) in the send buffer; the caller must fill the receive
 * buffer (world_size * words_per_rank words, rank r at offset r * words_per_rank) and
 * then call end, which enqueues bitmap->list conversion and delivery. */
SPICE_API spice_status spice_exchange_begin(spice_net *net);
SPICE_API spice_status spice_exchange_end(spice_net *net);
/* The NCCL graph's G > 1 step sequence (padded layout): end_fused enqueues bitmap->list
 * + descriptors of step t and the fused kernel (delivery of t, update of t + 1), leaving
 * step t+1's bitmap in the send buffer, so the next step starts with the exchange (no
 * begin).  Sequence: begin; (exchange, end_fused) x (T - 1); exchange, end.  The network
 * state is consistent only after a plain end.  SPICE_ESTATE when the network has no fused
 * G > 1 path (G = 1, unpadded layout, global atomics). */
SPICE_API spice_status spice_exchange_end_fused(spice_net *net);
/* Device-to-device copy of src's send buffer into dst's receive segment for src's rank
 * (both handles on the same device; ordered after src's update; returns when done). */
SPICE_API spice_status spice_exchange_put(spice_net *dst, spice_net *src);

/* External exchange over the caller's own transport (MPI, a custom NVLink kernel, ...;
 * P:287-290 §III-D/E: every rank needs every rank's spikes of the step).  get_send copies
 * this rank's send buffer (words_per_rank u32 words: the step's spike bitmap, valid after
 * spice_exchange_begin or spice_exchange_end_fused) to `out`; set_recv fills rank r's
 * receive segment (words_per_rank words) from `words`.  on_device != 0: device pointers on
 * the network's device, the copy is enqueued on the network's stream (asynchronous, stream
 * ordered, capturable); 0: host memory, the call returns when the copy is done.  The caller
 * owns both buffers; bits past rank r's owned neurons are ignored.  SPICE_EINVAL for a null pointer or rank >= world_size, SPICE_ESTATE
 * for a network without SPICE_FLAG_EXTERNAL_EXCHANGE. */
SPICE_API spice_status spice_exchange_get_send(spice_net *net, uint32_t *out, int on_device);
SPICE_API spice_status spice_exchange_set_recv(spice_net *net, uint32_t rank, const uint32_t *words, int on_device);

/* PEER exchange (spice_config.exchange = SPICE_EXCHANGE_PEER, world_size > 1): the
 * device-initiated spike synchronisation (§III-D/E, "the
 * spike synchronization time is entirely dominated by CUDA API overhead").  Every rank owns a
 * receive window of 2 x G x W words (step parity x rank x bitmap word) plus G arrival flags;
 * the neuron-update kernel stores its bitmap words straight into all G windows (NVLink /
 * NVSwitch stores through CUDA IPC mappings, or plain stores on the same GPU), a one-thread
 * kernel then releases this rank's flag for the step in every window, and before
 * bitmap->list each rank's one-thread wait kernel acquires all G flags.  No host round trip
 * and no library call per step.  Setup: create every rank, get each rank's 128-byte handle
 * with spice_peer_handle, all-gather them (rank order) with any host transport, and pass
 * the G x 128 bytes to spice_peer_connect, which maps the peers' windows and captures the
 * step graphs; spice_step returns ESTATE until then.  Ranks of one process may share a GPU
 * (the handle carries the process ID; same-process windows are used directly).  A peer
 * that stalls > 20 s makes the next synchronising call return SPICE_ENCCL. */
SPICE_API spice_status spice_peer_handle(spice_net *net, void *out128);
SPICE_API spice_status spice_peer_connect(spice_net *net, const void *handles);

/* ------------------- static partition (host-only, no GPU needed) -------------- */
/* PAPER.md §III-F P:376 strided slices, Listing 1 P:496 (reading R1). */
SPICE_API uint32_t spice_partition_owner(uint64_t j, uint32_t world_size, uint32_t slice_width);
SPICE_API uint64_t spice_partition_local_to_global(uint64_t i, uint32_t rank, uint32_t world_size,
                                         uint32_t slice_width);
SPICE_API uint64_t spice_partition_owned_count(uint64_t n, uint32_t rank, uint32_t world_size,
                                     uint32_t slice_width);
/* Decode one step's gathered bitmaps (G segments of W words; bit i of segment r =
 * local index i of rank r) into ascending global IDs (the union of all ranks' spikes,
 * Fig. 2).  ETRUNC with *total when cap is too small. */
SPICE_API spice_status spice_decode_bitmaps(const uint32_t *words, uint32_t world_size, uint32_t W,
                                            uint32_t slice_width, uint32_t *ids, uint64_t cap,
                                            uint64_t *total);
/* Default S: a multiple of 32 giving each rank >= ~100 slices when N allows. */
SPICE_API uint32_t spice_default_slice_width(uint64_t n, uint32_t world_size);

#ifdef __cplusplus
}
#endif
#endif /* SPICE_H */
