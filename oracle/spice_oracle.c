/*
 * spice_oracle.c — CPU ORACLE for the Spice hot path (arXiv 2102.04681).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2102_04681_b200/) never links, imports or executes anything in oracle/.
 * This file shares no code, header, table or constant generator with the CUDA
 * path; both receive the same inputs (workloads/) and derive everything else on
 * their own.
 *
 * What it computes: the plain time-driven simulation the method reaches exactly
 * (§III-A..C, Listing 1).  It is single-threaded, slow
 * and literal:
 *   build:  every descriptor rule {range1, range2, p} (§III-B) is expanded by
 *           brute force over all (source, target) pairs (fixed probability) or all
 *           (target, k) draws (fixed in-degree, reading R9); rows are the sorted target
 *           lists of each source ("Each row's entries are sorted").  An optional
 *           ownership filter keeps only targets owned by rank g of G with slice width
 *           S (the descriptor split of P:279-283 §III-D with the strided slices of
 *           P:376 §III-F and Listing 1).
 *   step t: (1) update every neuron in ascending ID order, reading and clearing its
 *           input slot I[t mod D] (P:161 onUpdate; readings R2-R5, R12);
 *           (2) S_t = the sorted set of neurons that spiked;
 *           (3) Brunel+: eager STDP (reading R13);
 *           (4) for s in S_t ascending, for each target i of row s ascending:
 *               I[(t+delay) mod D][i] += q(s)   ("delivered to all neighbors
 *               in said row"; reading R10 for integer receptor counts);
 *           (5) record S_t.
 *
 * Precision: compiled twice.  -DORC_REAL=float gives "mirror32", the paper's
 * "single precision arithmetic and Euler integration" (§IV-A) with every
 * operation written out separately (no contraction: built with -ffp-contract=off).
 * -DORC_REAL=double gives "ref64", used for the closed-form pins.
 *
 * Parity pins: see tests/test_oracle_*.py.  Parts without an external pin are
 * marked "parity unpinned" below and in DESIGN.md.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORC_TRACE_LEN 8192    /* closed-form trace table length (reading R13) */
#ifndef ORC_REAL
#define ORC_REAL float
#endif
typedef ORC_REAL real;

#define EXPORT __attribute__((visibility("default")))

enum { ORC_VOGELS = 1, ORC_BRUNEL = 2, ORC_BRUNEL_PLUS = 3, ORC_SYNTH = 4 };
enum { ORC_FIXED_PROB = 0, ORC_FIXED_INDEGREE = 1 };
/* Philox counter word 3 stream tags (reading R9 / SURVEY App. B) */
enum { TAG_CONN = 1, TAG_INDEG = 2, TAG_INIT = 3, TAG_EXT = 4, TAG_FIRE = 5, TAG_DELAY = 6 };

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:  */
/* as easy as 1, 2, 3"): 10 rounds of the 4x32 S-box with Weyl key schedule.  */
/* Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt). */
/* ------------------------------------------------------------------------- */
EXPORT void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint32_t philox_word(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                            uint32_t key0, uint32_t key1, unsigned which)
{
    uint32_t ctr[4] = { w0, w1, w2, w3 }, key[2] = { key0, key1 }, out[4];
    orc_philox(ctr, key, out);
    return out[which];
}

/* Bernoulli threshold floor(p * 2^32) (reading R9), as a 64-bit value so p = 1
 * gives 2^32 (every 32-bit draw is below it). */
static uint64_t prob_threshold(double p)
{
    if (p <= 0.0) return 0;
    if (p >= 1.0) return (uint64_t)1 << 32;
    return (uint64_t)floor(p * 4294967296.0);
}

/* Poisson inversion table (reading R12): T_k = floor(2^32 F(k)), F the Poisson
 * CDF accumulated as p0 = exp(-lambda), p_k = p_{k-1} * lambda / k.  The table
 * stops at the first k with T_k >= 2^32 - 1 (that entry is stored as 2^32).
 * Pinned against scipy.stats.poisson.cdf (tests/test_oracle_pins.py). */
EXPORT uint32_t orc_poisson_table(double lambda, uint64_t *out, uint32_t cap)
{
    double pk = exp(-lambda), F = pk;
    for (uint32_t k = 0; k < cap; k++) {
        double T = floor(F * 4294967296.0);
        if (T >= 4294967295.0) { out[k] = (uint64_t)1 << 32; return k + 1; }
        out[k] = (uint64_t)T;
        pk = pk * lambda / (double)(k + 1);
        F = F + pk;
    }
    return 0; /* cap too small */
}

/* ------------------------------------------------------------------------- */
/* Static strided partition (§III-F, Listing 1, reading R1).    */
/* ------------------------------------------------------------------------- */
EXPORT uint32_t orc_owner(uint64_t j, uint32_t G, uint32_t S) { return (uint32_t)((j / S) % G); }

/* Listing 1: j = (i / S * NGPU + GID) * S + i % S   (the "% S" lost at P:496). */
EXPORT uint64_t orc_local_to_global(uint64_t i, uint32_t g, uint32_t G, uint32_t S)
{
    return (i / S * G + g) * S + i % S;
}

/* ------------------------------------------------------------------------- */
/* Network                                                                    */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint32_t src_begin, src_end, dst_begin, dst_end;
    uint32_t kind, k, plastic;
    uint16_t delay_min, delay_max;    /* per-synapse delays (reading R19); 0 = network delay */
    double p;
} orc_rule;

typedef struct {
    uint32_t model, n, n_exc, delay, D, n_rules;
    uint32_t key0, key1;
    double dt, activity;
    double prm[32];
    uint32_t pg, pG, pS;              /* ownership filter (pG = 1: everything) */
    orc_rule *rules;
    /* connectivity: CSR over all n sources, global target IDs, rows ascending */
    uint64_t *row_ptr;
    uint32_t *tgt;
    uint8_t *plastic;                 /* per edge */
    uint16_t *dly;                    /* per edge: synaptic delay in steps (reading R19) */
    real *w;                          /* per edge (Brunel+ plastic edges) */
    uint64_t nnz;
    /* CSC index of plastic edges (for eager potentiation, R13) */
    uint64_t *in_ptr;
    uint64_t *in_edge;
    uint32_t *edge_src;
    /* state (SoA) */
    real *v, *ge, *gi;
    /* STDP traces in event-driven closed form (reading R13): per neuron the step of its last
     * spike (-1 none) and the pre / post trace values just after it, cx = X(ts) + 1,
     * cy = Y(ts) + 1; X(t) = cx P+[t - ts], Y(t) = cy P-[t - ts] */
    int64_t *ts;
    real *cx, *cy;
    real *pp, *pm;                    /* P+[k] = exp(-k dt / tau+), P-[k], k < ORC_TRACE_LEN */
    uint32_t *ref, *acc;
    uint32_t *ring;                   /* D x n packed receptor counts (R10) */
    int64_t *pring;                   /* D x n plastic fixed-point sums (R10) */
    /* derived scalars */
    real h, ke, ki, dge, dgi, JE, JI, Ap, Am, wmax;
    real EL, Vt, Vr, Ee, Ei, theta;
    uint32_t R;
    uint64_t thr_fire;
    uint64_t ptab[256];
    uint32_t ptab_len;
    /* run record */
    uint64_t t;
    uint32_t *sp; uint64_t sp_len, sp_cap;
    uint64_t *sp_off; uint64_t off_cap;   /* sp_off[t] .. sp_off[t+1] */
    uint64_t *delivered;
    /* teacher forcing: one pending forced step; mode 1 replace S_t, 2 add to S_t */
    int64_t force_t;
    int force_mode;
    uint8_t *force_bits;
} orc_net;

static void *xcalloc(size_t n, size_t sz) { void *p = calloc(n ? n : 1, sz); return p; }

/* Sort each row's (target, plastic) pairs ascending by target (stable for equal
 * targets is irrelevant: equal targets have equal plastic flags within a rule and
 * rules of one source have disjoint destination ranges — enforced by build). */
typedef struct { uint32_t t; uint32_t pl; } tgt_pl;
static int cmp_tp(const void *a, const void *b)
{
    const tgt_pl *x = a, *y = b;
    if (x->t != y->t) return (x->t > y->t) - (x->t < y->t);
    return (x->pl > y->pl) - (x->pl < y->pl);
}

static int owned(const orc_net *N, uint64_t j) { return N->pG <= 1 || orc_owner(j, N->pG, N->pS) == N->pg; }

/* The two edge rules (reading R9), written once and used by the build and by the
 * sampled-row / sampled-column queries below. */
static int prob_edge(uint32_t key0, uint32_t key1, uint32_t r, uint64_t thr, uint64_t s, uint64_t j)
{
    /* edge s -> j iff Philox(ctr=(s, j>>2, r, TAG_CONN))[j & 3] < floor(p 2^32) */
    uint32_t x = philox_word((uint32_t)s, (uint32_t)(j >> 2), r, TAG_CONN, key0, key1, (unsigned)(j & 3));
    return (uint64_t)x < thr;
}
static uint64_t indeg_source(uint32_t key0, uint32_t key1, uint32_t r, const orc_rule *R, uint64_t j, uint32_t k)
{
    /* target j's k-th draw: r64 from Philox(ctr=(j, k>>1, r, TAG_INDEG)) words 2(k&1),
     * 2(k&1)+1; source = src_begin + floor(r64 |src| / 2^64). */
    uint64_t nsrc = (uint64_t)R->src_end - R->src_begin;
    uint32_t ctr[4] = { (uint32_t)j, k >> 1, r, TAG_INDEG }, key[2] = { key0, key1 }, o[4];
    orc_philox(ctr, key, o);
    uint64_t r64 = ((uint64_t)o[2 * (k & 1) + 1] << 32) | o[2 * (k & 1)];
    return R->src_begin + (uint64_t)(((unsigned __int128)r64 * nsrc) >> 64);
}

/* Edge enumeration by brute force.  pass 0 counts per source, pass 1 fills.  */
static void enumerate_edges(orc_net *N, int pass, uint64_t *cursor)
{
    for (uint32_t r = 0; r < N->n_rules; r++) {
        const orc_rule *R = &N->rules[r];
        if (R->kind == ORC_FIXED_PROB) {
            uint64_t thr = prob_threshold(R->p);
            for (uint64_t s = R->src_begin; s < R->src_end; s++)
                for (uint64_t j = R->dst_begin; j < R->dst_end; j++) {
                    if (!owned(N, j)) continue;
                    if (prob_edge(N->key0, N->key1, r, thr, s, j)) {
                        if (pass == 0) N->row_ptr[s + 1]++;
                        else { uint64_t e = cursor[s]++; N->tgt[e] = (uint32_t)j; N->plastic[e] = (uint8_t)R->plastic; }
                    }
                }
        } else {
            for (uint64_t j = R->dst_begin; j < R->dst_end; j++) {
                if (!owned(N, j)) continue;
                for (uint32_t k = 0; k < R->k; k++) {
                    uint64_t s = indeg_source(N->key0, N->key1, r, R, j, k);
                    if (pass == 0) N->row_ptr[s + 1]++;
                    else { uint64_t e = cursor[s]++; N->tgt[e] = (uint32_t)j; N->plastic[e] = (uint8_t)R->plastic; }
                }
            }
        }
    }
}

static int cmp_u32v(const void *a, const void *b)
{
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

/* Per-synapse delay (reading R19, "per-synapse delays"): a rule with delay range
 * [dmin, dmax] gives synapse s -> j the delay dmin + floor(x (dmax - dmin + 1) / 2^32),
 * x = Philox(ctr=(s, j>>2, r, TAG_DELAY))[j&3]; a rule without a range (delay_min = 0)
 * uses the network delay.  Multapses of one pair share the delay. */
static uint32_t rule_dmin(const orc_rule *R, uint32_t net_delay) { return R->delay_min ? R->delay_min : net_delay; }
static uint32_t rule_dmax(const orc_rule *R, uint32_t net_delay)
{
    uint32_t lo = rule_dmin(R, net_delay);
    return R->delay_min && R->delay_max > lo ? R->delay_max : lo;
}
static uint32_t edge_delay(uint32_t key0, uint32_t key1, const orc_rule *R, uint32_t r, uint32_t net_delay,
                           uint64_t s, uint64_t j)
{
    uint32_t lo = rule_dmin(R, net_delay), hi = rule_dmax(R, net_delay);
    if (hi == lo) return lo;
    uint32_t x = philox_word((uint32_t)s, (uint32_t)(j >> 2), r, TAG_DELAY, key0, key1, (unsigned)(j & 3));
    return lo + (uint32_t)(((uint64_t)x * (uint64_t)(hi - lo + 1)) >> 32);
}

/* Sampled row: the sorted targets of source s under all rules (brute force over all
 * targets; fixed in-degree rules scan every target's draws), restricted to targets
 * owned by rank pg of pG with slice width pS.  Returns the row length (writes at most cap). */
EXPORT uint64_t orc_row(const orc_rule *rules, uint32_t n_rules, uint64_t seed, uint32_t s,
                        uint32_t pg, uint32_t pG, uint32_t pS, uint32_t *out, uint64_t cap)
{
    uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    uint64_t n = 0;
    for (uint32_t r = 0; r < n_rules; r++) {
        const orc_rule *R = &rules[r];
        if (R->kind == ORC_FIXED_PROB) {
            if (s < R->src_begin || s >= R->src_end) continue;
            uint64_t thr = prob_threshold(R->p);
            for (uint64_t j = R->dst_begin; j < R->dst_end; j++) {
                if (pG > 1 && orc_owner(j, pG, pS) != pg) continue;
                if (prob_edge(key0, key1, r, thr, s, j)) { if (n < cap) out[n] = (uint32_t)j; n++; }
            }
        } else {
            for (uint64_t j = R->dst_begin; j < R->dst_end; j++) {
                if (pG > 1 && orc_owner(j, pG, pS) != pg) continue;
                for (uint32_t k = 0; k < R->k; k++)
                    if (indeg_source(key0, key1, r, R, j, k) == s) { if (n < cap) out[n] = (uint32_t)j; n++; }
            }
        }
    }
    if (n <= cap) qsort(out, n, sizeof(uint32_t), cmp_u32v);
    return n;
}

/* Sampled column: the sources (with multiplicity, sorted) of all edges into target j. */
EXPORT uint64_t orc_col(const orc_rule *rules, uint32_t n_rules, uint64_t seed, uint32_t j,
                        uint32_t *out, uint64_t cap)
{
    uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    uint64_t n = 0;
    for (uint32_t r = 0; r < n_rules; r++) {
        const orc_rule *R = &rules[r];
        if (j < R->dst_begin || j >= R->dst_end) continue;
        if (R->kind == ORC_FIXED_PROB) {
            uint64_t thr = prob_threshold(R->p);
            for (uint64_t s = R->src_begin; s < R->src_end; s++)
                if (prob_edge(key0, key1, r, thr, s, j)) { if (n < cap) out[n] = (uint32_t)s; n++; }
        } else {
            for (uint32_t k = 0; k < R->k; k++) {
                uint64_t s = indeg_source(key0, key1, r, R, j, k);
                if (n < cap) out[n] = (uint32_t)s;
                n++;
            }
        }
    }
    if (n <= cap) qsort(out, n, sizeof(uint32_t), cmp_u32v);
    return n;
}

static real init_uniform(const orc_net *N, uint32_t j, uint32_t field, double lo, double hi)
{
    /* u = (x >> 8) 2^-24 exactly; value = lo + u (hi - lo)  (reading R15) */
    uint32_t x = philox_word(j >> 2, field, 0, TAG_INIT, N->key0, N->key1, j & 3);
    real u = (real)(x >> 8) * (real)(1.0 / 16777216.0);
    real a = (real)lo, b = (real)hi;
    real span = b - a;
    real prod = u * span;
    return a + prod;
}

EXPORT void orc_free(orc_net *N);

EXPORT orc_net *orc_create(uint32_t model, uint32_t n, uint32_t n_exc,
                           const orc_rule *rules, uint32_t n_rules,
                           double dt_ms, uint32_t delay, uint64_t seed, double activity,
                           const double *params, uint32_t n_params,
                           uint32_t pg, uint32_t pG, uint32_t pS)
{
    if (n == 0 || delay == 0 || n_params > 32 || (pG > 1 && (pS == 0 || pg >= pG))) return NULL;
    orc_net *N = xcalloc(1, sizeof *N);
    N->model = model; N->n = n; N->n_exc = n_exc; N->delay = delay;
    {   /* the ring holds the longest delay of any synapse (reading R19): max rule delay + 1,
         * the network delay + 1 when there are no synapses */
        uint32_t dmax = 0;
        for (uint32_t r = 0; r < n_rules; r++)
            if (rules[r].src_begin < rules[r].src_end && rules[r].dst_begin < rules[r].dst_end) {
                uint32_t hi = rule_dmax(&rules[r], delay);
                if (hi > dmax) dmax = hi;
            }
        N->D = (dmax ? dmax : delay) + 1;
    }
    N->key0 = (uint32_t)seed; N->key1 = (uint32_t)(seed >> 32);
    N->dt = dt_ms; N->activity = activity;
    for (uint32_t i = 0; i < n_params; i++) N->prm[i] = params[i];
    N->pg = pg; N->pG = pG ? pG : 1; N->pS = pS ? pS : 1;
    N->n_rules = n_rules;
    N->rules = xcalloc(n_rules, sizeof(orc_rule));
    memcpy(N->rules, rules, n_rules * sizeof(orc_rule));
    for (uint32_t r = 0; r < n_rules; r++)
        if (rules[r].src_begin > rules[r].src_end || rules[r].src_end > n ||
            rules[r].dst_begin > rules[r].dst_end || rules[r].dst_end > n ||
            rules[r].p < 0 || rules[r].p > 1) { orc_free(N); return NULL; }

    /* ---- build (§III-B) ---- */
    N->row_ptr = xcalloc((size_t)n + 1, sizeof(uint64_t));
    enumerate_edges(N, 0, NULL);
    for (uint32_t s = 0; s < n; s++) N->row_ptr[s + 1] += N->row_ptr[s];
    N->nnz = N->row_ptr[n];
    N->tgt = xcalloc(N->nnz, sizeof(uint32_t));
    N->plastic = xcalloc(N->nnz, 1);
    uint64_t *cursor = xcalloc(n, sizeof(uint64_t));
    for (uint32_t s = 0; s < n; s++) cursor[s] = N->row_ptr[s];
    enumerate_edges(N, 1, cursor);
    free(cursor);
    /* rows sorted ascending */
    for (uint32_t s = 0; s < n; s++) {
        uint64_t b = N->row_ptr[s], e = N->row_ptr[s + 1];
        int sorted = 1;
        for (uint64_t q = b + 1; q < e; q++) if (N->tgt[q - 1] > N->tgt[q]) { sorted = 0; break; }
        if (sorted) continue;
        tgt_pl *tmp = malloc((e - b) * sizeof(tgt_pl));
        for (uint64_t q = b; q < e; q++) { tmp[q - b].t = N->tgt[q]; tmp[q - b].pl = N->plastic[q]; }
        qsort(tmp, e - b, sizeof(tgt_pl), cmp_tp);
        for (uint64_t q = b; q < e; q++) { N->tgt[q] = tmp[q - b].t; N->plastic[q] = (uint8_t)tmp[q - b].pl; }
        free(tmp);
    }
    /* per-edge delays: the rule of (s, j) is unique (rules of one source have disjoint
     * destination ranges) */
    N->dly = xcalloc(N->nnz, sizeof(uint16_t));
    for (uint32_t s = 0; s < n; s++)
        for (uint64_t e = N->row_ptr[s]; e < N->row_ptr[s + 1]; e++) {
            uint32_t j = N->tgt[e];
            N->dly[e] = (uint16_t)delay;
            for (uint32_t r = 0; r < n_rules; r++) {
                const orc_rule *R = &N->rules[r];
                if (s >= R->src_begin && s < R->src_end && j >= R->dst_begin && j < R->dst_end) {
                    N->dly[e] = (uint16_t)edge_delay(N->key0, N->key1, R, r, delay, s, j);
                    break;
                }
            }
        }

    /* ---- derived scalars: computed in double from the inputs, rounded once ---- */
    const double *P = N->prm;
    if (model == ORC_VOGELS) {
        N->h = (real)(dt_ms / P[0]); N->EL = (real)P[1]; N->Vt = (real)P[2]; N->Vr = (real)P[3];
        N->R = (uint32_t)llround(P[4] / dt_ms); N->Ee = (real)P[5]; N->Ei = (real)P[6];
        N->ke = (real)(dt_ms / P[7]); N->ki = (real)(dt_ms / P[8]);
        N->dge = (real)P[9]; N->dgi = (real)P[10];
    } else if (model == ORC_BRUNEL || model == ORC_BRUNEL_PLUS) {
        N->h = (real)(dt_ms / P[0]); N->EL = (real)P[1]; N->theta = (real)P[2]; N->Vr = (real)P[3];
        N->R = (uint32_t)llround(P[4] / dt_ms);
        N->JE = (real)P[5]; N->JI = (real)(-P[6] * P[5]);
        N->ptab_len = orc_poisson_table(P[7], N->ptab, 256);
        if (N->ptab_len == 0) { orc_free(N); return NULL; }
        if (model == ORC_BRUNEL_PLUS) {
            N->Ap = (real)P[12]; N->Am = (real)P[13]; N->wmax = (real)P[14];
        }
    } else if (model == ORC_SYNTH) {
        N->thr_fire = prob_threshold(activity);
    } else { orc_free(N); return NULL; }

    /* ---- state (SoA) ---- */
    N->v = xcalloc(n, sizeof(real)); N->ge = xcalloc(n, sizeof(real)); N->gi = xcalloc(n, sizeof(real));
    N->ts = xcalloc(n, sizeof(int64_t));
    for (uint32_t j = 0; j < n; j++) N->ts[j] = -1;
    N->cx = xcalloc(n, sizeof(real)); N->cy = xcalloc(n, sizeof(real));
    N->pp = xcalloc(ORC_TRACE_LEN, sizeof(real)); N->pm = xcalloc(ORC_TRACE_LEN, sizeof(real));
    if (model == ORC_BRUNEL_PLUS)
        for (uint32_t k = 0; k < ORC_TRACE_LEN; k++) {
            N->pp[k] = (real)exp(-(double)k * dt_ms / P[10]);
            N->pm[k] = (real)exp(-(double)k * dt_ms / P[11]);
        }
    N->ref = xcalloc(n, sizeof(uint32_t)); N->acc = xcalloc(n, sizeof(uint32_t));
    N->ring = xcalloc((size_t)N->D * n, sizeof(uint32_t));
    N->pring = xcalloc((size_t)N->D * n, sizeof(int64_t));
    for (uint32_t j = 0; j < n; j++) {
        if (model == ORC_VOGELS) {
            N->v[j] = init_uniform(N, j, 0, P[11], P[12]);
            N->ge[j] = init_uniform(N, j, 1, P[13], P[14]);
            N->gi[j] = init_uniform(N, j, 2, P[15], P[16]);
        } else if (model == ORC_BRUNEL || model == ORC_BRUNEL_PLUS) {
            N->v[j] = init_uniform(N, j, 0, P[8], P[9]);
        }
    }
    if (model == ORC_BRUNEL_PLUS) {
        N->w = xcalloc(N->nnz, sizeof(real));
        uint64_t np = 0;
        for (uint64_t e = 0; e < N->nnz; e++) if (N->plastic[e]) { N->w[e] = (real)P[15]; np++; }
        /* CSC index over plastic edges: in_ptr[i]..in_ptr[i+1] lists edges into i */
        N->in_ptr = xcalloc((size_t)n + 1, sizeof(uint64_t));
        N->edge_src = xcalloc(N->nnz, sizeof(uint32_t));
        for (uint32_t s = 0; s < n; s++)
            for (uint64_t e = N->row_ptr[s]; e < N->row_ptr[s + 1]; e++) {
                N->edge_src[e] = s;
                if (N->plastic[e]) N->in_ptr[N->tgt[e] + 1]++;
            }
        for (uint32_t i = 0; i < n; i++) N->in_ptr[i + 1] += N->in_ptr[i];
        N->in_edge = xcalloc(np, sizeof(uint64_t));
        uint64_t *cur = xcalloc(n, sizeof(uint64_t));
        for (uint32_t i = 0; i < n; i++) cur[i] = N->in_ptr[i];
        for (uint64_t e = 0; e < N->nnz; e++) if (N->plastic[e]) N->in_edge[cur[N->tgt[e]]++] = e;
        free(cur);
    }
    N->force_t = -1;
    N->force_bits = xcalloc(n, 1);
    N->off_cap = 1024;
    N->sp_off = xcalloc(N->off_cap + 1, sizeof(uint64_t));
    N->delivered = xcalloc(N->off_cap, sizeof(uint64_t));
    N->sp_cap = 1024;
    N->sp = xcalloc(N->sp_cap, sizeof(uint32_t));
    return N;
}

EXPORT void orc_free(orc_net *N)
{
    if (!N) return;
    free(N->rules); free(N->row_ptr); free(N->tgt); free(N->plastic); free(N->w); free(N->dly);
    free(N->in_ptr); free(N->in_edge); free(N->edge_src);
    free(N->v); free(N->ge); free(N->gi); free(N->ts); free(N->cx); free(N->cy); free(N->pp); free(N->pm);
    free(N->ref); free(N->acc);
    free(N->ring); free(N->pring); free(N->sp); free(N->sp_off); free(N->delivered); free(N->force_bits);
    free(N);
}

/* Receptor packing (reading R10): an excitatory source adds 1 to the low 16 bits,
 * an inhibitory source adds 1 to the high 16 bits.  A single-population model
 * (n_exc == n) has only the low word, which then spans all 32 bits. */
static uint32_t q_of(const orc_net *N, uint32_t s) { return s < N->n_exc ? 1u : 65536u; }

static void record_spike(orc_net *N, uint32_t j)
{
    if (N->sp_len == N->sp_cap) { N->sp_cap *= 2; N->sp = realloc(N->sp, N->sp_cap * sizeof(uint32_t)); }
    N->sp[N->sp_len++] = j;
}

/* One neuron update, P:161 onUpdate; model readings R3-R5, R12. Returns
 * whether the threshold was crossed. */
static int update_neuron(orc_net *N, uint32_t j, uint64_t t, uint32_t c, int64_t pin, int forced, int force_val)
{
    /* forced: 0 none, 1 replace the threshold decision by force_val, 2 OR force_val into it */
    int spiked = 0;
    switch (N->model) {
    case ORC_SYNTH: {
        N->acc[j] = N->acc[j] + c;
        uint32_t x = philox_word(j >> 2, (uint32_t)t, 0, TAG_FIRE, N->key0, N->key1, j & 3);
        spiked = (uint64_t)x < N->thr_fire;
        if (forced == 1) spiked = force_val; else if (forced == 2) spiked = spiked || force_val;
        break;
    }
    case ORC_VOGELS: {
        uint32_t ne = c & 0xFFFFu, ni = c >> 16;
        real ge = N->ge[j], gi = N->gi[j], v = N->v[j];
        ge = ge + N->dge * (real)ne;
        gi = gi + N->dgi * (real)ni;
        if (N->ref[j] > 0) {
            N->ref[j] -= 1;
            v = N->Vr;
            spiked = 0;
        } else {
            real a = N->EL - v;
            real b = ge * (N->Ee - v);
            real cc = gi * (N->Ei - v);
            real sum = (a + b) + cc;
            v = v + N->h * sum;
            spiked = v >= N->Vt;
        }
        if (forced == 1) spiked = force_val; else if (forced == 2) spiked = spiked || force_val;
        if (spiked) { v = N->Vr; N->ref[j] = N->R; }
        ge = ge - N->ke * ge;
        gi = gi - N->ki * gi;
        N->v[j] = v; N->ge[j] = ge; N->gi[j] = gi;
        break;
    }
    case ORC_BRUNEL:
    case ORC_BRUNEL_PLUS: {
        real v = N->v[j];
        if (N->ref[j] > 0) {
            N->ref[j] -= 1;
            v = N->Vr;            /* input and drive discarded while refractory (R5) */
            spiked = 0;
        } else {
            uint32_t x = philox_word(j >> 2, (uint32_t)t, 0, TAG_EXT, N->key0, N->key1, j & 3);
            uint32_t next = 0;
            while ((uint64_t)x >= N->ptab[next]) next++;       /* min{k : x < T_k} */
            uint32_t ne = c & 0xFFFFu, ni = c >> 16;
            v = v + N->h * (N->EL - v);
            v = v + N->JE * (real)(ne + next);
            v = v + N->JI * (real)ni;
            if (N->model == ORC_BRUNEL_PLUS) v = v + (real)pin * (real)(1.0 / 4294967296.0);
            spiked = v >= N->theta;
        }
        if (forced == 1) spiked = force_val; else if (forced == 2) spiked = spiked || force_val;
        if (spiked) { v = N->Vr; N->ref[j] = N->R; }
        N->v[j] = v;
        break;
    }
    }
    return spiked;
}

/* Event-driven trace evaluation (reading R13): X_j(t) = cx_j P+[t - ts_j] for t > ts_j
 * (one rounded product; P+[k] = exp(-k dt/tau+) computed in double, rounded once; 0 for
 * k >= ORC_TRACE_LEN, where it is below 2^-24 of any trace); 0 before the first spike.
 * The value excludes a spike at t itself (it is the sum over spikes t' < t). */
static real trace_at(const orc_net *N, const real *c, const real *tab, uint32_t j, uint64_t t)
{
    if (N->ts[j] < 0) return (real)0;
    uint64_t k = t - (uint64_t)N->ts[j];
    if (k >= ORC_TRACE_LEN) return (real)0;
    return c[j] * tab[k];
}

/* Fixed-point quantisation of a plastic weight (reading R10): rint(w 2^32). */
static int64_t wq(real w) { return (int64_t)llrint((double)w * 4294967296.0); }

EXPORT int orc_step(orc_net *N, uint64_t n_steps)
{
    const uint32_t n = N->n, D = N->D;
    uint8_t *spk = xcalloc(n, 1);
    for (uint64_t it = 0; it < n_steps; it++) {
        uint64_t t = N->t;
        if (t + 1 >= N->off_cap) {
            N->off_cap *= 2;
            N->sp_off = realloc(N->sp_off, (N->off_cap + 1) * sizeof(uint64_t));
            N->delivered = realloc(N->delivered, N->off_cap * sizeof(uint64_t));
        }
        N->sp_off[t] = N->sp_len;
        uint32_t *slot = N->ring + (size_t)(t % D) * n;
        int64_t *pslot = N->pring + (size_t)(t % D) * n;
        int forced = (N->force_t == (int64_t)t) ? N->force_mode : 0;
        /* (1) update every neuron, ascending ID */
        for (uint32_t j = 0; j < n; j++) {
            uint32_t c = slot[j]; slot[j] = 0;
            int64_t pin = pslot[j]; pslot[j] = 0;
            spk[j] = (uint8_t)update_neuron(N, j, t, c, pin, forced, forced ? N->force_bits[j] : 0);
        }
        if (forced) N->force_t = -1;
        /* (2) S_t, ascending (R11) */
        for (uint32_t j = 0; j < n; j++) if (spk[j]) record_spike(N, j);
        uint64_t s_begin = N->sp_off[t], s_end = N->sp_len;
        /* (3) eager STDP, Brunel+ (R13): (i) potentiation at post spikes, (ii) depression at pre spikes */
        if (N->model == ORC_BRUNEL_PLUS) {
            for (uint64_t q = s_begin; q < s_end; q++) {
                uint32_t i = N->sp[q];
                for (uint64_t a = N->in_ptr[i]; a < N->in_ptr[i + 1]; a++) {
                    uint64_t e = N->in_edge[a];
                    real inc = N->Ap * trace_at(N, N->cx, N->pp, N->edge_src[e], t);
                    real w = N->w[e] + inc;
                    N->w[e] = w < N->wmax ? w : N->wmax;
                }
            }
            for (uint64_t q = s_begin; q < s_end; q++) {
                uint32_t j = N->sp[q];
                for (uint64_t e = N->row_ptr[j]; e < N->row_ptr[j + 1]; e++) {
                    if (!N->plastic[e]) continue;
                    real dec = N->Am * trace_at(N, N->cy, N->pm, N->tgt[e], t);
                    real w = N->w[e] - dec;
                    N->w[e] = w > (real)0 ? w : (real)0;
                }
            }
        }
        /* (4) deliver S_t row by row into I[(t + d_e) mod D], d_e the synapse's delay
         * (per-synapse delays P:485, reading R19) */
        uint64_t events = 0;
        for (uint64_t q = s_begin; q < s_end; q++) {
            uint32_t s = N->sp[q];
            uint32_t qs = q_of(N, s);
            for (uint64_t e = N->row_ptr[s]; e < N->row_ptr[s + 1]; e++) {
                size_t slot = (size_t)((t + N->dly[e]) % D) * n;
                if (N->model == ORC_BRUNEL_PLUS && N->plastic[e]) N->pring[slot + N->tgt[e]] += wq(N->w[e]);
                else N->ring[slot + N->tgt[e]] += qs;
                events++;
            }
        }
        N->delivered[t] = events;
        /* traces: a spike at t restarts both closed forms from their value at t plus one (R13) */
        if (N->model == ORC_BRUNEL_PLUS) {
            for (uint32_t j = 0; j < n; j++) {
                if (!spk[j]) continue;
                real xs = trace_at(N, N->cx, N->pp, j, t) + (real)1;
                real ys = trace_at(N, N->cy, N->pm, j, t) + (real)1;
                N->cx[j] = xs; N->cy[j] = ys; N->ts[j] = (int64_t)t;
            }
        }
        N->t = t + 1;
        N->sp_off[t + 1] = N->sp_len;
    }
    free(spk);
    return 0;
}

/* ---------------------------- accessors ---------------------------------- */
EXPORT uint64_t orc_nnz(const orc_net *N) { return N->nnz; }
EXPORT uint64_t orc_time(const orc_net *N) { return N->t; }
EXPORT void orc_row_ptr(const orc_net *N, uint64_t *out) { memcpy(out, N->row_ptr, ((size_t)N->n + 1) * sizeof(uint64_t)); }
EXPORT void orc_targets(const orc_net *N, uint32_t *out) { memcpy(out, N->tgt, N->nnz * sizeof(uint32_t)); }
EXPORT void orc_plastic_flags(const orc_net *N, uint8_t *out) { memcpy(out, N->plastic, N->nnz); }
EXPORT void orc_delays(const orc_net *N, uint16_t *out) { memcpy(out, N->dly, N->nnz * sizeof(uint16_t)); }
EXPORT uint32_t orc_ring_slots(const orc_net *N) { return N->D; }
EXPORT int orc_weights(const orc_net *N, real *out) { if (!N->w) return -1; memcpy(out, N->w, N->nnz * sizeof(real)); return 0; }
EXPORT uint64_t orc_spike_count_total(const orc_net *N) { return N->sp_len; }
EXPORT void orc_spike_offsets(const orc_net *N, uint64_t *out) { memcpy(out, N->sp_off, (N->t + 1) * sizeof(uint64_t)); }
EXPORT void orc_spikes_all(const orc_net *N, uint32_t *out) { memcpy(out, N->sp, N->sp_len * sizeof(uint32_t)); }
EXPORT void orc_delivered(const orc_net *N, uint64_t *out) { memcpy(out, N->delivered, N->t * sizeof(uint64_t)); }
EXPORT uint32_t orc_sizeof_real(void) { return (uint32_t)sizeof(real); }

/* field: 0 v, 1 ge, 2 gi, 3 ref (u32), 4 acc (u32), 5 x trace, 6 y trace */
EXPORT int orc_get_state(const orc_net *N, uint32_t field, void *out)
{
    size_t n = N->n;
    switch (field) {
    case 0: memcpy(out, N->v, n * sizeof(real)); return 0;
    case 1: memcpy(out, N->ge, n * sizeof(real)); return 0;
    case 2: memcpy(out, N->gi, n * sizeof(real)); return 0;
    case 3: memcpy(out, N->ref, n * sizeof(uint32_t)); return 0;
    case 4: memcpy(out, N->acc, n * sizeof(uint32_t)); return 0;
    case 5: for (size_t j = 0; j < n; j++) ((real *)out)[j] = trace_at(N, N->cx, N->pp, (uint32_t)j, N->t); return 0;
    case 6: for (size_t j = 0; j < n; j++) ((real *)out)[j] = trace_at(N, N->cy, N->pm, (uint32_t)j, N->t); return 0;
    }
    return -1;
}

EXPORT int orc_set_state(orc_net *N, uint32_t field, const void *in)
{
    size_t n = N->n;
    switch (field) {
    case 0: memcpy(N->v, in, n * sizeof(real)); return 0;
    case 1: memcpy(N->ge, in, n * sizeof(real)); return 0;
    case 2: memcpy(N->gi, in, n * sizeof(real)); return 0;
    case 3: memcpy(N->ref, in, n * sizeof(uint32_t)); return 0;
    case 4: memcpy(N->acc, in, n * sizeof(uint32_t)); return 0;
    }
    return -1;
}

/* Input slot that the update of step (t_now + rel) will read, rel in [0, D). */
EXPORT int orc_get_input(const orc_net *N, uint32_t rel, uint32_t *counts, int64_t *plastic_fx)
{
    if (rel >= N->D) return -1;
    size_t s = (size_t)((N->t + rel) % N->D) * N->n;
    if (counts) memcpy(counts, N->ring + s, N->n * sizeof(uint32_t));
    if (plastic_fx) memcpy(plastic_fx, N->pring + s, N->n * sizeof(int64_t));
    return 0;
}

/* Overwrite the input slot that the update of step (t_now + rel) will read. */
EXPORT int orc_set_input(orc_net *N, uint32_t rel, const uint32_t *counts)
{
    if (rel >= N->D) return -1;
    memcpy(N->ring + (size_t)((N->t + rel) % N->D) * N->n, counts, N->n * sizeof(uint32_t));
    return 0;
}

/* Jump the step counter (the oracle's state is then treated as the state at step t);
 * used to replay one step of a GPU run at full size. */
EXPORT void orc_set_time(orc_net *N, uint64_t t) { N->t = t; if (N->t + 1 >= N->off_cap) { N->off_cap = N->t + 1024; N->sp_off = realloc(N->sp_off, (N->off_cap + 1) * sizeof(uint64_t)); N->delivered = realloc(N->delivered, N->off_cap * sizeof(uint64_t)); } for (uint64_t q = 0; q <= t; q++) N->sp_off[q] = N->sp_len; for (uint64_t q = 0; q < t; q++) N->delivered[q] = 0; }

/* Teacher forcing of the NEXT step (t_now): mode 1 replaces its spike set by ids,
 * mode 2 adds ids to the naturally emitted set.  A forced spike resets the neuron
 * like a natural one. */
EXPORT int orc_force_next(orc_net *N, const uint32_t *ids, uint64_t n, int mode)
{
    if (mode != 1 && mode != 2) return -1;
    N->force_mode = mode;
    memset(N->force_bits, 0, N->n);
    for (uint64_t q = 0; q < n; q++) { if (ids[q] >= N->n) return -1; N->force_bits[ids[q]] = 1; }
    N->force_t = (int64_t)N->t;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Synth checkers for sizes the oracle cannot simulate (reading R17; SURVEY     */
/* C17).  Both are the plain definitions: the synth spike set of step t is the  */
/* Bernoulli draw of reading R12 for every neuron, and a synth accumulator is   */
/* the number of spikes its in-synapses carried (P:200 delivery, reading R10).  */
/* ------------------------------------------------------------------------- */

/* Synth spikes of step t (reading R12): j fires iff Philox(j>>2, t, 0, TAG_FIRE)[j&3] <
 * floor(a 2^32), ascending.  Returns the count (writes at most cap ids). */
EXPORT uint64_t orc_synth_fired(uint32_t n, double activity, uint64_t seed, uint64_t t,
                                uint32_t *out, uint64_t cap)
{
    uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    uint64_t thr = prob_threshold(activity), c = 0;
    for (uint32_t j = 0; j < n; j++) {
        uint32_t x = philox_word(j >> 2, (uint32_t)t, 0, TAG_FIRE, key0, key1, j & 3);
        if ((uint64_t)x < thr) { if (c < cap) out[c] = j; c++; }
    }
    return c;
}

/* Synth accumulator of target j after T steps (no teacher forcing): acc_j = sum over
 * in-synapses (s -> j), with multiplicity, of the number of steps t with t + d_sj < T at
 * which s fired (a spike of step t reaches the update of step t + d_sj; d_sj the
 * synapse's delay, the network delay d for rules without a delay range). */
static uint64_t spikes_before(uint32_t key0, uint32_t key1, uint64_t thr, uint32_t s, uint64_t T, uint32_t d)
{
    uint64_t c = 0;
    for (uint64_t t = 0; t + d < T; t++)
        c += (uint64_t)philox_word(s >> 2, (uint32_t)t, 0, TAG_FIRE, key0, key1, s & 3) < thr;
    return c;
}
EXPORT uint64_t orc_synth_acc(const orc_rule *rules, uint32_t n_rules, uint64_t seed, double activity,
                              uint32_t j, uint64_t T, uint32_t d)
{
    uint32_t key0 = (uint32_t)seed, key1 = (uint32_t)(seed >> 32);
    uint64_t thr = prob_threshold(activity), acc = 0;
    for (uint32_t r = 0; r < n_rules; r++) {
        const orc_rule *R = &rules[r];
        if (j < R->dst_begin || j >= R->dst_end) continue;
        if (R->kind == ORC_FIXED_PROB) {
            uint64_t pthr = prob_threshold(R->p);
            for (uint64_t s = R->src_begin; s < R->src_end; s++)
                if (prob_edge(key0, key1, r, pthr, s, j))
                    acc += spikes_before(key0, key1, thr, (uint32_t)s, T, edge_delay(key0, key1, R, r, d, s, j));
        } else {
            for (uint32_t k = 0; k < R->k; k++) {
                uint64_t s = indeg_source(key0, key1, r, R, j, k);
                acc += spikes_before(key0, key1, thr, (uint32_t)s, T, edge_delay(key0, key1, R, r, d, s, j));
            }
        }
    }
    return acc;
}
