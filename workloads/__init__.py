"""Seeded synthetic workload definitions shared by the oracle tests, the CUDA parity
tests, ``smoke()`` and ``bench.py``.

This module holds *inputs only*: network descriptors in the paper's
``{range1, range2, p}`` form (§III-B), the model constants
(frozen once here; the paper defers them to its citations, §IV — see
DESIGN.md "Readings" R7/R8), sizes, delays and seeds.  It contains none of the
method's arithmetic: no Philox, no thresholds, no integration, no delivery.  Both
``oracle/`` and ``paper_2102_04681_b200`` receive these numbers and derive
everything else independently.

Every random number the method draws comes from the counter-based Philox4x32-10
generator that each side implements on its own (R9), keyed by ``seed``.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple

# model ids (include/spice.h SPICE_MODEL_*; oracle/spice_oracle.c ORC_MODEL_*)
VOGELS, BRUNEL, BRUNEL_PLUS, SYNTH = 1, 2, 3, 4
MODEL_NAMES = {VOGELS: "vogels", BRUNEL: "brunel", BRUNEL_PLUS: "brunel+", SYNTH: "synth"}
# connectivity rule kinds
FIXED_PROB, FIXED_INDEGREE = 0, 1


@dataclass(frozen=True)
class Rule:
    """One descriptor entry ``{range1, range2, p}`` (§III-B), half-open
    global ID ranges.  ``kind=FIXED_INDEGREE`` (each target draws ``k`` sources) is the
    BASELINE synth rule ("fixed in-degree", BASELINE.json configs[3])."""
    src: Tuple[int, int]
    dst: Tuple[int, int]
    kind: int = FIXED_PROB
    p: float = 0.0
    k: int = 0
    plastic: bool = False
    # per-synapse delays in steps (reading R19): each synapse of the
    # rule draws a delay uniformly from [delay_min, delay_max]; 0 = the network delay
    delay_min: int = 0
    delay_max: int = 0


@dataclass(frozen=True)
class NetConfig:
    name: str
    model: int
    n: int                 # neuron count N
    n_exc: int             # [0, n_exc) excitatory, [n_exc, n) inhibitory
    rules: Tuple[Rule, ...]
    dt_ms: float = 0.1
    delay: int = 1         # uniform synaptic delay in steps
    seed: int = 1
    activity: float = 0.0  # synth per-step firing probability
    params: Tuple[float, ...] = field(default_factory=tuple)

    @property
    def expected_synapses(self) -> float:
        tot = 0.0
        for r in self.rules:
            ns, nd = r.src[1] - r.src[0], r.dst[1] - r.dst[0]
            tot += ns * nd * r.p if r.kind == FIXED_PROB else nd * r.k
        return tot


# ---------------------------------------------------------------------------
# Model constant vectors (order documented in include/spice.h).  † = not in PAPER.md.
# ---------------------------------------------------------------------------

def vogels_params(dg_e: float = 0.6, dg_i: float = 6.7) -> Tuple[float, ...]:
    """Vogels-Abbott COBA benchmark (Brette et al. 2007) constants †.
    [tau_m, E_L, V_t, V_r, t_ref, E_e, E_i, tau_e, tau_i, dg_e, dg_i,
     v_lo, v_hi, ge_lo, ge_hi, gi_lo, gi_hi]  (ms, mV, conductances in units of g_L).
    E_L = -49 mV (rest above threshold, as in the Brian CUBA/COBA benchmark scripts)
    so activity is self-sustained without a stimulus phase (reading R7;
    with E_L = -60 mV the network falls silent within 20 ms)."""
    return (20.0, -49.0, -50.0, -60.0, 5.0, 0.0, -80.0, 5.0, 10.0, dg_e, dg_i,
            -60.0, -50.0, 0.0, 8.0, 0.0, 40.0)


def brunel_params(j_e: float, lam: float, g: float = 5.0, t_ref: float = 2.0,
                  v_lo: float = 0.0, v_hi: float = 20.0) -> Tuple[float, ...]:
    """Brunel (2000) model A constants †.
    [tau_m, V_L, theta, V_r, t_ref, J_E, g, lambda_ext, v_lo, v_hi]."""
    return (20.0, 0.0, 20.0, 10.0, t_ref, j_e, g, lam, v_lo, v_hi)


def brunel_scaled_weights(n: int, eps: float = 0.1, eta: float = 2.0):
    """Weight scaling with network size ("scaling factor … detailed in
    [bautembach2020]"; reading R8): J_E = 0.1 mV * 1000 / C_E and the external
    Poisson count per step lambda = eta * theta * dt / (J_E * tau) so that the mean
    external drive per step (lambda * J_E = 0.2 mV) is size-invariant."""
    c_e = eps * 0.8 * n
    j_e = 0.1 * 1000.0 / c_e
    lam = eta * 20.0 * 0.1 / (j_e * 20.0)
    return round(j_e, 12), round(lam, 9)   # freeze decimal values (0.0125, 16.0, ...)


def stdp_params(j_e: float) -> Tuple[float, ...]:
    """Brunel+ STDP constants † (reading R13): [tau_plus, tau_minus, A_plus, A_minus,
    w_max, w0] in ms / mV."""
    a_plus = 0.01 * j_e
    return (20.0, 20.0, a_plus, 1.05 * a_plus, 2.0 * j_e, j_e)


# ---------------------------------------------------------------------------
# Named configurations (BASELINE.json configs)
# ---------------------------------------------------------------------------

def vogels(n: int = 4000, p: float = 0.02, seed: int = 1, delay: int = 1) -> NetConfig:
    ne = n * 4 // 5
    rules = (Rule((0, ne), (0, n), FIXED_PROB, p), Rule((ne, n), (0, n), FIXED_PROB, p))
    return NetConfig(f"vogels{n}", VOGELS, n, ne, rules, 0.1, delay, seed, 0.0, vogels_params())


def brunel(n: int = 100_000, p: float = 0.1, seed: int = 1, delay: int = 15) -> NetConfig:
    ne = n * 4 // 5
    j_e, lam = brunel_scaled_weights(n, p)
    rules = (Rule((0, ne), (0, n), FIXED_PROB, p), Rule((ne, n), (0, n), FIXED_PROB, p))
    return NetConfig(f"brunel{n}", BRUNEL, n, ne, rules, 0.1, delay, seed, 0.0,
                     brunel_params(j_e, lam))


def brunel_plus(n: int = 50_000, p: float = 0.1, seed: int = 1, delay: int = 15,
                stdp_on: bool = True) -> NetConfig:
    ne = n * 4 // 5
    j_e, lam = brunel_scaled_weights(n, p)
    sp = stdp_params(j_e)
    if not stdp_on:
        sp = sp[:2] + (0.0, 0.0) + sp[4:]
    rules = (Rule((0, ne), (0, ne), FIXED_PROB, p, plastic=True),
             Rule((0, ne), (ne, n), FIXED_PROB, p),
             Rule((ne, n), (0, n), FIXED_PROB, p))
    return NetConfig(f"brunelplus{n}", BRUNEL_PLUS, n, ne, rules, 0.1, delay, seed, 0.0,
                     brunel_params(j_e, lam) + sp)


def synth(n: int, k: int, activity: float = 0.005, seed: int = 1, delay: int = 1) -> NetConfig:
    """Synth: one intra-connected population, fixed in-degree k,
    Bernoulli firing with per-step probability ``activity``, unit weights, delay 1."""
    return NetConfig(f"synth{n}k{k}", SYNTH, n, n, (Rule((0, n), (0, n), FIXED_INDEGREE, k=k),),
                     0.1, delay, seed, activity, ())


SYNTH_DENSITY = 0.00156   # PAPER.md:389 Fig. 6 caption "density=0.156%"
SYNTH_ACTIVITY = 0.005    # PAPER.md:389 "activity=0.5%"


def synth_for_synapses(total_synapses: float, seed: int = 1) -> NetConfig:
    """Synth at fixed density 0.156 %: N = sqrt(S / density), K = round(density N)."""
    n = int(round((total_synapses / SYNTH_DENSITY) ** 0.5))
    k = int(round(SYNTH_DENSITY * n))
    return synth(n, k, SYNTH_ACTIVITY, seed)


# BASELINE.json configs
CONFIGS = {
    "vogels4000": lambda: vogels(4000),                 # configs[0]
    "brunel100k": lambda: brunel(100_000),               # configs[1]
    "brunelplus50k": lambda: brunel_plus(50_000),        # configs[2]
    "synth3b": lambda: synth(1_386_750, 2163),           # configs[3] per GPU (G=1 point)
    "synth24b": lambda: synth(3_922_323, 6119),          # configs[3] whole box, G=8
    "synth250m": lambda: synth_for_synapses(250e6),      # configs[4] low end
}


def synth_weak(g: int) -> NetConfig:
    """Weak-scaling point: 3e9 synapses per GPU at fixed density."""
    return synth_for_synapses(3.0e9 * g)
