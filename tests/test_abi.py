"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the
header declares, and its host-only partition helpers reproduce the paper's worked
examples (Fig. 4, Listing 1; tests/golden)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spice.h")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def S():
    from paper_2102_04681_b200 import build as B
    B.build()
    from paper_2102_04681_b200 import spice
    spice.lib()
    return spice


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"SPICE_API[^;(]*?\b(spice_\w+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("spice_create_network", "spice_step", "spice_read_spikes", "spice_free"):
        assert s in syms


def test_library_exports_every_declared_symbol(S):
    out = subprocess.run(["nm", "-D", "--defined-only", S.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (spice_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    L = S.lib()
    for s in declared_symbols():
        assert hasattr(L, s)


def test_library_is_sm100a(S):
    out = subprocess.run(["cuobjdump", "--list-elf", S.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_partition_helpers_match_golden(S):
    for line in open(os.path.join(GOLD, "partition.txt")):
        if line.startswith("#") or not line.strip():
            continue
        head, ids = line.split(":")
        N, G, Sw, g = map(int, head.split())
        want = list(map(int, ids.split()))
        assert [j for j in range(N) if S.partition_owner(j, G, Sw) == g] == want
        assert S.partition_owned_count(N, g, G, Sw) == len(want)
        assert [S.partition_local_to_global(i, g, G, Sw) for i in range(len(want))] == want
    for line in open(os.path.join(GOLD, "listing1.txt")):
        if line.startswith("#") or not line.strip():
            continue
        Sw, G, g, i, j = map(int, line.split())
        assert S.partition_local_to_global(i, g, G, Sw) == j


@pytest.mark.parametrize("N,G", [(4000, 1), (100_000, 8), (3_922_323, 8), (1_386_750, 2), (1001, 3)])
def test_partition_counts_cover_and_balance(S, N, G):
    Sw = S.default_slice_width(N, G)
    assert Sw % 32 == 0
    counts = [S.partition_owned_count(N, g, G, Sw) for g in range(G)]
    assert sum(counts) == N
    assert max(counts) - min(counts) <= Sw
    if N >= 100 * 32 * G:
        assert N / (Sw * G) >= 100                             # "hundreds" of slices


def test_create_without_gpu_fails_loudly(S):
    """No CPU fallback: on a machine without a usable GPU, create raises."""
    import workloads as W
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(S.SpiceError):
        S.Network(W.vogels(4000))


def test_config_validation_errors(S):
    """EINVAL paths are checked before any device work (include/spice.h conventions)."""
    import dataclasses
    import workloads as W
    bad = [dataclasses.replace(W.vogels(100), n=0),
           dataclasses.replace(W.vogels(100), delay=0),
           dataclasses.replace(W.vogels(100), rules=(W.Rule((0, 100), (0, 101), W.FIXED_PROB, 0.1),)),
           dataclasses.replace(W.vogels(100), rules=(W.Rule((0, 100), (0, 100), W.FIXED_PROB, 1.5),)),
           dataclasses.replace(W.vogels(100), params=(1.0, 2.0))]
    for cfg in bad:
        with pytest.raises(S.SpiceError) as e:
            S.Network(cfg)
        assert e.value.status == S.EINVAL
