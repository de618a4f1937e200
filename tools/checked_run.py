"""Bounds-checked run of every step-kernel family (diagnostics; compute-sanitizer is closed on
the GPU pool): builds the library with -DSPICE_CHECKS=1 (device-side index checks that trap:
window and entry indices within the stored entries, every entry within the tile's counters,
descriptor reservations within their lists, spike-list positions within their regions) and
runs tools/sanitize.py's cases against the oracle with it.

    python tools/checked_run.py [case ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if __name__ == "__main__":
    import importlib.util
    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2102_04681_b200", "build.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    lib = B.build(out="/tmp/libspice_checks.so", defines=["SPICE_CHECKS=1"])
    env = dict(os.environ, SPICE_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py")] + sys.argv[1:], env=env)
    rc = r.returncode
    if not sys.argv[1:]:    # and the full-size workloads in the bench's launch configuration
        for w in ("synth", "brunel100k", "brunelplus50k"):
            b = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", w, "--steps", "300",
                                "--warmup", "5", "--profile-steps", "2", "--e2e-steps", "128", "--no-cpu-baseline"],
                               env=env, capture_output=True, text=True)
            line = (b.stdout.strip().splitlines() or ["(none)"])[-1]
            print(f"bench {w} with bounds checks: rc {b.returncode}, "
                  f"parity {line.split('\"parity\": ')[1][:30] if '\"parity\": ' in line else '?'}", flush=True)
            rc = rc or b.returncode
    sys.exit(rc)
