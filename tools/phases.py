"""In-kernel phase timeline of the fused kernel (diagnostics; SPICE_PHASES=1).
Usage: python tools/phases.py [synth|brunel100k|vogels4000] [steps] [ctas_per_tile]"""
import os
import sys

os.environ["SPICE_PHASES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# the phase clocks are compiled out of the product library: build a variant with them
_EXTRA = [d for d in os.environ.get("SPICE_DEFINES", "").split(",") if d]
_VARIANT = "/tmp/libspice_phases%s.so" % ("_" + "_".join(_EXTRA) if _EXTRA else "")
if "SPICE_LIB" not in os.environ:
    import importlib.util  # noqa: E402
    _spec = importlib.util.spec_from_file_location(
        "_spice_build", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2102_04681_b200", "build.py"))
    _B = importlib.util.module_from_spec(_spec)
    _spec.loader.exec_module(_B)                   # (not via the package: it loads the library)
    _B.build(out=_VARIANT, defines=["SPICE_PHASES_BUILD=1"] + _EXTRA)
    os.environ["SPICE_LIB"] = _VARIANT
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2102_04681_b200 import spice as S  # noqa: E402

NAMES = {1: "counters zeroed", 2: "region prefix / rows issued", 3: "staged / s_off", 4: "warp0 delivered",
         5: "barrier / list published", 6: "cluster reduce / rows landed", 7: "update loop / desc issued", 8: "spike rows / publ. bar",
         10: "(pro) zeroed / rows", 11: "(pro) fired / reserved", 9: "descriptors written", 12: "end"}
which = sys.argv[1] if len(sys.argv) > 1 else "synth"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg, _ = bench.workload(which, 1)
mhz = float(os.environ.get("SM_MHZ", "1965"))
with S.Network(cfg, record_steps=64, ctas_per_tile=ctas) as net:
    net.step(256)
    net.sync()
    p0 = net.debug_phases().astype(np.float64)
    net.step(steps)
    net.sync()
    p = net.debug_phases().astype(np.float64) - p0
    gl = net.debug_phases()
launches = p[:, 13]
print(f"{which}: {p.shape[0]} CTAs, {int(launches[0])} fused launches each; SM clock assumed {mhz} MHz")
prev = np.zeros(p.shape[0])
for s, nm in NAMES.items():
    us = p[:, s] / launches / mhz
    print(f"  slot {s:2d} {nm:20s} mean {us.mean():7.2f} us  max {us.max():7.2f}  (+{(us - prev).mean():6.2f})")
    prev = us
st, en = gl[:, 14].astype(np.int64), gl[:, 15].astype(np.int64)
print(f"  last launch: CTA start spread {(st.max() - st.min()) / 1e3:.2f} us, end spread {(en.max() - en.min()) / 1e3:.2f} us, "
      f"first start -> last end {(en.max() - st.min()) / 1e3:.2f} us")
if os.environ.get("PHASES_DUMP"):
    np.savez(os.environ["PHASES_DUMP"], p=p, gl=gl.astype(np.int64), mhz=mhz)
    print("  per-CTA phase clocks saved to", os.environ["PHASES_DUMP"])
