"""Small GPU run against the oracle (debug helper): python tools/small_run.py [vogels|synth|brunel]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2102_04681_b200 import spice as S  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "synth"
cfg = {"vogels": W.vogels(4000), "synth": W.synth(20000, 31, 0.005, seed=3),
       "brunel": W.brunel(3000, 0.1, seed=5, delay=15)}[which]
T = 40
o = O.OracleNet(cfg)
o.step(T)
with S.Network(cfg, record_steps=T) as net:
    net.step(T)
    got = net.read_spikes(0, T)
want = o.spikes()
bad = [t for t in range(T) if not np.array_equal(got[t], want[t])]
print(which, "mismatching steps:", bad[:10], "of", T)
