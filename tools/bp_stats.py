import sys; sys.path.insert(0,'.')
import bench
from paper_2102_04681_b200 import spice as S
cfg,_=bench.workload('brunelplus50k',1)
with S.Network(cfg, record_steps=64) as net:
    net.step(500); net.sync()
    d0=net.stats()["delivered"]
    sp=[len(x) for x in net.read_spikes(436,500)]
    net.step(1000); net.sync()
    d1=net.stats()["delivered"]
    info=net.info()
    print("delivered/step", (d1-d0)/1000, "spikes/step", sum(sp)/len(sp), info)
