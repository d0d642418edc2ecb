import cProfile, pstats, sys, io
sys.path.insert(0, '/root/repo')
import torch, bench
import paper_2208_14228_b200 as bt
from paper_2208_14228_b200 import engine
cfg = bench.make_cfg(bt)
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
engine.run_steps(ts, 20)
def loop():
    for _ in range(300):
        engine.run_steps(ts, 20)
pr = cProfile.Profile()
pr.enable(); loop(); pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats('tottime').print_stats(25)
print(s.getvalue())
