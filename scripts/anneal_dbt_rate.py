import sys, time
sys.path.insert(0, ".")
import paper_2105_14088_b200 as rw
m = rw.fixtures.config_matrix("C3", "fixed")
prob = rw.Problem(m)
spec = rw.CollectiveSpec(rw.Algorithm.DoubleBinaryTree, 256, rw.fixtures.SIZE_FIXED)
prob.anneal(spec, rw.SolverConfig(seed=1, budget=1e6, steps_per_temperature=64), chains=1, max_proposals=20000)
t = time.perf_counter()
o, c, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=1024), chains=1, max_proposals=2000000)
dt = time.perf_counter() - t
print(f"{rep['proposals']/dt:.4e} proposals/s cost {c}")
