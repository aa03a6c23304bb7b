import sys; sys.path.insert(0, ".")
import paper_2105_14088_b200 as rw
m = rw.fixtures.config_matrix("C4", "fixed")
prob = rw.Problem(m)
spec = rw.fixtures.ring_spec(1024, rw.fixtures.SIZE_FIXED)
order, cost, ev, rep = prob.anneal(spec, rw.SolverConfig(seed=0, budget=1e6, steps_per_temperature=8), chains=65536, schedule="calibrated")
print(cost, rep['proposals'])
