import cProfile, pstats, sys, time
sys.path.insert(0, ".")
from paper_2601_06765_b200.groebner import F4Config, GroebnerState, f4_step, update_pairs
from paper_2601_06765_b200.polynomials import poly_monic
from paper_2601_06765_b200.systems import gen_random_quadratic
ring, polys = gen_random_quadratic(16, 32, density=1.0, seed=0, p=31)
st = GroebnerState(ring)
[update_pairs(st, poly_monic(f)) for f in polys]
cfg = F4Config(numeric="wiedemann")
for k in range(3):
    f4_step(st, cfg)
pr = cProfile.Profile(); pr.enable(); t = time.time(); f4_step(st, cfg); print("step3", time.time() - t); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
