import cProfile, pstats, time, sys
sys.path.insert(0, '/root/repo')
from paper_2601_06765_b200.groebner import f4_groebner
from paper_2601_06765_b200.systems import gen_cyclic
ring, polys = gen_cyclic(8, 32003)
t0 = time.time(); f4_groebner(polys, ring); print("warm run", time.time() - t0)
pr = cProfile.Profile(); pr.enable()
t0 = time.time(); f4_groebner(polys, ring); t1 = time.time()
pr.disable()
print("second run", t1 - t0)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
