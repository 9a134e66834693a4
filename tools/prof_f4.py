"""cProfile of the F4 loop of a named system (diagnostic): where the host time goes.
usage: python tools/prof_f4.py cyclic 8 | katsura 11"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2601_06765_b200.groebner import GroebnerState, f4_step, update_pairs
    from paper_2601_06765_b200.polynomials import poly_monic
    from paper_2601_06765_b200.systems import gen_cyclic, gen_katsura

    fam, n = sys.argv[1], int(sys.argv[2])
    gen = gen_cyclic if fam == "cyclic" else gen_katsura
    for rep in range(2):
        ring, polys = gen(n, 32003)
        st = GroebnerState(ring)
        for f in polys:
            update_pairs(st, poly_monic(f))
        pr = cProfile.Profile()
        t = time.perf_counter()
        if rep == 1:
            pr.enable()
        while st.n_pairs():
            f4_step(st)
        if rep == 1:
            pr.disable()
        print("f4 loop", time.perf_counter() - t, "s")
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
