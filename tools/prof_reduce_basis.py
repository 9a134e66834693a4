"""cProfile of reduce_basis_device on the Katsura-11 basis (diagnostic)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2601_06765_b200.groebner import GroebnerState, f4_step, reduce_basis_device, update_pairs
    from paper_2601_06765_b200.polynomials import poly_monic
    from paper_2601_06765_b200.systems import gen_katsura

    ring, polys = gen_katsura(int(sys.argv[1]) if len(sys.argv) > 1 else 11, 32003)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    while st.n_pairs():
        f4_step(st)
    t = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    gb = reduce_basis_device(st.basis, ring, st.soa())
    pr.disable()
    print("reduce_basis_device", time.perf_counter() - t, "s", len(gb))
    pstats.Stats(pr).sort_stats("cumtime").print_stats(18)


if __name__ == "__main__":
    main()
