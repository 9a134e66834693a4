import sys, json, time, hashlib
sys.path.insert(0, '.')
import __graft_entry__ as G
G.smoke()
from paper_2601_06765_b200.systems import gen_cyclic, gen_katsura, format_system
from paper_2601_06765_b200.groebner import f4_groebner, GroebnerState, update_pairs, f4_step, reduce_basis
from paper_2601_06765_b200.polynomials import poly_monic
from paper_2601_06765_b200.symbolic import plan_digest
import oracle
for name, gen, args in (("cyclic5_p32003", gen_cyclic, (5,32003)), ("cyclic6_p32003", gen_cyclic, (6,32003)), ("katsura6_p32003", gen_katsura, (6,32003)), ("katsura8_p32003", gen_katsura, (8,32003)), ("cyclic7_p65521", gen_cyclic, (7,65521))):
    gold = json.load(open(f'tests/golden/{name}.json'))
    ring, polys = gen(*args)
    st = GroebnerState(ring)
    for f in polys: update_pairs(st, poly_monic(f))
    k = 0; bad = 0; t0 = time.time(); tsym = 0; tnum = 0
    while st.n_pairs():
        plan, ech, _ = f4_step(st)
        g = gold['steps'][k]
        pd = plan_digest(plan)
        rd = oracle.rref_sha256(ech.pivot_rows, ech.nonpivot_rows) if k < 100 else None
        if pd != g['plan_sha256'] or rd != g['rref_sha256']:
            bad += 1
            print(name, 'step', k, 'plan', pd == g['plan_sha256'], 'rref', rd == g['rref_sha256'], plan.counters, flush=True)
        s = st.stats[-1]; tsym += s.timings_ns['dict_build'] + s.timings_ns['row_assemble']; tnum += s.timings_ns['numeric_core']
        k += 1
    t1 = time.time()
    gb = reduce_basis(st.basis, ring)
    dig = hashlib.sha256(format_system(ring, gb).encode()).hexdigest()
    print(name, 'steps', k, 'bad', bad, 'final', dig == gold.get('final_sha256'), 'loop_s %.2f sym_ms %.2f num_ms %.2f reduce_s %.2f' % (t1-t0, tsym/1e6, tnum/1e6, time.time()-t1), flush=True)
