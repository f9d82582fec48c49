import sys, traceback
sys.path.insert(0, '/root/repo')
import paper_1301_4019_b200.bench_grid as B
for alg in ("multinomial", "multinomial-serial", "stratified", "systematic", "metropolis", "rejection", "rejection-capped"):
    for n in (64, 1024):
        try:
            r = B.run_cell(alg, n, 1.0, 0)
            print("ok", alg, n, r.elapsed_ns, flush=True)
        except Exception as e:
            print("FAIL", alg, n, repr(e)[:300], flush=True)
            traceback.print_exc()
            sys.exit(1)
