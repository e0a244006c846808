import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["stages"]["jacobi"], d["debug"]["jacobi_max_sweeps"], d["debug"]["jacobi_total_sweeps"], d["F_rel"], d["sigma_rel"])
