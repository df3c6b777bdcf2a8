import numpy as np, sys
sys.path.insert(0, "/root/repo")
import workloads as W
from oracle import dense
from paper_2404_13184_b200 import Simulator
for n in (6, 7, 8):
    c, nm = W.config_workload(4, n=n)
    ref = dense.run(c, nm)
    for mirror in (True, False):
        with Simulator(n) as sim:
            st = sim.run_circuit(c, nm, mirror=mirror)
            got = sim.get_state().reshape(2**n, 2**n).T
        print(n, mirror, st["n_k3"], np.abs(got - ref).max(), flush=True)
