"""Quick end-to-end timing of the cfg2 workload through run_multi (GPU)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from cases import CASES, make_source
from paper_1503_08294_b200 import EngineParams, run_multi
for name in sys.argv[1:] or ["cfg1", "cfg2"]:
    case = CASES[name]
    params = EngineParams(**case["params"])
    for rep in range(2):
        net, st = run_multi(make_source(case["source"]), params, case["seed"])
        print(f"{name} rep{rep}: conv={st.converged} V={st.units} E={st.connections} "
              f"iters={st.iterations} signals={st.signals} disc={st.discarded} total={st.total_s:.3f}s "
              f"sample={st.sample_s:.3f} find={st.find_s:.3f} update={st.update_s:.3f} "
              f"-> {st.signals/st.total_s/1e6:.3f} M signals/s", flush=True)
