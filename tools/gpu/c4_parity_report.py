"""C3 / C4 ML-CPCP parity numbers against the reference fixtures (the gate
itself is tests/test_gpu_large.py::test_cpcp_full_size_envelope)."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import test_gpu_large as T

for name, cap in [("C3", 5000), ("C4", 300)]:
    g = T.fixture(f"{name.lower()}_cpcp")
    st = T.run_cpcp(name, g, cap)
    env_obj = np.asarray(g["env_obj"], dtype=np.float64)
    ref = float(env_obj[0])
    spread = (env_obj.max() - env_obj.min()) / ref
    dobj = abs(st.objective_history[-1] - ref) / ref
    rows = g["rows"]
    rs = T.relf(st.s[rows].cpu().numpy(), g["s_rows"])
    rl = T.relf(st.l[rows].cpu().numpy(), g["l_rows"])
    sk = T.device_sketches(st.s, "s")
    lk = T.device_sketches(st.l, "l")
    print(name, "iters", st.iter, "env", list(np.asarray(g["env_iter"])), "dobj %.2e spread %.2e" % (dobj, spread),
          "relF rows S %.2e L %.2e" % (rs, rl), "sketch S %.2e L %.2e" % (T.relf(sk["s_q"], g["s_q"]), T.relf(lk["l_q"], g["l_q"])),
          flush=True)
