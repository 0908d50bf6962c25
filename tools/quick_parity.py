import numpy as np, torch, time, sys
sys.path.insert(0, "/root/repo")
from inputs import configs
import oracle
from paper_1912_09238_b200 import Context
from tests.gpu_common import assert_moments_close, to_np
for name in ["cfg1", "cfg2", "cfg3"]:
    cfg = configs.parity_variant(name)
    g = Context(cfg); o = oracle.Oracle(cfg)
    t0 = time.time(); u_o, l_o, io = o.run(); t1 = time.time()
    u_g, l_g, ig = g.run(); torch.cuda.synchronize(); t2 = time.time()
    sc = np.abs(u_o[:, 0, :]).max(axis=0)
    print(name, io["steps"], ig["steps"], io["t"], ig["t"], "err", (np.abs(to_np(u_g) - u_o) / sc).max(), f"ora {t1-t0:.2f}s gpu {t2-t1:.2f}s", flush=True)
