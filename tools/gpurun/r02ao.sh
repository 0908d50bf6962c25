set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "farfield" > gpurun_out/r02ao_farfield_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02ao_farfield_tests.log
timeout 600 python - > gpurun_out/r02ao_adaptive_stress_levels.txt 2>&1 <<'PY'
# diagnostic: level agreement of the adaptive config-4 run from the seeded stress state, Dirichlet vs far field
import numpy as np, torch, oracle
from inputs import configs
from tests.gpu_common import mesh_arrays, stress_inputs, to_np
from tests.test_gpu_parity import _farfield
from paper_1912_09238_b200 import Context
for name, cfg in [("dirichlet", configs.parity_variant("cfg4")), ("farfield", _farfield(configs.parity_variant("cfg4")))]:
    ma = mesh_arrays(cfg)
    o, g = oracle.Oracle(cfg, ma), Context(cfg, ma)
    base, z, amp = stress_inputs(cfg, 37, ma)
    lam = o.stress_dual(base, z, amp); u0 = o.moments_from_dual_all(lam)
    ug, lg = torch.from_numpy(u0.copy()).cuda(), torch.from_numpy(lam.copy()).cuda()
    uo, lo = u0.copy(), lam.copy()
    for s in range(3):
        o.step(uo, lo); g.ipm_step(ug, lg)
        print(name, s, "level mismatch", (o.levels() != to_np(g.levels())).mean(), "moment diff", np.abs(to_np(ug) - uo).max(), flush=True)
PY
