"""C-ABI checks that need no GPU: libipm.so loads, exports every entry point include/ipm.h declares,
the ctypes structures match the C layout, and calls fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ipm.h")


@pytest.fixture(scope="module")
def ipm():
    from paper_1912_09238_b200 import build, ipm

    build.build()
    return ipm


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^IPM_API\s+[\w\s\*]*?\b(ipm_\w+)\s*\(", src, flags=re.M)))


def test_every_declared_symbol_is_exported(ipm):
    names = declared()
    assert len(names) >= 20
    L = C.CDLL(ipm.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert sorted(ipm.EXPORTS) == names
    out = subprocess.check_output(["nm", "-D", "--defined-only", ipm.LIB_PATH]).decode()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(names) <= exported


def test_ctypes_layout_matches_c(ipm, tmp_path):
    prog = tmp_path / "layout.c"
    prog.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HDR}"
#define O(T, f) printf(#T "." #f " %zu\\n", offsetof(T, f))
int main(void) {{
  printf("ipm_config %zu\\n", sizeof(ipm_config));
  printf("ipm_state %zu\\n", sizeof(ipm_state));
  printf("ipm_ic %zu\\n", sizeof(ipm_ic));
  printf("ipm_step_info %zu\\n", sizeof(ipm_step_info));
  O(ipm_config, gamma); O(ipm_config, x0); O(ipm_config, h_vert); O(ipm_config, bc_kind);
  O(ipm_config, bc_state); O(ipm_config, tau); O(ipm_config, cfl); O(ipm_config, n_levels);
  O(ipm_config, delta_dec); O(ipm_config, rank); O(ipm_config, reserved_ptr); O(ipm_config, stream);
  O(ipm_ic, xs0); O(ipm_ic, state); O(ipm_step_info, newton_iters); O(ipm_step_info, worst_status);
  O(ipm_config, n_retard); O(ipm_config, retard_level); O(ipm_config, retard_eps); O(ipm_config, quad_kind);
  O(ipm_config, quad_level); O(ipm_config, hessian_kind); O(ipm_config, lbfgs_m);
  O(ipm_config, level_q1d);
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-o", str(exe), str(prog)])
    lines = dict(ln.rsplit(" ", 1) for ln in subprocess.check_output([str(exe)]).decode().split("\n") if ln)
    assert int(lines["ipm_config"]) == C.sizeof(ipm.ipm_config)
    assert int(lines["ipm_state"]) == C.sizeof(ipm.ipm_state)
    assert int(lines["ipm_ic"]) == C.sizeof(ipm.ipm_ic)
    assert int(lines["ipm_step_info"]) == C.sizeof(ipm.ipm_step_info)
    for key, val in lines.items():
        if "." in key:
            struct, field = key.split(".")
            assert getattr(getattr(ipm, struct), field).offset == int(val), key
    # and as compiled into the library (nvcc / host compiler of the .so)
    L = ipm.lib()
    assert L.ipm_struct_size(0) == C.sizeof(ipm.ipm_config)
    assert L.ipm_struct_size(1) == C.sizeof(ipm.ipm_ic)
    assert L.ipm_struct_size(2) == C.sizeof(ipm.ipm_step_info)


def test_oracle_problem_layout_matches_c():
    import oracle.oracle as orc

    assert orc.lib().orc_problem_size() == C.sizeof(orc.Problem)


def test_no_cpu_fallback(ipm):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = ipm.lib()
    cfg = ipm.ipm_config()
    h = C.c_void_p()
    rc = L.ipm_init(C.byref(cfg), C.byref(h))
    assert rc == 2  # IPM_ERR_CUDA
    assert b"no CUDA device" in L.ipm_last_error()


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1912_09238_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.lower() or f == "__init__.py" and "oracle" not in src, f
