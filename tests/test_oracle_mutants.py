"""The 2D oracle pins catch plausible mistakes: each mutant below is oracle/ipm_oracle.c with ONE
deliberate error (the kind a reader could miss by eye), built with gcc into a temporary library and
loaded through ORACLE_LIB; the listed pins of tests/test_oracle_fv2d.py must fail on it.
("Next round" item 1: Rusanov dissipation, y-face order, quadrant assignment,
2D/triangle CFL, wall and free-stream ghosts.)"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "ipm_oracle.c")
PINS = "tests/test_oracle_fv2d.py"

# name: (original text, mutated text, pins that must fail)
MUTANTS = {
    "rusanov_speed_uses_|v|_not_|v.n|": (
        "double al = fabs(vl) + cl, ar = fabs(vr) + cr;",
        "double al = sqrt(ul[1] * ul[1] + ul[2] * ul[2]) / ul[0] + cl,"
        " ar = sqrt(ur[1] * ur[1] + ur[2] * ur[2]) / ur[0] + cr;",
        ["test_rusanov_hand_computed_values", "test_cartesian_step_is_numpy_2d_rusanov_fv"]),
    "rusanov_dissipation_without_half": (
        "- 0.5 * amax * (ur[a] - ul[a])", "- amax * (ur[a] - ul[a])",
        ["test_rusanov_hand_computed_values", "test_triangle_step_is_numpy_fv"]),
    "cartesian_y_faces_swapped": (
        "orc_flux_g(c, uj, nb_u[3], ny, 0.0, gp);\n    orc_flux_g(c, nb_u[2], uj, ny, 0.0, gm);",
        "orc_flux_g(c, uj, nb_u[2], ny, 0.0, gp);\n    orc_flux_g(c, nb_u[3], uj, ny, 0.0, gm);",
        ["test_cartesian_step_is_numpy_2d_rusanov_fv", "test_quadrant_ic_fractions_and_trajectory"]),
    "quadrants_NW_SE_swapped": (
        "fx * (1.0 - fy) * us[1][a] + fx * fy * us[2][a] +\n              (1.0 - fx) * fy * us[3][a]",
        "fx * (1.0 - fy) * us[3][a] + fx * fy * us[2][a] +\n              (1.0 - fx) * fy * us[1][a]",
        ["test_quadrant_ic_fractions_and_trajectory", "test_quadrant_ic_xi_dependent_projection"]),
    "cfl_2d_uses_dx_for_y": (
        "wave_speed(c, u, ny) * c->coef[j * 4 + 2]", "wave_speed(c, u, ny) * c->coef[j * 4 + 0]",
        ["test_cfl_step_closed_form_uniform_state", "test_cartesian_step_is_numpy_2d_rusanov_fv"]),
    "slip_ghost_half_reflection": (
        "ug[1 + q] = uin[1 + q] - 2.0 * mn * n[q];", "ug[1 + q] = uin[1 + q] - mn * n[q];",
        ["test_slip_wall_closed_form_single_triangle", "test_triangle_step_is_numpy_fv"]),
    "triangle_cfl_without_perimeter": (
        "return speed_norm(c, u) * c->perim[j] / c->area[j];", "return speed_norm(c, u) / c->area[j];",
        ["test_triangle_step_is_numpy_fv"]),  # (single triangle: its wall ghosts carry the same rate)
    "freestream_mach_on_wrong_xi": (
        "double Ma = s->q0[2] + s->q0[3] * xi[s->dim_a];", "double Ma = s->q0[2] + s->q0[3] * xi[s->dim_b];",
        ["test_free_stream_parallel_to_walls_is_preserved"]),
    "triangle_edge_flux_reversed": (
        "orc_flux_g(c, uj, nb_u[f], c->nrm + (j * F + f) * 2, 0.0, gp);",
        "orc_flux_g(c, nb_u[f], uj, c->nrm + (j * F + f) * 2, 0.0, gp);",
        ["test_triangle_step_is_numpy_fv", "test_slip_wall_closed_form_single_triangle"]),
}


@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_pins_fail_on_mutated_oracle(name, tmp_path):
    orig, mut, pins = MUTANTS[name]
    src = open(SRC).read()
    assert src.count(orig) == 1, f"mutation site of {name} not found exactly once"
    msrc = tmp_path / "ipm_oracle.c"
    msrc.write_text(src.replace(orig, mut))
    lib = tmp_path / "libipm_oracle_mutant.so"
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-I", os.path.join(ROOT, "oracle"),
                           "-o", str(lib), str(msrc), "-lm"])
    env = dict(os.environ, ORACLE_LIB=str(lib), OMP_NUM_THREADS="2")
    for pin in pins:
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", f"{PINS}::{pin}"],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
        # pytest exit code 1 = tests ran and at least one failed (2+ would be a collection/usage error)
        assert r.returncode == 1, f"{name}: pin {pin} did not fail (rc {r.returncode})\n{r.stdout[-2000:]}"
