"""GPU parity of the kinetic-flux moment update (SURVEY §8a row a11 + projection, PAPER.md:130 and
182-185) for every cartesian flux kernel (IPM_FLUX_KERNEL = strip (default), cart, warp) against the
oracle, on meshes that exercise the strip kernel's edges: ragged strips (nx not a multiple of the strip
width), a single narrow column, periodic wrap in x and y, ghost-state and slip-wall boundaries, both
update forms; and the kernels against each other at rounding level."""
import numpy as np
import pytest

from inputs import configs

from .gpu_common import stress_inputs, to_np

pytestmark = pytest.mark.gpu

GAMMA = 1.4
FS = {"freestream": dict(rho=1.0, p=1.0 / GAMMA, mach0=0.5, dmach=0.05, dim_mach=0, theta0_deg=20.0,
                         dtheta_deg=5.0, dim_theta=1)}

CASES = {
    "ragged_13x7": dict(mesh=dict(nx=13, ny=7)),
    "narrow_1x9": dict(mesh=dict(nx=1, ny=9)),
    "single_3x2": dict(mesh=dict(nx=3, ny=2)),
    "periodic_16x5": dict(mesh=dict(nx=16, ny=5, periodic=True)),
    "ghost_slip_9x11": dict(mesh=dict(nx=9, ny=11), bc=[("slip", None), ("state", FS), ("state", FS), ("slip", None)]),
    "cform_24x17": dict(mesh=dict(nx=24, ny=17), update="paper_c"),
    # more strips (151) than CTAs (148 SMs): the contiguous (non-banded) work split of k_flux_strip
    "wide_1201x3": dict(mesh=dict(nx=1201, ny=3)),
}


@pytest.fixture(scope="module")
def torch():
    import torch as t

    if not t.cuda.is_available():
        pytest.fail("GPU test needs CUDA (no CPU fallback exists)")
    return t


def _cfg(case):
    kw = dict(CASES[case])
    mesh = kw.pop("mesh")
    cfg = configs.get("cfg3", mesh=mesh)
    cfg.update(kw)
    return cfg


def _gpu_update(torch, cfg, lam_star, u_o, dt):
    from paper_1912_09238_b200 import Context

    g = Context(cfg)
    lam = torch.tensor(lam_star, device="cuda")
    u = torch.tensor(u_o, device="cuda")
    unew = g.zeros()
    g.ipm_flux_update(lam, u, unew, dt)
    torch.cuda.synchronize()
    return to_np(unew)


def _inputs(cfg, seed):
    import oracle

    o = oracle.Oracle(cfg)
    base, z, amp = stress_inputs(cfg, seed=seed)
    lam_star = o.stress_dual(base, z, amp)
    u_o = o.moments_from_dual_all(lam_star)
    return o, lam_star, u_o


@pytest.mark.parametrize("kernel", ["strip", "cart", "warp"])
@pytest.mark.parametrize("case", list(CASES))
def test_flux_update_matches_oracle(torch, monkeypatch, case, kernel):
    monkeypatch.setenv("IPM_FLUX_KERNEL", kernel)
    cfg = _cfg(case)
    o, lam_star, u_o = _inputs(cfg, seed=11)
    dt = 1e-4
    ref = o.flux_update(lam_star, u_o, dt)
    got = _gpu_update(torch, cfg, lam_star, u_o, dt)
    sc = np.maximum(np.abs(ref[:, 0, :]).max(axis=0), 1e-300)
    err = (np.abs(got - ref) / sc[None, None, :]).max()
    assert err <= 1e-12, f"{case} {kernel}: {err:.3e}"


@pytest.mark.parametrize("case", list(CASES))
def test_strip_kernel_matches_cart_kernel(torch, monkeypatch, case):
    """the strip kernel forms every Rusanov ingredient once and every y face once; with the same
    face formula and accumulation order as k_flux_cart its results agree to rounding"""
    cfg = _cfg(case)
    _, lam_star, u_o = _inputs(cfg, seed=5)
    out = {}
    for kern in ("strip", "cart"):
        monkeypatch.setenv("IPM_FLUX_KERNEL", kern)
        out[kern] = _gpu_update(torch, cfg, lam_star, u_o, 2e-4)
    sc = np.maximum(np.abs(out["cart"][:, 0, :]).max(axis=0), 1e-300)
    err = (np.abs(out["strip"] - out["cart"]) / sc[None, None, :]).max()
    assert err <= 1e-14, f"{case}: {err:.3e}"
