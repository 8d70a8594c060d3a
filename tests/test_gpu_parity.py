"""CUDA path vs golden fixtures made by the reference (bitwise where the
reference is bitwise; rtol 1e-12 per cell otherwise, north_star tolerance).
All calls go through the C-ABI library libomb200.so."""

import numpy as np
import pytest

from _cases import EOS, DensityGravity, bitwise_mismatch, case_tree, golden, rel_close, sources_gravity, state_of

pytestmark = pytest.mark.gpu

CORE = (slice(None), slice(None), slice(2, 12), slice(2, 12), slice(2, 12))


@pytest.fixture(scope="module")
def K():
    return golden("kernels")


@pytest.fixture(scope="module")
def kern():
    from paper_2107_10987_b200 import kernels

    return kernels


def test_library_is_native(kern):
    from paper_2107_10987_b200 import _lib

    L = _lib.load()
    assert L.omb_abi_version() == _lib.ABI_VERSION
    assert kern.BACKEND_NAME == "b200"


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_kernel_module_parity(K, kern, seed):
    import oracle  # checker only

    u = K[f"s{seed}_u"]
    prim = kern.primitives(u, 1.4, 1e-3)
    assert bitwise_mismatch(prim, oracle.primitives(u, 1.4, 1e-3)) == 0
    for new in (True, False):
        for contact in (False, True):
            tag = f"s{seed}_{'new' if new else 'old'}_{'c' if contact else 'nc'}"
            lo, hi, fb = kern.reconstruct(prim, 8, new, contact, 1.4)
            lo_r, hi_r, fb_r = oracle.reconstruct(prim, 8, new, contact, 1.4)
            assert fb == fb_r == int(K[tag + "_fallback"])
            nl = 13 if new else 3
            assert bitwise_mismatch(lo[:nl][CORE], lo_r[:nl][CORE]) == 0
            assert bitwise_mismatch(hi[:nl][CORE], hi_r[:nl][CORE]) == 0
            if not new:
                assert np.all(lo[3] == 0.0)  # tests/test_hydro.py:172-178
            if contact:
                continue
            for ov in ((False, True) if new else (False,)):
                t2 = tag + ("_ov" if ov else "")
                fx, fy, fz, am = kern.fluxes(lo, hi, 8, 1.4, new, ov)
                for got, key in ((fx, "_fx"), (fy, "_fy"), (fz, "_fz")):
                    assert bitwise_mismatch(got, K[t2 + key]) == 0
                assert am == float(K[t2 + "_amax"])


@pytest.mark.parametrize("tag", ["fb", "fb2"])
def test_fallback_cases(K, kern, tag):
    prim = kern.primitives(K[tag + "_u"], 1.4, 1e-3)
    lo, hi, fb = kern.reconstruct(prim, 8, True, False, 1.4)
    assert fb == int(K[tag + "_fallback"])
    fx, fy, fz, am = kern.fluxes(lo, hi, 8, 1.4, True, False)
    for got, key in ((fx, "_fx"), (fy, "_fy"), (fz, "_fz")):
        assert bitwise_mismatch(got, K[tag + key]) == 0


def _stepper(t, **kw):
    from paper_2107_10987_b200 import HydroMode
    from paper_2107_10987_b200.stepper import B200HydroStepper

    mode = kw.pop("mode", HydroMode("new"))
    eos = kw.pop("eos", EOS)
    return B200HydroStepper(t, eos, mode, **kw)


def _check_state(t, g, key="state1"):
    got = state_of(t)
    ref = g[key]
    # every field bitwise, tau included (the device pow is glibc's, csrc/omb_pow.cuh)
    assert bitwise_mismatch(got[:, :5], ref[:, :5]) == 0
    assert bitwise_mismatch(got, ref) == 0
    assert rel_close(got, ref, 1e-12) == 0


@pytest.mark.parametrize("name", ["smooth_periodic", "smooth_reflecting", "sedov_c1", "amr_sedov_small"])
@pytest.mark.parametrize("max_run", [1, 4])
def test_step_parity(name, max_run):
    t, g = case_tree(name)
    st = _stepper(t, max_run=max_run)
    dt = st.cfl_dt(0.4)
    assert dt == float(g["dts"][0])
    stats = st.rk3_step(dt)
    _check_state(t, g)
    assert stats.amax == float(g["amax"][0])
    assert stats.fallback_count == int(g["fallback"][0])
    assert stats.kernel_launches == 6 * len(t.sorted_leaves())


@pytest.mark.parametrize("name", ["sedov_c1", "amr_sedov_small"])
@pytest.mark.parametrize("split", ["4", "6,3", "100"])
def test_step_parity_split_tail(monkeypatch, name, split):
    """Runs of mixed lengths (the last k runs split in halves; "6,3" splits twice; "100"
    is skipped for the 16-run c1 batch, not below its run count) give the golden step."""
    monkeypatch.setenv("OMB_SPLIT_TAIL", split)
    t, g = case_tree(name)
    st = _stepper(t)
    lens = np.diff(st.batch.run_off)
    if split != "100" or st.batch.nruns > 100:
        assert lens.min() < lens.max()
    stats = st.rk3_step(st.cfl_dt(0.4))
    _check_state(t, g)
    assert stats.amax == float(g["amax"][0])
    assert stats.fallback_count == int(g["fallback"][0])


def test_old_scheme_two_steps():
    from paper_2107_10987_b200 import HydroMode

    t, g = case_tree("smooth_old")
    st = _stepper(t, mode=HydroMode("old"))
    for s in range(2):
        dt = st.cfl_dt(0.3)
        assert dt == float(g["dts"][s])
        st.rk3_step(dt)
        if s == 0:
            _check_state(t, g)
    _check_state(t, g, "final")


def test_sedov_c1_ten_steps_totals():
    from octomini_host import conservation_totals

    t, g = case_tree("sedov_c1")
    st = _stepper(t)
    for s in range(10):
        dt = st.cfl_dt(0.4)
        assert dt == float(g["dts"][s])
        st.rk3_step(dt)
    tot = np.array(list(conservation_totals(t).values()))
    ref = g["totals"]
    assert np.all(np.abs(tot - ref) <= 1e-12 * np.maximum(np.abs(ref), 1e-30))


def test_sources_floors():
    t, g = case_tree("sources")
    grav = sources_gravity(t, g)
    from paper_2107_10987_b200 import EosConfig, FloorConfig

    fl = [float(x) for x in g["floors"]]
    st = _stepper(t, eos=EosConfig(gamma=float(g["gamma"])), gravity=grav, omega=float(g["omega"]),
                  floors=FloorConfig(rho=fl[0], tau=fl[1], vmax=fl[2]))
    dt = st.cfl_dt(0.4)
    assert dt == float(g["dts"][0])
    st.rk3_step(dt)
    _check_state(t, g)


def test_gather_matches_ghost_golden():
    import ctypes

    import torch

    import octomini_host as mesh
    from paper_2107_10987_b200 import _lib
    from paper_2107_10987_b200.batch import LeafBatch

    g = golden("ghosts")
    L = _lib.load()
    for bnd in ("periodic", "reflecting", "outflow"):
        t = mesh.build_uniform_tree(1, 8, boundary=bnd)
        for lf, u in zip(t.sorted_leaves(), g[bnd]):
            lf.subgrid.interior[:] = u[:, 3:11, 3:11, 3:11]
        b = LeafBatch(t)
        U = torch.from_numpy(np.ascontiguousarray(b.pack())).cuda()
        info = torch.from_numpy(b.info.view(np.uint8).copy()).cuda()
        for i in range(b.L):
            out = torch.empty((6, 14, 14, 14), dtype=torch.float64, device="cuda")
            _lib.check(L.omb_gather(U.data_ptr(), b.fstride, info.data_ptr(), i, b.bc, out.data_ptr(),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "gather")
            assert bitwise_mismatch(out.cpu().numpy(), g[bnd][i]) == 0


def test_cfl_abort_raises_and_rolls_back():
    from paper_2107_10987_b200 import NumericsError

    t, g = case_tree("smooth_periodic")
    st = _stepper(t)
    before = state_of(t).copy()
    with pytest.raises(NumericsError):
        st.rk3_step(dt=10.0)
    assert bitwise_mismatch(state_of(t), before) == 0  # stage 1 aborted: interiors untouched


def test_non_finite_speed_raises():
    from paper_2107_10987_b200 import NumericsError

    t, g = case_tree("smooth_periodic")
    t.sorted_leaves()[3].subgrid.interior[0, 0, 0, 0] = 0.0
    st = _stepper(t)
    with pytest.raises(NumericsError, match="non-finite wave speed"):
        st.cfl_dt(0.4)


def test_reciprocal_division_is_ieee_exact():
    """div_by (one reciprocal + two fma corrections, used for the six KT
    quotients) must equal IEEE division bit for bit: 2^30 random pairs."""
    import ctypes

    import torch

    from paper_2107_10987_b200 import _lib

    L = _lib.load()
    bad = torch.zeros(8, dtype=torch.int64, device="cuda")
    _lib.check(L.omb_selftest_div(12345, 1 << 30, bad.data_ptr(),
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "selftest")
    b = bad.cpu().numpy()
    assert int(b[0]) == 0, ("first mismatch a, b, a/b, div_by, kt form:", b[1:6].view(np.float64).tolist())


def test_amr_reflux_two_steps_gpu():
    """AMR tree (level-1 + one refined corner, periodic): coarse/fine ghosts, reflux, 2 steps."""
    import hashlib

    t, g = case_tree("amr_reflux")
    st = _stepper(t)
    for s in range(2):
        dt = st.cfl_dt(0.4)
        assert dt == float(g["dts"][s])
        stats = st.rk3_step(dt)
        if s == 0:
            _check_state(t, g)
        assert stats.amax == float(g["amax"][s])
    got = np.ascontiguousarray(state_of(t))
    assert hashlib.sha256(got.tobytes()).hexdigest() == str(g["final_sha"])


def test_synthetic_star_matches_oracle():
    """Config c5 stand-in (rotating frame + fixed gravity + floors, outflow): GPU vs the CPU oracle, 2 steps."""
    from oracle.step import OracleStepper
    from paper_2107_10987_b200 import HydroMode
    from octomini_host import synthetic_star
    from paper_2107_10987_b200.stepper import B200HydroStepper

    tg, eos, grav, om, fl = synthetic_star(level=2)
    tc, _, gravc, _, _ = synthetic_star(level=2)
    gpu = B200HydroStepper(tg, eos, HydroMode("new"), gravity=grav, omega=om, floors=fl)
    ref = OracleStepper(tc, eos.gamma, omega=om, gravity=gravc, floors=(fl.rho, fl.tau, fl.vmax))
    for _ in range(2):
        dt = gpu.cfl_dt(0.4)
        assert dt == ref.cfl_dt(0.4)
        gpu.rk3_step(dt)
        ref.rk3_step(dt)
    a, b = state_of(tg), state_of(tc)
    # the atmosphere uses the dual-energy tau branch (pressure from tau**gamma): with glibc's
    # pow on the device every field is bitwise
    assert rel_close(a, b, 1e-12) == 0
    assert bitwise_mismatch(a, b) == 0


def _ghosts(t):
    out = []
    for lf in t.sorted_leaves():
        u = lf.subgrid.u.copy()
        u[:, 3:11, 3:11, 3:11] = 0.0
        out.append(u)
    return np.stack(out)


@pytest.mark.parametrize("xfer", ["mapped", "mapped-tail", "threads", "hybrid"])
def test_host_transfer_paths(monkeypatch, xfer):
    """Every host<->device transfer path gives the golden step, leaves the host
    ghost cells exactly as they were (the mapped path writes whole 64 B lines,
    restoring the neighbouring ghost doubles from its stash), and picks up leaf
    arrays a user replaced.  mapped-tail: the last stage in one-run launch parts,
    each part's leaves written to the host while the next computes.  hybrid: the
    GPU gathers part of the leaves while host threads pack the others."""
    monkeypatch.setenv("OMB_HOST_XFER", xfer.split("-")[0])
    monkeypatch.setenv("OMB_GATHER_FRAC", "0.4")
    if xfer == "mapped-tail":
        monkeypatch.setenv("OMB_TAIL_RUNS", "1")
    t, g = case_tree("smooth_reflecting")
    rng = np.random.default_rng(11)
    for lf in t.sorted_leaves():  # distinctive host ghost values
        u = lf.subgrid.u
        keep = u[:, 3:11, 3:11, 3:11].copy()
        u[...] = rng.standard_normal(u.shape)
        u[:, 3:11, 3:11, 3:11] = keep
    ghosts = _ghosts(t)
    st = _stepper(t)
    assert (st._mapped is not None) == (xfer != "threads")
    assert (st._gather_frac is not None) == (xfer == "hybrid")
    assert (st._tail is not None) == (xfer == "mapped-tail")
    st.rk3_step(st.cfl_dt(0.4))
    _check_state(t, g)
    assert bitwise_mismatch(_ghosts(t), ghosts) == 0
    for lf, a in zip(t.sorted_leaves(), g["init"]):  # new arrays holding the initial state
        u = lf.subgrid.u.copy()
        u[:, 3:11, 3:11, 3:11] = a
        lf.subgrid._u = u
    st.rk3_step(st.cfl_dt(0.4))
    _check_state(t, g)
    assert bitwise_mismatch(_ghosts(t), ghosts) == 0


@pytest.mark.parametrize("xfer", ["threads", "mapped", "hybrid"])
@pytest.mark.parametrize("part_runs", [1, 3, 7])
def test_overlapped_download(monkeypatch, part_runs, xfer):
    """The last stage launched in parts with each part's leaves copied back while
    the next computes gives the golden step (and the CFL-abort rollback still holds)."""
    monkeypatch.setenv("OMB_HOST_XFER", xfer)
    monkeypatch.setenv("OMB_GATHER_FRAC", "0.3")
    monkeypatch.setenv("OMB_TAIL_RUNS", str(part_runs))
    t, g = case_tree("sedov_c1")
    st = _stepper(t)
    assert st._tail is not None and len(st._tail["cuts"]) > 2
    stats = st.rk3_step(st.cfl_dt(0.4))
    _check_state(t, g)
    assert stats.amax == float(g["amax"][0])
    before = state_of(t).copy()
    from paper_2107_10987_b200 import NumericsError

    with pytest.raises(NumericsError):
        st.rk3_step(dt=10.0)
    assert bitwise_mismatch(state_of(t), before) == 0


@pytest.mark.parametrize("max_run", [1, 4])
def test_contact_detection_steps(max_run):
    """HydroMode('new', contact_detection=True) through the fused kernel (the
    steepener of _core.pyx:107-142 inside k_stage), 2 steps vs the reference."""
    from paper_2107_10987_b200 import HydroMode

    t, g = case_tree("contact_step")
    st = _stepper(t, mode=HydroMode("new", contact_detection=True), max_run=max_run)
    for s in range(2):
        dt = st.cfl_dt(0.4)
        assert dt == float(g["dts"][s])
        stats = st.rk3_step(dt)
        if s == 0:
            _check_state(t, g)
        assert stats.amax == float(g["amax"][s])
        assert stats.fallback_count == int(g["fallback"][s])
    _check_state(t, g, "final")


@pytest.mark.parametrize("mode", ["override", "old"])
@pytest.mark.parametrize("max_run", [1, 4])
def test_override_equals_old_ten_steps(mode, max_run):
    """new + quadrature_override == old, bitwise over 10 steps at a fixed dt
    (reference tests/test_hydro_step.py:151-164): both modes reproduce the
    reference's 10-step state."""
    from paper_2107_10987_b200 import HydroMode

    t, g = case_tree("override_10")
    m = HydroMode("new", quadrature_override=True) if mode == "override" else HydroMode("old")
    st = _stepper(t, mode=m, max_run=max_run)
    dt = st.cfl_dt(0.3)
    assert dt == float(g["dt"])
    for _ in range(10):
        st.rk3_step(dt)
    _check_state(t, g, "final")


@pytest.mark.parametrize("name", ["gravity_density", "gravity_density_amr"])
def test_state_dependent_host_gravity(name):
    """A host gravity object that reads the stage state (g from density
    differences across ghost cells, dphi/dt from momenta) is solved every stage on
    the stage state with filled ghosts, as HydroStepper._stage does (step.py:106-113)."""
    t, g = case_tree(name)
    st = _stepper(t, gravity=DensityGravity(), omega=0.2 if name == "gravity_density" else 0.0)
    for s in range(len(g["dts"])):
        dt = st.cfl_dt(0.4)
        assert dt == float(g["dts"][s])
        stats = st.rk3_step(dt)
        if s == 0:
            _check_state(t, g)
        assert stats.amax == float(g["amax"][s])
    if "final" in g:
        _check_state(t, g, "final")


def test_gather_matches_amr_ghost_golden():
    """omb_gather_leaves after omb_amr_ghosts = the reference's exchange_ghosts on an
    AMR tree (coarse/fine prolongation + restriction regions included)."""
    import ctypes
    import json

    import torch

    import octomini_host as mesh
    from paper_2107_10987_b200 import _lib
    from paper_2107_10987_b200._abi import OmbAmrDesc
    from paper_2107_10987_b200.batch import LeafBatch

    g = golden("ghosts")
    L = _lib.load()
    t = mesh.build_uniform_tree(1, 8, boundary="reflecting")
    t.split(t.leaf_at(1, (0, 0, 0)))
    t.reindex()
    assert [json.loads(p) for p in g["amr_paths"]] == [list(lf.path) for lf in t.sorted_leaves()]
    for lf, u in zip(t.sorted_leaves(), g["amr"]):
        lf.subgrid.interior[:] = u[:, 3:11, 3:11, 3:11]
    b = LeafBatch(t)
    U = torch.from_numpy(np.ascontiguousarray(b.pack())).cuda()
    info = torch.from_numpy(b.info.view(np.uint8).copy()).cuda()
    tasks = torch.from_numpy(b.amr_tasks.reshape(-1).copy()).cuda()
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ad = OmbAmrDesc(u=U.data_ptr(), fstride=b.fstride, tasks=tasks.data_ptr(), ntasks=b.nvirtual)
    _lib.check(L.omb_amr_ghosts(ctypes.byref(ad), sh), "omb_amr_ghosts")
    out = torch.empty((b.L, 6, 14, 14, 14), dtype=torch.float64, device="cuda")
    _lib.check(L.omb_gather_leaves(U.data_ptr(), b.fstride, info.data_ptr(), 0, b.L, b.bc, out.data_ptr(), sh),
               "omb_gather_leaves")
    assert bitwise_mismatch(out.cpu().numpy(), g["amr"]) == 0


def test_kernels_module_threads_and_devices():
    """The C ABI's one-time setup is per device and thread-safe: the kernels shim
    called from 8 host threads at once (the reference's scheduler threads call
    kernels concurrently, _core.pyx:60,239), and on every visible device."""
    import threading

    import torch

    from paper_2107_10987_b200 import kernels

    K = golden("kernels")
    u = K["s0_u"]
    ref_fx = K["s0_new_nc_fx"]
    errs = []

    def work(dev):
        try:
            with torch.cuda.device(dev):
                torch.cuda.set_device(dev)
                prim = kernels.primitives(u, 1.4, 1e-3)
                lo, hi, _ = kernels.reconstruct(prim, 8, True, False, 1.4)
                fx, _, _, _ = kernels.fluxes(lo, hi, 8, 1.4, True, False)
                if bitwise_mismatch(fx, ref_fx):
                    errs.append(f"device {dev}: flux mismatch")
        except Exception as e:  # noqa: BLE001
            errs.append(f"device {dev}: {e!r}")

    ndev = torch.cuda.device_count()
    th = [threading.Thread(target=work, args=(k % ndev,)) for k in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs


def test_stepper_on_second_device():
    """B200HydroStepper(device='cuda:1') while cuda:0 is current: allocations,
    library setup and launches all land on device 1 (one step == golden)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    torch.cuda.set_device(0)
    t, g = case_tree("sedov_c1")
    st = _stepper(t, device="cuda:1")
    assert st.state_tensor().device.index == 1
    dt = st.cfl_dt(0.4)
    assert dt == float(g["dts"][0])
    st.rk3_step(dt)
    _check_state(t, g)
    assert torch.cuda.current_device() == 0


def test_device_pow_is_glibc():
    """pow_glibc on the device == the host libm's pow, bit for bit: 2^22 random
    pairs over every exponent, the exponents the step uses, and edge cases."""
    import ctypes

    import torch

    import oracle  # checker only
    from paper_2107_10987_b200 import _lib

    rng = np.random.default_rng(7)
    n = 1 << 22
    xb = rng.integers(0, 2 ** 63, n, dtype=np.uint64)
    x = xb.view(np.float64).copy()
    y = rng.integers(0, 2 ** 63, n, dtype=np.uint64).view(np.float64).copy()
    y[::2] = rng.choice([1.4, 1 / 1.4, 5 / 3, 0.6], n // 2)
    x[1::4] = np.exp(rng.uniform(-30, 30, len(x[1::4])))
    x[3::8] = -x[3::8]
    y[3::16] = 3.0
    edge = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 5e-324, 2.2250738585072014e-308, 1e-300, 1e300])
    ex, ey = np.meshgrid(edge, np.array([0.0, 1.0, -1.0, 2.0, 0.5, 1.4, -1.4, np.inf, -np.inf, np.nan, 1e300]))
    x = np.concatenate([x, ex.ravel()])
    y = np.concatenate([y, ey.ravel()])
    ref = oracle.pow_batch(x, y)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    out = torch.empty_like(dx)
    L = _lib.load()
    _lib.check(L.omb_selftest_pow(dx.data_ptr(), dy.data_ptr(), x.size, out.data_ptr(),
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "omb_selftest_pow")
    got = out.cpu().numpy()
    assert bitwise_mismatch(got, ref) == 0


@pytest.mark.parametrize("name", ["sedov_n16", "sedov_n32", "smooth_n16", "fallback_n16"])
def test_subgrid_sizes_16_32(name):
    """octomini's 16^3 and 32^3 sub-grids (tree.py:13) through B200HydroStepper: every step
    bitwise, the per-leaf fallback count exact, kernel_launches counted per leaf of the tree."""
    t, g = case_tree(name)
    st = _stepper(t)
    for s in range(len(g["dts"])):
        dt = st.cfl_dt(0.1 if name == "fallback_n16" else 0.4)
        assert dt == float(g["dts"][s])
        stats = st.rk3_step(dt)
        if s == 0:
            _check_state(t, g)
        assert stats.amax == float(g["amax"][s])
        assert stats.fallback_count == int(g["fallback"][s])
        assert stats.kernel_launches == 6 * len(t.leaves())
    if "final" in g:
        _check_state(t, g, "final")
