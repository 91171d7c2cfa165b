"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star, A13): per state
max_i |x_gpu - x_oracle| / max_i |x_oracle| <= 1e-10 (fp64), <= 1e-4 (fp32).
FD is judged by backward error (A14) plus a cond-scaled forward error.
"""
import numpy as np
import pytest

import oracle
import synth
from conftest import rel_err_per_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {torch.float64: 1e-10, torch.float32: 1e-4}


def parity_sample(B, tile=256, seed=99):
    """SURVEY §8(d) parity sample of a B-state launch: the first and last 1024
    states, both neighbours of EVERY tile boundary of the thread kernel (tiles of
    `tile` = 32 W states, W = 8 fp64 / 16 fp32, so 256 covers both), every shard
    boundary of k = 2, 4, 8 ranks +-16, and 65,536 random indices (seed 99)."""
    rng = np.random.default_rng(seed)
    parts = [np.arange(min(B, 1024)), np.arange(max(0, B - 1024), B), rng.integers(0, B, 65536)]
    edges = np.arange(tile, B, tile)
    parts += [edges - 1, edges]
    for k in (2, 4, 8):
        for r in range(1, k):
            b = (B // k) * r + min(r, B % k)
            parts.append(np.arange(max(0, b - 16), min(B, b + 16)))
    return np.unique(np.concatenate(parts))


@pytest.fixture(scope="module")
def rd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1609_04493_b200 as rd
    rd.lib()
    return rd


def dev(x, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype=dtype)


def run_id(rd, model, q, qd, qdd, dtype=torch.float64):
    tq, tqd, tqdd = dev(q, dtype), dev(qd, dtype), dev(qdd, dtype)
    tau = rd.inverse_dynamics(model, tq, tqd, tqdd)
    torch.cuda.synchronize()
    # the oracle sees exactly the (rounded) inputs the kernel saw
    return tau.double().cpu().numpy(), (tq.double().cpu().numpy(), tqd.double().cpu().numpy(),
                                        tqdd.double().cpu().numpy())


def check_id(rd, robot, g, q, qd, qdd, dtype=torch.float64, strategy="auto", sample=None):
    model = rd.Model.from_robot(robot, g)
    model.set_strategy(strategy)
    tau, (q64, qd64, qdd64) = run_id(rd, model, q, qd, qdd, dtype)
    cols = np.arange(q.shape[1]) if sample is None else sample
    ref = oracle.rnea_batch(robot, g, q64[:, cols], qd64[:, cols], qdd64[:, cols])
    err = rel_err_per_state(tau[:, cols], ref)
    assert np.all(np.isfinite(tau[:, cols]))
    assert err.max() <= TOL[dtype], f"max rel err {err.max():.3e} (strategy {strategy}, {dtype})"
    return err.max()


# ------------------------------------------------------------------ configs
def test_C1_planar2_closed_form_config(rd):
    cfg = synth.CONFIGS["C1"]
    q, qd, qdd = synth.states(cfg["seed"], 2, 0, cfg["batch"], cfg["ranges"])
    for strat in ("auto", "thread", "generic", "warp_scan"):
        check_id(rd, synth.planar2(), cfg["gravity"], q, qd, qdd, strategy=strat)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_C2_arm7(rd, dtype):
    cfg = synth.CONFIGS["C2"]
    q, qd, qdd = synth.states(cfg["seed"], 7, 0, cfg["batch"], cfg["ranges"])
    for strat in ("thread", "generic", "warp_scan"):
        check_id(rd, synth.arm7(), cfg["gravity"], q, qd, qdd, dtype, strategy=strat)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_C3_full_size_sampled(rd, dtype):
    # Full 1M-state launch (the bench configuration), sampled oracle comparison:
    # first/last 1024, every 128-state tile boundary neighbourhood, and random states.
    cfg = synth.CONFIGS["C3"]
    n, B = cfg["n"], cfg["batch"]
    q, qd, qdd = synth.states(cfg["seed"], n, 0, B, cfg["ranges"])
    sample = parity_sample(B)
    assert sample.size >= 65536
    check_id(rd, synth.robot_for(cfg), cfg["gravity"], q, qd, qdd, dtype, sample=sample)


def test_C5_full_size_sampled(rd):
    # BASELINE config C5: 10^7 states on one GPU (the single-GPU bench workload of
    # --config C5; 1.25M per GPU at 8 GPUs), the launch bench.py times.  Inputs are
    # generated chunk by chunk straight into device memory; the oracle checks a
    # sample: both ends, tile-boundary neighbourhoods and random states.
    cfg = synth.CONFIGS["C5"]
    n, B = cfg["n"], cfg["batch"]
    tq, tqd, tqdd = (torch.empty((n, B), dtype=torch.float64, device="cuda") for _ in range(3))
    chunk = 1_000_000
    for b0 in range(0, B, chunk):
        b1 = min(B, b0 + chunk)
        for t, x in zip((tq, tqd, tqdd), synth.states(cfg["seed"], n, b0, b1, cfg["ranges"])):
            t[:, b0:b1].copy_(torch.from_numpy(x))
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    assert model.resolve_strategy(B, True) == "thread"
    tau = rd.inverse_dynamics(model, tq, tqd, tqdd)
    sample = parity_sample(B)
    assert sample.size >= 65536
    idx = torch.from_numpy(sample).cuda()
    got = tau[:, idx].cpu().numpy()
    q, qd, qdd = (t[:, idx].cpu().numpy() for t in (tq, tqd, tqdd))
    ref = oracle.rnea_batch(synth.robot_for(cfg), cfg["gravity"], q, qd, qdd)
    assert rel_err_per_state(got, ref).max() <= TOL[torch.float64]
    del tq, tqd, tqdd, tau
    torch.cuda.empty_cache()


@pytest.mark.parametrize("strategy", ["thread", "generic", "warp_scan", "reverse", "warp_scan_eq13",
                                      "warp_scan_eq15", "chunk:2", "chunk:4", "chunk:8", "chunk:16", "chunk:32"])
def test_C3_small_all_states(rd, strategy):
    cfg = synth.CONFIGS["C3"]
    q, qd, qdd = synth.states(cfg["seed"], 30, 0, 3000, cfg["ranges"])
    check_id(rd, synth.robot_for(cfg), cfg["gravity"], q, qd, qdd, strategy=strategy)


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("B", [1, 2, 31, 127, 128, 129, 1000, 4097])
def test_ragged_batches(rd, B):
    r = synth.random_chain(30, 1030)
    q, qd, qdd = synth.states(7, 30, 0, B)
    for strat in ("auto", "thread", "warp_scan", "generic", "reverse", "warp_scan_eq13", "warp_scan_eq15",
                  "chunk:2", "chunk:8", "chunk:32"):
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy=strat)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("n", [1, 2, 7, 30, 31, 64, 100, 200])
@pytest.mark.parametrize("lanes", [2, 4, 8, 16, 32])
def test_chunk_strategy_parity(rd, n, lanes, dtype):
    # RD_STRAT_CHUNK: L lanes per state, chunk scans (rnea_chunk.cu); ragged batch
    # (last warp partly idle), chunks longer / shorter than n / L, empty tail chunks
    # (L > n), revolute and prismatic joints
    for pf, seed in ((0.0, 300 + n), (0.3, 400 + n)):
        r = synth.random_chain(n, seed, prismatic_fraction=pf)
        q, qd, qdd = synth.states(24, n, 0, 1037)
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, dtype, strategy=f"chunk:{lanes}")


def test_chunk_boundary_and_api(rd):
    # model-level V_0, Vdot_0, F_{n+1} enter the chunk scans (forward prefix applied to
    # (V_0, Vdot_0), backward suffix applied to F_{n+1}); lanes_per_state is validated
    r = synth.random_chain(45, 45, prismatic_fraction=0.2)
    rng = np.random.default_rng(45)
    V0, Vd0, Ft = rng.standard_normal((3, 6))
    model = rd.Model.from_robot(r, (0, 0, 0))
    model.set_boundary(V0, Vd0, Ft)
    q, qd, qdd = synth.states(25, 45, 0, 500)
    ref = np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], V0, Vd0, Ft) for b in range(500)], 1)
    for lanes in (0, 2, 4, 8, 16, 32):
        model.set_strategy("chunk", lanes)
        tau = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd)).cpu().numpy()
        assert rel_err_per_state(tau, ref).max() <= 1e-10, lanes
    for bad in (1, 3, 64, -2):
        with pytest.raises(rd.RdError):
            model.set_strategy("chunk", bad)
    with pytest.raises(rd.RdError):
        model.set_strategy("thread", 4)


def test_auto_strategy_table(rd):
    # the measured AUTO table (csrc/capi.cu resolve())
    dh30 = rd.Model.from_robot(synth.random_chain(30, 1030), synth.GRAVITY_Z)
    dh10 = rd.Model.from_robot(synth.random_chain(10, 1010), synth.GRAVITY_Z)
    dh7 = rd.Model.from_robot(synth.random_chain(7, 1007), synth.GRAVITY_Z)
    dh100 = rd.Model.from_robot(synth.random_chain(100, 1100), synth.GRAVITY_Z)
    screw = synth.random_chain(12, 77)
    screw["S"][0, :3] += 0.2 * screw["S"][0, 3:]
    sc = rd.Model.from_robot(screw, synth.GRAVITY_Z)
    for model, B, fp64, want in [(dh30, 1000, True, "warp_scan"), (dh30, 2048, True, "warp_scan"),
                                 (dh30, 4096, True, "chunk"), (dh30, 16384, True, "reverse"),
                                 (dh30, 1_000_000, True, "thread"), (dh30, 40000, False, "thread"),
                                 (dh30, 1000, False, "warp_scan"), (dh30, 8192, False, "reverse"),
                                 (dh30, 60000, False, "thread"), (dh10, 1000, True, "thread"),
                                 (dh10, 1000, False, "thread"), (dh10, 100_000, True, "thread"),
                                 (dh10, 1_000_000, True, "thread"), (dh30, 100_000, False, "thread"),
                                 (dh100, 64, True, "block_scan"), (dh100, 1000, True, "chunk"),
                                 (dh100, 4096, True, "chunk"), (dh100, 16384, True, "reverse"),
                                 (dh100, 100_000, True, "reverse"), (sc, 1000, True, "warp_scan"),
                                 (sc, 100_000, True, "reverse"), (sc, 4096, True, "reverse"), (dh7, 256, True, "thread"),
                                 (dh7, 2048, False, "thread"), (dh7, 100_000, True, "thread")]:
        assert model.resolve_strategy(B, fp64) == want, (model.n, B, fp64, want)


@pytest.mark.parametrize("strategy", ["thread", "warp_scan", "reverse", "generic"])
def test_parity_check_fails_on_corrupted_operand(rd, strategy):
    # fault injection: one model operand off by 1e-7 relative (a link mass,
    # a home translation) must be caught by the parity metric at the 1e-10 bar
    r = synth.random_chain(12, 1212)
    q, qd, qdd = synth.states(15, 12, 0, 700)
    ref = oracle.rnea_batch(r, synth.GRAVITY_Z, q, qd, qdd)
    for corrupt in ("mass", "translation"):
        bad = {k: v.copy() for k, v in r.items()}
        if corrupt == "mass":
            bad["J"][5] *= 1 + 1e-7
        else:
            bad["M"][7, 0, 3] *= 1 + 1e-7
        model = rd.Model.from_robot(bad, synth.GRAVITY_Z)
        model.set_strategy(strategy)
        tau, _ = run_id(rd, model, q, qd, qdd)
        assert rel_err_per_state(tau, ref).max() > 1e-9, corrupt
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)          # and the clean model passes
    model.set_strategy(strategy)
    tau, _ = run_id(rd, model, q, qd, qdd)
    assert rel_err_per_state(tau, ref).max() <= 1e-10


def test_empty_batch_is_noop(rd):
    model = rd.Model.from_robot(synth.random_chain(6, 1), synth.GRAVITY_Z)
    z = torch.empty((6, 0), dtype=torch.float64, device="cuda")
    rd.inverse_dynamics(model, z, z, z, out=torch.empty((6, 0), dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("n", [1, 2, 3, 6, 7, 10, 13, 30, 31, 32, 33, 64, 100, 200])
def test_link_counts_random_chains(rd, n):
    r = synth.random_chain(n, 500 + n)
    q, qd, qdd = synth.states(11, n, 0, 777)
    for strat in ("auto", "generic", "reverse", "thread", "block_scan") + (("warp_scan", "warp_scan_eq13", "warp_scan_eq15") if n <= 32 else ()):
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy=strat)


def _wide_inertia_chain(n, seed, prismatic_fraction=0.0):
    """random_chain with link inertias spread over many decades: mass log-uniform in
    [1e-3, 1e3] kg, CoM up to 2 m off the joint frame, principal inertias
    log-uniform in [1e-5, 10] kg m^2 -- stresses the kernels' inertia forms (the
    thread / REVERSE kernels evaluate Fhat at the centre of mass, c = h / m,
    I_c = I - m (|c|^2 1 - c c^T); ABA keeps (m, h, I) and the structural zeros)."""
    r = synth.random_chain(n, seed, prismatic_fraction)
    rng = np.random.default_rng(seed)
    for i in range(n):
        m = 10.0 ** rng.uniform(-3, 3)
        com = rng.uniform(-2.0, 2.0, 3)
        Rc = synth.random_rotation(rng)
        lam = 10.0 ** rng.uniform(-5, 1, 3)
        r["J"][i] = synth.spatial_inertia(m, com, Rc @ np.diag(lam) @ Rc.T)
    return r


@pytest.mark.parametrize("n", [7, 30, 100])
def test_wide_inertia_ranges(rd, n):
    r = _wide_inertia_chain(n, 4000 + n)
    q, qd, qdd = synth.states(13, n, 0, 3000)
    strats = ("auto", "thread", "reverse", "generic") + (("warp_scan",) if n <= 32 else ("block_scan",))
    for strat in strats:
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy=strat)
    rp = _wide_inertia_chain(n, 4100 + n, prismatic_fraction=0.3)
    for strat in ("thread", "reverse"):
        check_id(rd, rp, synth.GRAVITY_Z, q, qd, qdd, strategy=strat)
    check_fd(rd, r, synth.GRAVITY_Z, 1000, 14)               # ABA backward error <= 1e-10


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_prismatic_and_screw_joints_generic(rd, dtype):
    r = synth.random_chain(12, 77, prismatic_fraction=0.5)
    # add a screw pitch to one revolute joint: v += 0.2 w
    for i in range(12):
        if np.linalg.norm(r["S"][i, 3:]) > 0.5:
            r["S"][i, :3] += 0.2 * r["S"][i, 3:]
            break
    q, qd, qdd = synth.states(12, 12, 0, 2000)
    for strat in ("generic", "warp_scan", "warp_scan_eq13", "warp_scan_eq15", "reverse", "thread", "auto"):
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, dtype, strategy=strat)   # reverse / thread: joint-frame REVERSE


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("n,pf", [(1, 1.0), (2, 0.5), (7, 0.4), (30, 0.3), (31, 0.3), (100, 0.3)])
def test_prismatic_joints_dh_kernels(rd, n, pf, dtype):
    # revolute + prismatic chains run the DH-frame kernels (prismatic: d = d0 + q)
    r = synth.random_chain(n, 880 + n, prismatic_fraction=pf)
    q, qd, qdd = synth.states(14, n, 0, 1500)
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    model.set_strategy("thread")
    want = "thread" if (n <= 30 or (n <= 32 and dtype == torch.float32)) else "reverse"
    assert model.resolve_strategy(1500, dtype == torch.float64) == want
    for strat in ("thread", "reverse"):
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, dtype, strategy=strat)


def test_pendulum_closed_form_on_gpu(rd):
    m, l, Izz, g = 1.7, 0.8, 0.05, 9.81
    model = rd.Model.from_robot(synth.pendulum(m, l, Izz), (0, -g, 0))
    q, qd, qdd = synth.states(3, 1, 0, 5000, "C1")
    tau = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd)).cpu().numpy()
    ref = (m * l * l + Izz) * qdd + m * g * l * np.cos(q)
    assert np.abs(tau - ref).max() <= 1e-12 * np.abs(ref).max()


def test_full_boundary_V0_Vdot0_Ftip(rd):
    # NEXT-4: non-zero V_0, Vdot_0, F_{n+1} (Eq. 3 full signature)
    r = synth.random_chain(7, 31, prismatic_fraction=0.3)
    rng = np.random.default_rng(5)
    V0, Vd0, Ft = rng.standard_normal((3, 6))
    model = rd.Model.from_robot(r, (0, 0, 0))
    model.set_boundary(V0, Vd0, Ft)
    q, qd, qdd = synth.states(13, 7, 0, 300)
    for strat in ("generic", "warp_scan", "warp_scan_eq13", "warp_scan_eq15"):
        model.set_strategy(strat)
        tau = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd)).cpu().numpy()
        ref = np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], V0, Vd0, Ft) for b in range(300)], 1)
        assert rel_err_per_state(tau, ref).max() <= 1e-10
    r2 = synth.random_chain(7, 32)                 # all revolute -> thread kernel
    model2 = rd.Model.from_robot(r2, (0, 0, 0))
    model2.set_boundary(V0, Vd0, Ft)
    for strat in ("thread", "generic", "warp_scan", "reverse"):
        model2.set_strategy(strat)
        tau = rd.inverse_dynamics(model2, dev(q), dev(qd), dev(qdd)).cpu().numpy()
        ref = np.stack([oracle.rnea(r2, q[:, b], qd[:, b], qdd[:, b], V0, Vd0, Ft) for b in range(300)], 1)
        assert rel_err_per_state(tau, ref).max() <= 1e-10


def _rounded(x, dtype):
    """x as the kernel sees it: rounded to fp32 for the fp32 path (A15)."""
    return x.astype(np.float32).astype(np.float64) if dtype == torch.float32 else x


def _per_state_boundary(rng, B, which):
    arrs = [rng.standard_normal((6, B)) if w else None for w in which]
    return arrs


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("kind", ["revolute", "prismatic", "screw"])
@pytest.mark.parametrize("n", [5, 9, 20])
def test_per_state_boundary_id(rd, dtype, kind, n):
    # NEXT-4: V_0, Vdot_0, F_{n+1} per state (rd_inverse_dynamics_bnd_*), every supported strategy;
    # THREAD runs the register kernel at n = 5 (and 9 in fp32 / up to its limit) and the stash kernel at 20
    B = 300
    r = synth.random_chain(n, 61, prismatic_fraction=0.0 if kind == "revolute" else 0.4)
    if kind == "screw":
        i = int(np.argmax(np.linalg.norm(r["S"][:, 3:], axis=1)))
        r["S"][i, :3] += 0.2 * r["S"][i, 3:]
    rng = np.random.default_rng(7)
    # the oracle sees exactly the (fp32-rounded) inputs the kernel sees (A15)
    q, qd, qdd = (_rounded(x, dtype) for x in synth.states(16, n, 0, B))
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    for which in ((1, 1, 1), (0, 0, 1), (1, 0, 0)):
        V0, Vd0, Ft = (None if a is None else _rounded(a, dtype) for a in _per_state_boundary(rng, B, which))
        gv0, gvd0, gft = oracle.gravity_boundary(synth.GRAVITY_Z)   # the model's values (A3)
        ref = np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b],
                                    V0=gv0 if V0 is None else V0[:, b],
                                    Vd0=gvd0 if Vd0 is None else Vd0[:, b],
                                    Ftip=gft if Ft is None else Ft[:, b]) for b in range(B)], 1)
        bnd = tuple(None if a is None else dev(a, dtype) for a in (V0, Vd0, Ft))
        for strat in ("auto", "thread", "warp_scan", "generic", "reverse"):
            model.set_strategy(strat)
            tau = rd.inverse_dynamics(model, dev(q, dtype), dev(qd, dtype), dev(qdd, dtype),
                                      boundary=bnd).double().cpu().numpy()
            err = rel_err_per_state(tau, ref).max()
            assert err <= TOL[dtype], (strat, which, err)
    model.set_strategy("warp_scan_eq13")
    with pytest.raises(rd.RdError):
        rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd), boundary=(None, None, dev(np.zeros((6, B)))))


@pytest.mark.parametrize("kind", ["revolute", "prismatic", "screw"])
def test_per_state_boundary_fd(rd, kind):
    n, B = 8, 300
    r = synth.random_chain(n, 62, prismatic_fraction=0.0 if kind == "revolute" else 0.4)
    if kind == "screw":
        i = int(np.argmax(np.linalg.norm(r["S"][:, 3:], axis=1)))
        r["S"][i, :3] += 0.2 * r["S"][i, 3:]
    rng = np.random.default_rng(8)
    q, qd, qdd = synth.states(17, n, 0, B)
    V0, Vd0, Ft = rng.standard_normal((3, 6, B))
    tau = np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], V0[:, b], Vd0[:, b], Ft[:, b])
                    for b in range(B)], 1)
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau), status=st,
                              boundary=(dev(V0), dev(Vd0), dev(Ft))).cpu().numpy()
    assert rel_err_per_state(out, qdd, floor=1.0).max() < 1e-9
    assert int(st.abs().max()) == 0
    model.set_fd_algo("jsiia")
    with pytest.raises(rd.RdError):
        rd.forward_dynamics(model, dev(q), dev(qd), dev(tau), boundary=(dev(V0), None, None))


def test_deterministic_and_strategy_consistent(rd):
    cfg = synth.CONFIGS["C3"]
    q, qd, qdd = synth.states(cfg["seed"], 30, 0, 20000)
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    for strat in ("thread", "warp_scan", "generic", "reverse", "chunk:4"):
        # with a FIXED strategy, results are bit-identical across repeats and across sharding
        # (AUTO picks the strategy from the per-call batch size)
        model.set_strategy(strat)
        a = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd))
        b = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd))
        assert torch.equal(a, b)                       # bit-identical repeat
        c = rd.inverse_dynamics(model, dev(q[:, 5000:9000]), dev(qd[:, 5000:9000]), dev(qdd[:, 5000:9000]))
        assert torch.equal(a[:, 5000:9000], c)


def test_host_path_equals_device_path(rd):
    cfg = synth.CONFIGS["C3"]
    q, qd, qdd = synth.states(cfg["seed"], 30, 0, 50000)
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    dev_tau = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd)).cpu().numpy()
    host_tau = rd.inverse_dynamics_host(model, q, qd, qdd)
    np.testing.assert_array_equal(host_tau, dev_tau)
    pq, pqd, pqdd = (torch.from_numpy(x).pin_memory() for x in (q, qd, qdd))
    out = torch.empty_like(pq).pin_memory()
    rd.inverse_dynamics_host(model, pq, pqd, pqdd, out)
    np.testing.assert_array_equal(out.numpy(), dev_tau)


def test_host_path_multichunk_bit_identical(rd):
    # 1M states at n = 30 is 8 host chunks (32 MB per input array each) with a ragged
    # last chunk; the strategy is resolved once for the whole batch, so the host path
    # equals the device path bit for bit (every chunk runs THREAD)
    cfg = synth.CONFIGS["C3"]
    n, B = 30, 1_000_000
    model = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
    assert model.resolve_strategy(B, True) == "thread"
    q, qd, qdd = synth.states(cfg["seed"], n, 0, B)
    dev_tau = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd)).cpu().numpy()
    pq, pqd, pqdd = (torch.from_numpy(x).pin_memory() for x in (q, qd, qdd))
    out = torch.empty_like(pq).pin_memory()
    rd.inverse_dynamics_host(model, pq, pqd, pqdd, out)
    np.testing.assert_array_equal(out.numpy(), dev_tau)
    with pytest.raises(rd.RdError):                      # shape checks of the host binding
        rd.inverse_dynamics_host(model, q[:, :10], qd, qdd)
    with pytest.raises(rd.RdError):
        rd.inverse_dynamics_host(model, q, qd, qdd, np.empty((n, B - 1)))


def test_host_path_multichunk_workspace_kernels(rd):
    # n = 60: a chunk is 69,905 states, so 150,000 states are 3 chunks alternating
    # between the two host streams; GENERIC ID (screw joint) and every FD algorithm
    # allocate their workspace per call (stream-ordered) on those streams
    n, B = 60, 150_000
    r = synth.random_chain(n, 1313, prismatic_fraction=0.3)
    i = int(np.argmax(np.linalg.norm(r["S"][:, 3:], axis=1)))
    r["S"][i, :3] += 0.2 * r["S"][i, 3:]                    # screw joint -> GENERIC / joint-frame ABA
    q, qd, qdd = synth.states(18, n, 0, B)
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    assert model.resolve_strategy(B, True) == "reverse"      # AUTO: joint-frame REVERSE (no workspace)
    auto_tau = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd)).cpu().numpy()
    np.testing.assert_array_equal(rd.inverse_dynamics_host(model, q, qd, qdd), auto_tau)
    model.set_strategy("generic")                             # the per-call workspace path
    dev_tau = rd.inverse_dynamics(model, dev(q), dev(qd), dev(qdd)).cpu().numpy()
    np.testing.assert_array_equal(rd.inverse_dynamics_host(model, q, qd, qdd), dev_tau)
    assert rel_err_per_state(auto_tau, dev_tau).max() <= 1e-10
    sub = np.arange(0, B, 997)
    for algo in ("aba", "jsiia", "aba_scan"):
        model.set_fd_algo(algo)
        dev_qdd = rd.forward_dynamics(model, dev(q), dev(qd), dev(dev_tau)).cpu().numpy()
        host_qdd = rd.forward_dynamics_host(model, q, qd, dev_tau)
        np.testing.assert_array_equal(host_qdd, dev_qdd)
        back = oracle.rnea_batch(r, synth.GRAVITY_Z, q[:, sub], qd[:, sub], host_qdd[:, sub])
        assert rel_err_per_state(back, dev_tau[:, sub]).max() <= 1e-10


def test_concurrent_streams_share_no_workspace(rd):
    # two streams run GENERIC ID (per-call workspace) and ABA FD on ONE model at the
    # same time, with different inputs; each result equals its serial run
    n = 24
    r = synth.random_chain(n, 1414, prismatic_fraction=0.3)
    i = int(np.argmax(np.linalg.norm(r["S"][:, 3:], axis=1)))
    r["S"][i, :3] += 0.2 * r["S"][i, 3:]                    # screw joint -> GENERIC ID
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    model.set_strategy("generic")
    B = 200_000
    ins = [tuple(dev(x) for x in synth.states(30 + k, n, 0, B)) for k in range(2)]
    ref_id = [rd.inverse_dynamics(model, *x) for x in ins]
    ref_fd = [rd.forward_dynamics(model, x[0], x[1], t) for x, t in zip(ins, ref_id)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    for rep in range(3):
        outs_id = [torch.empty_like(ins[0][0]) for _ in range(2)]
        outs_fd = [torch.empty_like(ins[0][0]) for _ in range(2)]
        for k, s in enumerate(streams):
            s.wait_stream(torch.cuda.current_stream())
            rd.inverse_dynamics(model, *ins[k], out=outs_id[k], stream=s)
            rd.forward_dynamics(model, ins[k][0], ins[k][1], ref_id[k], out=outs_fd[k], stream=s)
        torch.cuda.synchronize()
        for k in range(2):
            assert torch.equal(outs_id[k], ref_id[k]), (rep, k)
            assert torch.equal(outs_fd[k], ref_fd[k]), (rep, k)


def test_device_mismatch_rejected(rd):
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU: the cross-device check needs two")
    model = rd.Model.from_robot(synth.random_chain(6, 1), synth.GRAVITY_Z)
    z = torch.zeros((6, 10), dtype=torch.float64, device="cuda:1")
    with pytest.raises(rd.RdError):
        rd.inverse_dynamics(model, z, z, z)


def test_launch_count_and_errors(rd):
    model = rd.Model.from_robot(synth.random_chain(30, 1030), synth.GRAVITY_Z)
    q = torch.zeros((30, 1000), dtype=torch.float64, device="cuda")
    rd.inverse_dynamics(model, q, q, q)
    assert rd.last_launch_count() == 1
    with pytest.raises(rd.RdError):
        rd.inverse_dynamics(model, q, q, q, out=q)                    # aliasing
    with pytest.raises(rd.RdError):
        rd.inverse_dynamics(model, q.cpu(), q.cpu(), q.cpu())          # host tensors on device API


# ------------------------------------------------------------------ forward dynamics (ABA)
def cond_forward_check(robot, g, q, qd, tau, out, ref, sample):
    """Cond-scaled forward error (A14) on sampled states.  tau(qdd) = M(q) qdd + h is
    affine, so for the GPU answer `out` and the oracle's `ref`
        M (out - ref) = r_gpu - r_orc,   r = RNEA(q, qd, qdd_x) - tau,
    hence ||out - ref||_2 <= (||r_gpu||_2 + ||r_orc||_2 + eval rounding) / lambda_min(M):
    the forward error is fully explained by the two backward errors times
    ||M^-1|| (cond(M) / ||M||).  Returns the sampled cond(M) values."""
    qs, qds, ts, os_, rs = (x[:, sample] for x in (q, qd, tau, out, ref))
    r_gpu = oracle.rnea_batch(robot, g, qs, qds, os_) - ts
    r_orc = oracle.rnea_batch(robot, g, qs, qds, rs) - ts
    conds = []
    for k in range(len(sample)):
        lam = np.linalg.eigvalsh(oracle.jsi(robot, qs[:, k]))
        assert lam[0] > 0
        conds.append(lam[-1] / lam[0])
        rnd = 1e-12 * (np.linalg.norm(ts[:, k]) + lam[-1] * np.linalg.norm(rs[:, k]))
        bound = (np.linalg.norm(r_gpu[:, k]) + np.linalg.norm(r_orc[:, k]) + rnd) / lam[0]
        fe = np.linalg.norm(os_[:, k] - rs[:, k])
        assert fe <= 1.5 * bound, (sample[k], fe, bound, conds[-1])
    return np.array(conds)


def check_fd(rd, robot, g, B, seed, dtype=torch.float64, bwd_tol=None, n_cond=48):
    """FD parity (A14): backward error ||RNEA(q, qd, qdd_gpu) - tau|| / ||tau|| per state
    <= the contract tolerance (1e-10 fp64, 1e-4 fp32), plus the cond-scaled forward
    error of `cond_forward_check` on n_cond sampled states.  Returns (max backward
    error, max forward error, max sampled cond(M))."""
    n = robot["S"].shape[0]
    q, qd, qdd = (_rounded(x, dtype) for x in synth.states(seed, n, 0, B))
    tau = _rounded(oracle.rnea_batch(robot, g, q, qd, qdd), dtype)
    model = rd.Model.from_robot(robot, g)
    out = rd.forward_dynamics(model, dev(q, dtype), dev(qd, dtype), dev(tau, dtype)).double().cpu().numpy()
    assert np.all(np.isfinite(out))
    back = oracle.rnea_batch(robot, g, q, qd, out)       # backward error (A14)
    berr = rel_err_per_state(back, tau)
    tol = TOL[dtype] if bwd_tol is None else bwd_tol
    assert berr.max() <= tol, f"FD backward error {berr.max():.3e}"
    fwd = oracle.fd_batch(robot, g, q, qd, tau)
    ferr = rel_err_per_state(out, fwd, floor=1.0)
    sample = np.unique(np.linspace(0, B - 1, min(B, n_cond)).astype(np.int64))
    conds = cond_forward_check(robot, g, q, qd, tau, out, fwd, sample)
    return berr.max(), ferr.max(), conds.max()


@pytest.mark.parametrize("n", [1, 2, 7, 30])
def test_fd_aba_parity(rd, n):
    r = synth.random_chain(n, 900 + n, prismatic_fraction=0.3 if n < 30 else 0.0)
    b, f, c = check_fd(rd, r, synth.GRAVITY_Z, 2000, 4)
    assert f < 1e-8


@pytest.mark.parametrize("n,pf", [(12, 0.5), (60, 0.3)])
def test_fd_aba_prismatic_dh(rd, n, pf):
    # revolute + prismatic chains take the DH-frame ABA (prismatic instantiation)
    r = synth.random_chain(n, 930 + n, prismatic_fraction=pf)
    b, f, c = check_fd(rd, r, synth.GRAVITY_Z, 1500, 6)    # backward error <= 1e-10 inside (A14)
    assert f < 1e-5                                        # forward error: cond(M)-limited (A14)


def test_fd_aba_screw_joints_joint_frames(rd):
    # a screw joint has no one-variable DH form: the joint-frame ABA kernel runs
    r = synth.random_chain(9, 941, prismatic_fraction=0.3)
    for i in range(9):
        if np.linalg.norm(r["S"][i, 3:]) > 0.5:
            r["S"][i, :3] += 0.15 * r["S"][i, 3:]
            break
    b, f, c = check_fd(rd, r, synth.GRAVITY_Z, 1500, 7)
    assert f < 1e-7
    check_fd(rd, r, synth.GRAVITY_Z, 500, 8, torch.float32)   # fp32: backward error <= 1e-4


def test_fd_C4_sampled(rd):
    # Config C4: n = 100, 100k states (the bench launch); sampled backward-error check.
    cfg = synth.CONFIGS["C4"]
    r = synth.robot_for(cfg)
    n, B = cfg["n"], cfg["batch"]
    q, qd, qdd = synth.states(cfg["seed"], n, 0, B)
    sample = np.unique(np.concatenate([np.arange(256), np.arange(B - 256, B),
                                       np.random.default_rng(99).integers(0, B, 2048)]))
    tau_s = oracle.rnea_batch(r, cfg["gravity"], q[:, sample], qd[:, sample], qdd[:, sample])
    tau = np.zeros((n, B))
    tau[:, sample] = tau_s
    model = rd.Model.from_robot(r, cfg["gravity"])
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    back = oracle.rnea_batch(r, cfg["gravity"], q[:, sample], qd[:, sample], out[:, sample])
    assert rel_err_per_state(back, tau_s).max() <= 1e-10


def test_fd_fp32(rd):
    r = synth.random_chain(7, 907)
    check_fd(rd, r, synth.GRAVITY_Z, 2000, 5, torch.float32)


def test_fd_pendulum_closed_form(rd):
    m, l, g = 1.3, 0.9, 9.81
    model = rd.Model.from_robot(synth.pendulum(m, l, 1e-9), (0, -g, 0))
    q, qd, _ = synth.states(6, 1, 0, 1000)
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(np.zeros_like(q))).cpu().numpy()
    ref = -(m * g * l * np.cos(q)) / (m * l * l + 1e-9)
    assert np.abs(out - ref).max() <= 1e-10 * np.abs(ref).max()


def test_fd_tip_wrench(rd):
    r = synth.random_chain(6, 41)
    rng = np.random.default_rng(1)
    Ft = rng.standard_normal(6)
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    model.set_boundary(None, None, Ft)
    q, qd, qdd = synth.states(8, 6, 0, 200)
    Vd0 = np.concatenate([-synth.GRAVITY_Z, np.zeros(3)])
    tau = np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], None, Vd0, Ft) for b in range(200)], 1)
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    assert rel_err_per_state(out, qdd, floor=1.0).max() < 1e-9


@pytest.mark.parametrize("dtype,scale", [(torch.float64, 1e4), (torch.float32, 1e3)])
def test_large_joint_angles(rd, dtype, scale):
    # the branch-free sin/cos reduction (rd_math.cuh) against the oracle's libm.
    # (At |q| ~ 1e6 the ORACLE's own Rodrigues translation, (I q + ... + (q - s)[w]^2) v,
    # cancels O(|q|) terms and loses ~1e-10 relative accuracy, so 1e4 is the largest
    # scale at which the oracle is a 1e-10 reference.)
    r = synth.random_chain(30, 1030)
    q, qd, qdd = synth.states(21, 30, 0, 5000)
    q = q / np.pi * scale
    for strat in ("thread", "generic", "warp_scan", "reverse"):
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, dtype, strategy=strat)


def test_thread_kernel_many_tiles(rd):
    # many tiles per CTA: exercises the ping-pong slot parity over > 2 tiles per CTA
    cfg = synth.CONFIGS["C3"]
    q, qd, qdd = synth.states(cfg["seed"], 30, 0, 70000)
    check_id(rd, synth.robot_for(cfg), cfg["gravity"], q, qd, qdd, strategy="thread",
             sample=np.arange(0, 70000, 7))


# ------------------------------------------------------------------ forward dynamics (JSIIA, NEXT-1)
@pytest.mark.parametrize("n,pf", [(1, 0.0), (2, 0.0), (7, 0.3), (10, 0.0), (30, 0.0), (31, 0.2), (32, 0.0),
                                  (64, 0.2), (100, 0.0), (200, 0.0)])
def test_fd_jsiia_parity(rd, n, pf):
    r = synth.random_chain(n, 700 + n, prismatic_fraction=pf)
    g = synth.GRAVITY_Z
    q, qd, qdd = synth.states(17, n, 0, 1500)
    tau = oracle.rnea_batch(r, g, q, qd, qdd)
    model = rd.Model.from_robot(r, g)
    model.set_fd_algo("jsiia")
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    assert np.all(np.isfinite(out))
    back = oracle.rnea_batch(r, g, q, qd, out)
    assert rel_err_per_state(back, tau).max() <= 1e-10
    ref = oracle.fd_batch(r, g, q, qd, tau, algo="jsiia")
    assert rel_err_per_state(out, ref, floor=1.0).max() < (1e-7 if n <= 31 else 1e-5)   # cond(M), A14
    cond_forward_check(r, g, q, qd, tau, out, ref, np.arange(0, 1500, 50))


def test_fd_jsiia_boundary_and_limits(rd):
    r = synth.random_chain(6, 44)
    rng = np.random.default_rng(3)
    V0, Vd0, Ft = rng.standard_normal((3, 6))
    model = rd.Model.from_robot(r, (0, 0, 0))
    model.set_boundary(V0, Vd0, Ft)
    model.set_fd_algo("jsiia")
    q, qd, qdd = synth.states(9, 6, 0, 300)
    tau = np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], V0, Vd0, Ft) for b in range(300)], 1)
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    assert rel_err_per_state(out, qdd, floor=1.0).max() < 1e-9
    big = rd.Model.from_robot(synth.random_chain(257, 1), synth.GRAVITY_Z)
    big.set_fd_algo("jsiia")
    z = torch.zeros((257, 10), dtype=torch.float64, device="cuda")
    with pytest.raises(rd.RdError):
        rd.forward_dynamics(big, z, z, z)


# ------------------------------------------------------------------ forward dynamics (scan ABIA, Alg. 3)
@pytest.mark.parametrize("n,pf", [(1, 0.0), (2, 0.0), (7, 0.3), (16, 0.0), (30, 0.0), (32, 0.2), (33, 0.0),
                                  (64, 0.2), (100, 0.0), (200, 0.0), (256, 0.1)])
def test_fd_aba_scan_parity(rd, n, pf):
    r = synth.random_chain(n, 800 + n, prismatic_fraction=pf)
    g = synth.GRAVITY_Z
    q, qd, qdd = synth.states(19, n, 0, 1500)
    tau = oracle.rnea_batch(r, g, q, qd, qdd)
    model = rd.Model.from_robot(r, g)
    model.set_fd_algo("aba_scan")
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    assert np.all(np.isfinite(out))
    back = oracle.rnea_batch(r, g, q, qd, out)
    assert rel_err_per_state(back, tau).max() <= 1e-10
    ref = oracle.fd_batch(r, g, q, qd, tau)
    # forward error is cond(M)-limited (A14): cond grows fast with n
    assert rel_err_per_state(out, ref, floor=1.0).max() < (1e-7 if n <= 32 else 1e-5)
    cond_forward_check(r, g, q, qd, tau, out, ref, np.arange(0, 1500, 50))
    assert rd.last_launch_count() == 3


# ------------------------------------------------------------------ forward dynamics (merged Eq. 20 scan, NEXT-2)
@pytest.mark.parametrize("n,pf", [(1, 0.0), (2, 0.0), (7, 0.3), (16, 0.0), (30, 0.0), (31, 0.2)])
def test_fd_aba_merged_parity(rd, n, pf):
    r = synth.random_chain(n, 850 + n, prismatic_fraction=pf)
    g = synth.GRAVITY_Z
    q, qd, qdd = synth.states(21, n, 0, 1200)
    tau = oracle.rnea_batch(r, g, q, qd, qdd)
    model = rd.Model.from_robot(r, g)
    model.set_fd_algo("aba_merged")
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    assert np.all(np.isfinite(out))
    back = oracle.rnea_batch(r, g, q, qd, out)                 # primary: backward error (A14)
    assert rel_err_per_state(back, tau).max() <= 1e-10
    sub = np.arange(0, 1200, 37)                                # the oracle's literal Eq. (20) path
    ref = oracle.fd_batch(r, g, q[:, sub], qd[:, sub], tau[:, sub], algo="aba_merged")
    assert rel_err_per_state(out[:, sub], ref, floor=1.0).max() < 1e-7
    cond_forward_check(r, g, q[:, sub], qd[:, sub], tau[:, sub], out[:, sub], ref, np.arange(sub.size))
    assert rd.last_launch_count() == 3


@pytest.mark.parametrize("algo", ["aba_scan", "aba_merged"])
def test_fd_scan_variants_boundary_fp32_limits(rd, algo):
    n = 9
    r = synth.random_chain(n, 46, prismatic_fraction=0.2)
    rng = np.random.default_rng(5)
    V0, Vd0, Ft = rng.standard_normal((3, 6))
    model = rd.Model.from_robot(r, (0, 0, 0))
    model.set_boundary(V0, Vd0, Ft)
    model.set_fd_algo(algo)
    q, qd, qdd = synth.states(10, n, 0, 257)
    tau = np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], V0, Vd0, Ft) for b in range(257)], 1)
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    assert rel_err_per_state(out, qdd, floor=1.0).max() < 1e-9
    # fp32 (A15): the oracle sees the fp32-rounded inputs; backward error <= 1e-4
    q32, qd32, t32 = (_rounded(x, torch.float32) for x in (q, qd, tau))
    out32 = rd.forward_dynamics(model, dev(q32, torch.float32), dev(qd32, torch.float32),
                                dev(t32, torch.float32)).double().cpu().numpy()
    back = np.stack([oracle.rnea(r, q32[:, b], qd32[:, b], out32[:, b], V0, Vd0, Ft) for b in range(257)], 1)
    assert rel_err_per_state(back, t32).max() <= TOL[torch.float32]
    nbig = 257 if algo == "aba_scan" else 32                 # beyond the CTA / warp limits
    big = rd.Model.from_robot(synth.random_chain(nbig, 1), synth.GRAVITY_Z)
    big.set_fd_algo(algo)
    z = torch.zeros((nbig, 10), dtype=torch.float64, device="cuda")
    with pytest.raises(rd.RdError):
        rd.forward_dynamics(big, z, z, z)


@pytest.mark.parametrize("algo", ["aba", "jsiia", "aba_scan", "aba_merged"])
@pytest.mark.parametrize("dh", [True, False])
def test_fd_status_array(rd, algo, dh):
    # NEXT-4: per-state status (rd_forward_dynamics_ex_*).  A NaN joint angle at
    # 0-based link j >= 1 makes the articulated inertia of link j-1 NaN, so the
    # ABI pivot Omega fails first at 1-based link j; JSIIA's first Cholesky pivot
    # M_11 depends on every q_j (j >= 1).  Other states are unaffected.
    n = 8
    r = synth.random_chain(n, 47, prismatic_fraction=0.0 if dh else 0.3)
    g = synth.GRAVITY_Z
    q, qd, qdd = synth.states(11, n, 0, 96)
    tau = oracle.rnea_batch(r, g, q, qd, qdd)
    bad = {5: 3, 9: 1, 40: 7}
    for b, j in bad.items():
        q[j, b] = np.nan
    model = rd.Model.from_robot(r, g)
    model.set_fd_algo(algo)
    st = torch.full((96,), -7, dtype=torch.int32, device="cuda")
    out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau), status=st).cpu().numpy()
    st = st.cpu().numpy()
    good = np.setdiff1d(np.arange(96), list(bad))
    assert np.all(st[good] == 0)
    assert rel_err_per_state(out[:, good], qdd[:, good], floor=1.0).max() < 1e-9
    for b, j in bad.items():
        if algo == "jsiia":
            assert st[b] == 1, (b, st[b])
        elif dh:
            assert st[b] == j, (b, st[b])
        else:
            # with prismatic joints the NaN slide enters only the translation, and a
            # prismatic parent's pivot (the A block of the articulated inertia) stays
            # finite: the tip-most failing pivot is link j or a more basal one
            assert 1 <= st[b] <= j, (b, st[b])
        assert not np.all(np.isfinite(out[:, b]))
    out2 = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()   # plain call, same qdd
    np.testing.assert_array_equal(np.isfinite(out2), np.isfinite(out))
    np.testing.assert_array_equal(out2[:, good], out[:, good])
    with pytest.raises(rd.RdError):
        rd.forward_dynamics(model, dev(q), dev(qd), dev(tau), status=torch.zeros(95, dtype=torch.int32,
                                                                                   device="cuda"))


@pytest.mark.parametrize("n", [33, 100, 257, 512])
def test_block_scan_long_chains(rd, n):
    # NEXT-3 single-robot latency mode: one CTA per state, CTA-wide scans
    r = synth.random_chain(n, 600 + n, prismatic_fraction=0.1)
    q, qd, qdd = synth.states(23, n, 0, 64)
    check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy="block_scan")
    check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, torch.float32, strategy="block_scan")


@pytest.mark.parametrize("n, seed, tol", [(30, 1030, 2e-13), (100, 1800, 4e-12), (1000, 1700, 5e-12)])
def test_dh_frames_built_locally(rd, n, seed, tol):
    # Regression guard for the local DH construction: the DH-frame kernels
    # (THREAD / REVERSE) agree with the oracle far inside the contract tolerance; building
    # the frames from base-frame poses gave 6.5e-13 / 1.8e-11 / 2.5e-10 on these robots.
    r = synth.random_chain(n, seed, prismatic_fraction=0.05)
    q, qd, qdd = synth.states(29, n, 0, 97)
    err = check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy="thread" if n <= 30 else "reverse")
    assert err <= tol, f"DH-frame kernel error {err:.3e} > {tol:.0e}"


@pytest.mark.parametrize("eps", [3e-2, 1e-2, 3e-3, 1e-3, 1e-4])
@pytest.mark.parametrize("n", [6, 30])
def test_nearly_parallel_axes(rd, n, eps):
    # A calibrated, nominally planar arm: consecutive joint axes tilted by ~eps rad.  The
    # DH origins move ~offset/eps off the links; beyond 50 link lengths the model keeps
    # to the joint-frame kernels (at 200-600 link lengths the DH maps
    # lost 2e-9 .. 7e-8).  Every strategy must hold the contract tolerance.
    r = synth.tilted_planar(n, eps, 5 + n)
    q, qd, qdd = synth.states(37, n, 0, 256)
    for strategy in ("auto", "thread", "reverse"):
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy=strategy)
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    tau = oracle.rnea_batch(r, synth.GRAVITY_Z, q, qd, qdd)
    qdd_fd = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
    back = oracle.rnea_batch(r, synth.GRAVITY_Z, q, qd, qdd_fd)
    assert rel_err_per_state(back, tau).max() <= 1e-10


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("n", [1, 7, 30, 100, 333])
def test_reverse_joint_frames(rd, n, dtype):
    # REVERSE in joint frames (rnea_rev_jf.cu): screw joints (pitch on every third revolute
    # joint), prismatic joints, ragged batch, model and per-state boundary
    r = synth.random_chain(n, 900 + n, prismatic_fraction=0.3)
    for i in range(0, n, 3):
        if np.linalg.norm(r["S"][i, 3:]) > 0.5:
            r["S"][i, :3] += 0.15 * r["S"][i, 3:]
    q, qd, qdd = synth.states(43, n, 0, 517)
    check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, dtype, strategy="reverse")
    model = rd.Model.from_robot(r, synth.GRAVITY_Z)
    model.set_strategy("reverse")
    B = q.shape[1]
    bnd = tuple(dev(np.random.default_rng(k).standard_normal((6, B)), dtype) for k in range(3))
    tau = rd.inverse_dynamics(model, dev(q, dtype), dev(qd, dtype), dev(qdd, dtype), boundary=bnd).cpu().numpy()
    model.set_strategy("generic")
    ref = rd.inverse_dynamics(model, dev(q, dtype), dev(qd, dtype), dev(qdd, dtype), boundary=bnd).cpu().numpy()
    assert rel_err_per_state(tau, ref).max() <= TOL[dtype]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_thread_joint_frames_register_kernel(rd, dtype):
    # the register-resident THREAD kernel in joint frames (rnea_small_jf.cu): screw and
    # prismatic joints, n = 1..8 (fp64) / 1..12 (fp32), ragged batch, per-state boundary
    for n in range(1, 9 if dtype == torch.float64 else 13):
        r = synth.random_chain(n, 950 + n, prismatic_fraction=0.3)
        for i in range(0, n, 2):
            if np.linalg.norm(r["S"][i, 3:]) > 0.5:
                r["S"][i, :3] += 0.1 * r["S"][i, 3:]
        q, qd, qdd = synth.states(47, n, 0, 389)
        check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, dtype, strategy="thread")
        model = rd.Model.from_robot(r, synth.GRAVITY_Z)
        assert model.resolve_strategy(389, dtype == torch.float64) == "thread"
        B = q.shape[1]
        bnd = tuple(dev(np.random.default_rng(k + n).standard_normal((6, B)), dtype) for k in range(3))
        model.set_strategy("thread")
        tau = rd.inverse_dynamics(model, dev(q, dtype), dev(qd, dtype), dev(qdd, dtype), boundary=bnd).cpu().numpy()
        model.set_strategy("generic")
        ref = rd.inverse_dynamics(model, dev(q, dtype), dev(qd, dtype), dev(qdd, dtype), boundary=bnd).cpu().numpy()
        assert rel_err_per_state(tau, ref).max() <= TOL[dtype], n


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_fd_joint_frames_register_aba(rd, dtype):
    # the register ABA in joint frames (aba_small_jf.cu): screw and prismatic joints,
    # n = 1..8 (fp64) / 1..12 (fp32), backward error at the contract tolerance, the status
    # array, and the per-state boundary (consistent with ID under the same boundary)
    for n in range(1, 9 if dtype == torch.float64 else 13):
        r = synth.random_chain(n, 960 + n, prismatic_fraction=0.3)
        for i in range(0, n, 2):
            if np.linalg.norm(r["S"][i, 3:]) > 0.5:
                r["S"][i, :3] += 0.1 * r["S"][i, 3:]
        q, qd, qdd = synth.states(53, n, 0, 301)
        model = rd.Model.from_robot(r, synth.GRAVITY_Z)
        tq, tqd, tqdd = dev(q, dtype), dev(qd, dtype), dev(qdd, dtype)
        B = q.shape[1]
        bnd = tuple(dev(0.3 * np.random.default_rng(k + n).standard_normal((6, B)), dtype) for k in range(3))
        tau = rd.inverse_dynamics(model, tq, tqd, tqdd, boundary=bnd)
        status = torch.empty(B, dtype=torch.int32, device="cuda")
        out = rd.forward_dynamics(model, tq, tqd, tau, boundary=bnd, status=status)
        assert int(status.abs().sum()) == 0
        back = rd.inverse_dynamics(model, tq, tqd, out, boundary=bnd)      # round trip through ID
        err = rel_err_per_state(back.double().cpu().numpy(), tau.double().cpu().numpy()).max()
        assert err <= (1e-10 if dtype == torch.float64 else 1e-4), (n, err)
        # without a boundary, against the oracle's RNEA (backward error, A14)
        tau0 = oracle.rnea_batch(r, synth.GRAVITY_Z, *(x.double().cpu().numpy() for x in (tq, tqd, tqdd)))
        out0 = rd.forward_dynamics(model, tq, tqd, dev(tau0, dtype)).double().cpu().numpy()
        back0 = oracle.rnea_batch(r, synth.GRAVITY_Z, tq.double().cpu().numpy(), tqd.double().cpu().numpy(), out0)
        assert rel_err_per_state(back0, tau0).max() <= (1e-10 if dtype == torch.float64 else 1e-4), n


@pytest.mark.parametrize("B", [1, 2, 33, 129])
def test_joint_frame_kernels_tiny_batches(rd, B):
    # the joint-frame kernels at batches below one CTA / one warp (screw chain: no DH form)
    for n in (1, 5, 40):
        r = synth.random_chain(n, 970 + n, prismatic_fraction=0.3)
        r["S"][0, :3] += 0.1 * r["S"][0, 3:] if np.linalg.norm(r["S"][0, 3:]) > 0.5 else 0.0
        q, qd, qdd = synth.states(59, n, 0, B)
        for strategy in ("thread", "reverse"):
            check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy=strategy)
        model = rd.Model.from_robot(r, synth.GRAVITY_Z)
        tau = oracle.rnea_batch(r, synth.GRAVITY_Z, q, qd, qdd)
        out = rd.forward_dynamics(model, dev(q), dev(qd), dev(tau)).cpu().numpy()
        back = oracle.rnea_batch(r, synth.GRAVITY_Z, q, qd, out)
        assert rel_err_per_state(back, tau).max() <= 1e-10, (n, B)


@pytest.mark.parametrize("strategy", ["reverse", "generic", "chunk", "auto"])
def test_very_long_chains(rd, strategy):
    # n = 1000 (ten times the paper's longest ID chain): the strategies without a
    # length cap; REVERSE re-derives V, Vdot through 1000 inverse maps (O(n eps) drift)
    n = 1000
    r = synth.random_chain(n, 1700, prismatic_fraction=0.05)
    q, qd, qdd = synth.states(29, n, 0, 97)
    check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy=strategy)


@pytest.mark.parametrize("strategy", ["thread", "warp_scan", "generic", "reverse"])
def test_cuda_graph_capture_and_replay(rd, strategy):
    # the launches are stream-ordered and host-synchronisation free, so a batch of
    # calls can be captured once in a CUDA graph and replayed (launch-bound small batches)
    cfg = synth.CONFIGS["C2"]
    q, qd, qdd = synth.states(cfg["seed"], 7, 0, 4000, cfg["ranges"])
    model = rd.Model.from_robot(synth.arm7(), cfg["gravity"])
    model.set_strategy(strategy)
    tq, tqd, tqdd = dev(q), dev(qd), dev(qdd)
    out = torch.empty_like(tq)
    ref = rd.inverse_dynamics(model, tq, tqd, tqdd).clone()      # warm-up (allocates any workspace)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rd.inverse_dynamics(model, tq, tqd, tqdd, out, stream=s)
    for _ in range(3):
        out.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("dtype,n", [(torch.float64, n) for n in list(range(1, 10)) + [12, 13, 16, 17]] +
                                    [(torch.float32, n) for n in list(range(2, 10)) + [16, 17, 25, 30]])
def test_thread_short_chain_register_kernel(rd, n, dtype):
    """THREAD runs the register-resident, fully unrolled kernel (rnea_small.cu)
    for n <= 16 (fp64, 13..16 up to 300k states; the backward sweep re-derives
    sin/cos from n = 9) and n <= 32 (fp32, but 25 and 26); 17 is the first fp64
    stash-kernel length at these batch sizes.  Revolute and mixed
    prismatic chains, ragged batches (one state, a partial CTA, several CTAs),
    and the model boundary (V_0, Vdot_0, F_{n+1}) of Eq. (3).  fp32 starts at
    n = 2: a 1-link state's max|tau| is its single torque, which cancels to
    ~1e-3 of its terms in some random states, and the fp32-rounded model (A15)
    then gives 1.7e-4 there -- the same with the stash kernel
    (profiles/r02/diag_small.txt); the fp32 1-link chain keeps its check in
    test_prismatic_joints_dh_kernels."""
    for pf, seed in ((0.0, 1200 + n), (0.4, 1300 + n)):
        r = synth.random_chain(n, seed, prismatic_fraction=pf)
        for B in (1, 127, 129, 3001):
            q, qd, qdd = synth.states(21, n, 0, B)
            check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, dtype, strategy="thread")
    rng = np.random.default_rng(n)
    V0, Vd0, Ft = rng.standard_normal((3, 6))
    r = synth.random_chain(n, 1400 + n, prismatic_fraction=0.3)
    model = rd.Model.from_robot(r, (0, 0, 0))
    model.set_boundary(V0, Vd0, Ft)
    model.set_strategy("thread")
    q, qd, qdd = synth.states(22, n, 0, 500)
    tau, (q64, qd64, qdd64) = run_id(rd, model, q, qd, qdd, dtype)
    ref = np.stack([oracle.rnea(r, q64[:, b], qd64[:, b], qdd64[:, b], V0, Vd0, Ft) for b in range(500)], 1)
    assert rel_err_per_state(tau, ref).max() <= TOL[dtype]


@pytest.mark.parametrize("n", [7, 12])
def test_thread_short_chain_many_waves(rd, n):
    """The capped-register build of the register kernel (fp64, n = 6..12, batches
    above 300k states; n = 7 and 12 re-derive sin/cos in the backward sweep) on a
    sample of 400k states: every CTA boundary neighbourhood plus random states."""
    B = 400_000
    r = synth.random_chain(n, 1500 + n, prismatic_fraction=0.3)
    q, qd, qdd = synth.states(23, n, 0, B)
    cols = parity_sample(B, tile=128)
    check_id(rd, r, synth.GRAVITY_Z, q, qd, qdd, strategy="thread", sample=cols)


@pytest.mark.parametrize("dtype,n", [(torch.float64, n) for n in (1, 2, 3, 5, 7, 8, 9, 12, 16, 17)] +
                                    [(torch.float32, n) for n in (2, 3, 5, 7, 8, 12, 20, 21)])
def test_fd_short_chain_register_aba(rd, n, dtype):
    """FD (ABA) for n <= 16 (fp64) / 20 (fp32) keeps sweep 2's per-link records
    in registers (aba_small.cuh); 17 / 21 are the first workspace-kernel lengths.  Backward error
    (A14) at the contract tolerance on revolute and mixed prismatic chains with
    ragged batches, the per-state failing-pivot status, the model boundary and
    per-state boundaries.  (fp32 from n = 2: a 1-link state's single torque can
    cancel, reading A16.)"""
    for pf, seed in ((0.0, 1600 + n), (0.4, 1700 + n)):
        r = synth.random_chain(n, seed, prismatic_fraction=pf)
        for B in (1, 129, 2000):
            check_fd(rd, r, synth.GRAVITY_Z, B, 31, dtype, n_cond=8)
    r = synth.random_chain(n, 1800 + n, prismatic_fraction=0.3)
    model = rd.Model.from_robot(r, (0, 0, 0))
    rng = np.random.default_rng(n)
    V0, Vd0, Ft = rng.standard_normal((3, 6))
    model.set_boundary(V0, Vd0, Ft)
    B = 300
    q, qd, qdd = (_rounded(x, dtype) for x in synth.states(32, n, 0, B))
    tau = _rounded(np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], V0, Vd0, Ft) for b in range(B)], 1), dtype)
    st = torch.full((B,), -1, dtype=torch.int32, device="cuda")
    out = rd.forward_dynamics(model, dev(q, dtype), dev(qd, dtype), dev(tau, dtype), status=st).double().cpu().numpy()
    assert int(st.abs().max()) == 0
    back = np.stack([oracle.rnea(r, q[:, b], qd[:, b], out[:, b], V0, Vd0, Ft) for b in range(B)], 1)
    assert rel_err_per_state(back, tau).max() <= TOL[dtype]
    # per-state boundary vectors (NEXT-4)
    model2 = rd.Model.from_robot(r, synth.GRAVITY_Z)
    Vs, Vds, Fs = (_rounded(a, dtype) for a in rng.standard_normal((3, 6, B)))
    tau2 = _rounded(np.stack([oracle.rnea(r, q[:, b], qd[:, b], qdd[:, b], Vs[:, b], Vds[:, b], Fs[:, b])
                              for b in range(B)], 1), dtype)
    out2 = rd.forward_dynamics(model2, dev(q, dtype), dev(qd, dtype), dev(tau2, dtype),
                               boundary=(dev(Vs, dtype), dev(Vds, dtype), dev(Fs, dtype))).double().cpu().numpy()
    back2 = np.stack([oracle.rnea(r, q[:, b], qd[:, b], out2[:, b], Vs[:, b], Vds[:, b], Fs[:, b])
                      for b in range(B)], 1)
    assert rel_err_per_state(back2, tau2).max() <= TOL[dtype]
