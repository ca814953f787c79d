"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded
inputs.  Bar (BJ north_star, R19): relative max-norm 1e-11 on matrix entries, 1e-8 on
the solved density; GEMV against a dense product of the same stored matrix at 1e-13."""
import os

import mpmath as mp
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1811_05224_b200 import stbem as S  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MAT_TOL = 1e-11
W_TOL = 1e-8


def relmax(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def cuda(x):
    return torch.tensor(np.asarray(x), dtype=torch.float64, device="cuda")


_cache = {}


def gpu_mats(name, n_slices=1, q_bulk=0, cache=True):
    key = (name, n_slices, q_bulk)
    if key in _cache:
        return _cache[key]
    w = W.get(name)
    m = S.Mesh.from_workload(w, n_slices=n_slices)
    out = (w, m, {k: getattr(m, f"assemble_{k}")(q_bulk=q_bulk) for k in "VKD"})
    if cache:
        _cache[key] = out
    return out


_ocache = {}


def oracle_dense(name, kind):
    if (name, kind) not in _ocache:
        _ocache[(name, kind)] = O.OracleMesh(W.get(name)).dense(kind)
    return _ocache[(name, kind)]


# ------------------------------------------------------------- special functions
def test_diag_fp64_rate_is_a_plausible_dfma_rate():
    """the live DFMA rate bench.py reports beside the assembly roofline: positive and below the
    max-clock FP64 peak (148 SMs x 64 DFMA/clk x 2 flops x 1.965 GHz = 37.2 TFLOP/s, + 2%)"""
    r = S.diag_fp64_rate(0.3)
    assert 5.0 < r < 37.2 * 1.02, r


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_special_functions_against_mpmath(which):
    xs = np.concatenate([np.logspace(-13, np.log10(3.999), 300), np.linspace(3.99, 4.01, 21),
                         np.linspace(4.0, 60.0, 300), [100.0, 300.0, 700.0]])
    mp.mp.dps = 30
    ref = []
    for x in xs:
        X = mp.mpf(float(x))
        e1 = mp.e1(X)
        if which == 0:
            r = e1
        elif which == 1:
            r = e1 + mp.euler + mp.log(X)
        elif which == 2:
            r = (1 + X) * e1 - mp.exp(-X)
        else:
            r = mp.exp(-X) / X - 1 / X - e1
        ref.append(float(r))
    ref = np.array(ref)
    out = S.eval_special(which, cuda(xs), torch.empty(len(xs), dtype=torch.float64, device="cuda")).cpu().numpy()
    # absolute error at the FP64 rounding level of the small-x values, relative in the tail
    scale = np.maximum(1.0, np.abs(np.log(xs))) if which != 3 else np.maximum(1.0 / xs, 1.0)
    err = np.abs(out - ref)
    assert np.all(err <= 4e-15 * scale + 1e-13 * np.abs(ref)), (which, float((err / (scale + np.abs(ref))).max()))


# ---------------------------------------------------------------- matrices
@pytest.mark.parametrize("name", ["T8", "LT", "C1"])
@pytest.mark.parametrize("kind", ["V", "K", "D"])
def test_matrix_full_parity(name, kind):
    w, m, A = gpu_mats(name)
    ref = oracle_dense(name, kind)
    got = A[kind].dense()
    err = relmax(got, ref)
    print(f"{name} {kind} rel max-norm error {err:.3e}")
    assert err <= MAT_TOL
    ng = w.n_gamma
    # causality zeros read back exactly
    for a in range(w.n_steps):
        assert np.all(got[a * ng:(a + 1) * ng, (a + 1) * ng:] == 0.0)


def sample_entries(w, rng, n_random=1500, rows_per=6):
    ng, nt = w.n_gamma, w.n_steps
    rows, cols = [], []
    for a in sorted({0, 1, 2, nt // 2, nt - 1}):
        for b in range(max(0, a - 3), a + 1):
            for i in rng.choice(ng, size=min(rows_per, ng), replace=False):
                for j in range(ng):
                    rows.append(a * ng + i)
                    cols.append(b * ng + j)
    a = rng.integers(0, nt, n_random)
    b = (rng.random(n_random) * (a + 1)).astype(np.int64)
    rows += list(a * ng + rng.integers(0, ng, n_random))
    cols += list(b * ng + rng.integers(0, ng, n_random))
    return np.array(rows), np.array(cols)


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_matrix_sampled_parity(name):
    """BJ configs C2, C3, C5: near/singular entries of the first, middle and last test steps plus
    seeded random entries (the full matrices are beyond the oracle's budget)."""
    w, m, A = gpu_mats(name, cache=(name == "C2"))
    rng = np.random.default_rng(1811)
    rows, cols = sample_entries(w, rng, n_random=1000, rows_per=3 if name != "C2" else 6)
    om = O.OracleMesh(w)
    for kind in "VKD":
        r_, c_ = (rows, cols) if kind != "D" else (rows[::3], cols[::3])
        ref = om.entries(kind, r_, c_)
        got = A[kind].entries(r_, c_)
        # max-norm over the matrix: the sample contains the diagonal blocks of test step 0
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        print(f"{name} {kind} sampled rel max-norm error {err:.3e} over {len(r_)} entries")
        assert err <= MAT_TOL


def test_virtual_slices_bitwise():
    """P = 4 temporal slices on one GPU (all blocks owned) store the same entries"""
    _, _, A1 = gpu_mats("C1")
    _, _, A4 = gpu_mats("C1", n_slices=4)
    for k in "VKD":
        assert np.array_equal(A1[k].dense(), A4[k].dense())


# ---------------------------------------------------------------- products
@pytest.mark.parametrize("n_slices", [1, 3])
def test_gemv(n_slices):
    w, m, A = gpu_mats("C1", n_slices=n_slices)
    x = W.random_vector(w.n)
    yprev = W.random_vector(w.n, seed=7)
    for k in "VKD":
        dense = A[k].dense()
        y = cuda(yprev)
        A[k].matvec(cuda(x), y, a=1.5, b=-0.5)
        ref = 1.5 * dense @ x - 0.5 * yprev
        assert relmax(y.cpu().numpy(), ref) <= 1e-13


def test_gemv_c3_ragged_rows():
    w, m, A = gpu_mats("C3", cache=False)
    x = W.random_vector(w.n)
    y = torch.empty(w.n, dtype=torch.float64, device="cuda")
    A["V"].matvec(cuda(x), y)
    y = y.cpu().numpy()
    ng = w.n_gamma
    for r in [0, 1, ng - 1, ng * 100 + 7, w.n - 1]:
        row = A["V"].get(r, 1, 0, w.n)[0]
        assert abs(y[r] - row @ x) <= 1e-13 * np.abs(row).sum() * 1.0


@pytest.mark.parametrize("name", ["C1", "ratio10", "pentagon", "LT"])
def test_mass_matrices(name):
    """primal, dual and lumped mass: products and the (transposed) cyclic
    solves against the oracle's dense matrices -- on non-uniform boundaries too, where the dual
    hats' node values v- != 1/2 (ratio10: neighbours of length ratio 10; pentagon and LT: unequal
    sides, graded steps) and the dual mass is not symmetric"""
    from workloads.edge import edge_workloads
    w = edge_workloads()[name] if name in ("ratio10", "pentagon") else W.get(name)
    m = S.Mesh.from_workload(w)
    om = O.OracleMesh(w)
    x = W.random_vector(w.n)
    refs = {S.MASS_PRIMAL: om.mass_primal(), S.MASS_DUAL: om.mass_dual(), S.MASS_DUAL_LUMPED: np.diag(om.lumped_dual())}
    for kind, Md in refs.items():
        M = m.assemble_M(kind)
        y = torch.zeros(w.n, dtype=torch.float64, device="cuda")
        M.matvec(cuda(x), y)
        assert relmax(y.cpu().numpy(), Md @ x) <= 1e-14
        if kind != S.MASS_PRIMAL:
            for tr in (False, True):
                z = M.solve(cuda(x), torch.empty_like(y), transpose=tr).cpu().numpy()
                ref = np.linalg.solve(Md.T if tr else Md, x)
                assert relmax(z, ref) <= 1e-12


def test_rhs_parity():
    w, m, A = gpu_mats("C1")
    g = W.dirichlet_data(w)
    b = torch.empty(w.n, dtype=torch.float64, device="cuda")
    S.rhs(A["K"], m.assemble_M(S.MASS_PRIMAL), cuda(g), b)
    om = O.OracleMesh(w)
    ref = om.rhs(oracle_dense("C1", "K"), g)
    assert relmax(b.cpu().numpy(), ref) <= 1e-11


# ---------------------------------------------------------------- solver
def solve(name, precond, tol):
    w, m, A = gpu_mats(name)
    g = cuda(W.dirichlet_data(w))
    b = torch.empty_like(g)
    S.rhs(A["K"], m.assemble_M(S.MASS_PRIMAL), g, b)
    M = m.assemble_M(S.MASS_DUAL_LUMPED if precond == 1 else S.MASS_DUAL) if precond else None
    wv = torch.zeros_like(g)
    rep = S.solve_gmres(A["V"], b, wv, D=A["D"] if precond else None, M=M, rel_tol=tol, max_iter=300, precond=precond)
    return wv.cpu().numpy(), rep


@pytest.mark.parametrize("name,precond", [("C1", 0), ("C1", 2), ("C2", 1), ("C2", 2)])
def test_true_residual_from_kept_products(name, precond):
    """the default true residual ||C(b - V w)|| / ||C b|| = ||beta q_0 - sum_i y_i C V q_i|| / beta
    from the products of the Arnoldi steps (by linearity) against fresh products C V w
    (BEM_GMRES_FRESH_RESIDUAL): the same solution, the same residual up to the rounding of the
    products, and one V_h and one D_h product fewer"""
    w, m, A = gpu_mats(name)
    g = cuda(W.dirichlet_data(w))
    b = torch.empty_like(g)
    S.rhs(A["K"], m.assemble_M(S.MASS_PRIMAL), g, b)
    M = m.assemble_M(S.MASS_DUAL_LUMPED if precond == 1 else S.MASS_DUAL) if precond else None
    out = []
    for fresh in (False, True):
        wv = torch.zeros_like(g)
        rep = S.solve_gmres(A["V"], b, wv, D=A["D"] if precond else None, M=M, rel_tol=1e-10, max_iter=300,
                            precond=precond, fresh_residual=fresh)
        out.append((wv.cpu().numpy(), rep))
    (w0, r0), (w1, r1) = out
    assert np.array_equal(w0, w1) and r0["iterations"] == r1["iterations"]
    assert abs(r0["true_rel_residual"] - r1["true_rel_residual"]) <= 1e-13 + 1e-3 * r1["true_rel_residual"], (r0, r1)
    assert r0["true_rel_residual"] <= 2e-10
    assert r1["n_matvec_V"] == r0["n_matvec_V"] + 1
    assert r1["n_matvec_D"] == r0["n_matvec_D"] + (1 if precond else 0)


@pytest.mark.parametrize("precond,band", [(0, (20, 35)), (1, (14, 26)), (2, (10, 22))])
def test_gmres_c1(precond, band):
    w = W.get("C1")
    wv, rep = solve("C1", precond, 1e-10)
    V, K = oracle_dense("C1", "V"), oracle_dense("C1", "K")
    om = O.OracleMesh(w)
    b = om.rhs(K, W.dirichlet_data(w))
    wd = O.block_forward_solve(V, b, om.ng)
    assert rep["converged"] and band[0] <= rep["iterations"] <= band[1], rep
    assert np.all(np.diff(rep["history"]) <= 1e-14)
    assert rep["true_rel_residual"] <= 1e-9
    assert relmax(wv, wd) <= W_TOL
    # same iteration count as the oracle's MGS GMRES on its own matrices (+-1: rounding)
    D = oracle_dense("C1", "D")
    C = O.make_preconditioner(precond, D, om.mass_dual(), om.lumped_dual())
    _, it, _ = O.gmres(lambda v: V @ v, C, b, 1e-10)
    assert abs(it - rep["iterations"]) <= 1


@pytest.mark.parametrize("precond", [1, 2])
def test_gmres_c2_against_golden(precond):
    path = os.path.join(GOLDEN, "C2_oracle_w.npy")
    if not os.path.exists(path):
        pytest.skip("tests/golden/C2_oracle_w.npy missing (python -m oracle.gen_golden C2)")
    wd = np.load(path)
    wv, rep = solve("C2", precond, 1e-10)
    assert rep["converged"] and rep["iterations"] <= 30, rep
    assert relmax(wv, wd) <= W_TOL


@pytest.mark.parametrize("name", ["T8", "LT"])
def test_touching_pairs_both_paths(name):
    """touching pairs through moment records (default where alpha (h_X+h_Y)^2 / (4 min h_t) < 4)
    and through the per-lag singular kernel (BEM_QUAD_LEGACY_SING) agree with the oracle"""
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    for kind in "VKD":
        ref = oracle_dense(name, kind)
        fused = getattr(m, f"assemble_{kind}")()
        legacy = getattr(m, f"assemble_{kind}")(legacy_sing=True)
        assert fused.stats()["fused_sing"] == 1 and legacy.stats()["fused_sing"] == 0
        for A in (fused, legacy):
            assert relmax(A.dense(), ref) <= MAT_TOL, (kind, relmax(A.dense(), ref))


@pytest.mark.parametrize("name", ["LT", "C1", "S32"])
def test_symmetric_packed_storage(name):
    """V_h, D_h with symmetric packed spatial blocks (default) against full storage: the same
    entries (the mirrored half is the same integral with the roles of the points exchanged) and
    the same products"""
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    x = W.random_vector(w.n)
    for kind in "VD":
        P = getattr(m, f"assemble_{kind}")()
        F = getattr(m, f"assemble_{kind}")(full_storage=True)
        dp, df = P.dense(), F.dense()
        assert relmax(dp, df) <= 1e-13
        ng = w.n_gamma
        scale = np.abs(dp).max()
        for a in range(w.n_steps):   # every spatial block of the packed matrix is symmetric
            blk = dp[a * ng:(a + 1) * ng, :(a + 1) * ng].reshape(ng, a + 1, ng)
            # only the upper triangle is stored, the lower one read back as its mirror: exactly symmetric
            assert np.array_equal(blk, blk.transpose(2, 1, 0))
        yp = torch.empty(w.n, dtype=torch.float64, device="cuda")
        yf = torch.empty_like(yp)
        P.matvec(cuda(x), yp)
        F.matvec(cuda(x), yf)
        assert relmax(yp.cpu().numpy(), yf.cpu().numpy()) <= 1e-13
        assert relmax(yp.cpu().numpy(), dp @ x) <= 1e-13
        # packed: the distinct entries (i <= j) of every spatial block; the stored doubles exceed them
        # only by the ragged parts of the last tile row / column
        nt = w.n_steps
        assert P.stats()["entries"] == ng * (ng + 1) // 2 * nt * (nt + 1) // 2
        assert P.info()["bytes"] >= 8 * P.stats()["entries"]
        if ng >= 64:   # (below, the one ragged 32 x 32 tile outweighs the halving)
            assert P.info()["bytes"] < F.info()["bytes"]


@pytest.mark.parametrize("name,n_slices", [("C1", 1), ("LT", 1), ("C1", 3), ("S32", 2)])
def test_rhs_fused(name, n_slices):
    """b = 1/2 M g + K g with K_h never stored (bem_rhs_fused) against the stored K_h product and
    the oracle's right-hand side"""
    w = W.get(name)
    m = S.Mesh.from_workload(w, n_slices=n_slices)
    g = cuda(W.dirichlet_data(w))
    Mp = m.assemble_M(S.MASS_PRIMAL)
    b_stored = torch.empty_like(g)
    S.rhs(m.assemble_K(), Mp, g, b_stored)
    b_fused = torch.empty_like(g)
    st = S.rhs_fused(m, Mp, g, b_fused, stats=True)
    bf, bs = b_fused.cpu().numpy(), b_stored.cpu().numpy()
    assert relmax(bf, bs) <= 1e-13, relmax(bf, bs)
    om = O.OracleMesh(w)
    ref = om.rhs(oracle_dense(name, "K") if name in ("C1", "LT") else om.dense("K"), W.dirichlet_data(w))
    assert relmax(bf, ref) <= 1e-11
    assert st["fused_sing"] == 1 and st["evals_bulk"] > 0


@pytest.mark.parametrize("name,n_slices", [("C1", 1), ("C1", 3), ("C2", 1), ("C2", 5), ("C5", 1), ("ragged33", 1),
                                          ("grade2", 2), ("pentagon", 1), ("alpha_small", 1), ("acute", 1)])
def test_rhs_fused_trial_moment_table(name, n_slices):
    """K_h g: the regime-A nodes of the interior bulk columns summed over the trial index first
    (k_kg_tab, the default) against every node evaluated pair by pair (BEM_QUAD_KG_ENTRYWISE):
    the same quadrature and regime forms re-associated, so equal to rounding; n_slices > 1 runs the
    per-block tables of the multi-block list (trial ranges b0..b1 inside the block triangle)"""
    from workloads.edge import edge_workloads
    w = edge_workloads()[name] if name in edge_workloads() else W.get(name)
    m = S.Mesh.from_workload(w, n_slices=n_slices)
    g = cuda(W.dirichlet_data(w))
    Mp = m.assemble_M(S.MASS_PRIMAL)
    b_tab, b_ent = torch.empty_like(g), torch.empty_like(g)
    st_t = S.rhs_fused(m, Mp, g, b_tab, stats=True)
    st_e = S.rhs_fused(m, Mp, g, b_ent, stats=True, entrywise=True)
    err = relmax(b_tab.cpu().numpy(), b_ent.cpu().numpy())
    assert err <= 1e-12, err   # re-association over up to N_Gamma trial pairs (C5: 1.1e-13)
    # the same nodes by regime; the table took a share of the regime-A ones (none without bulk nodes
    # three steps apart)
    assert st_t["nodes_bulk"] == st_e["nodes_bulk"]
    assert st_e["nodes_bulk_tab"] == 0
    assert st_t["nodes_bulk_tab"] <= st_t["nodes_bulk"][0]
    if name in ("C1", "C2", "C5"):
        assert st_t["nodes_bulk_tab"] > 0.5 * st_t["nodes_bulk"][0]


@pytest.mark.parametrize("name", ["C1", "S32", "ragged33"])
def test_block_toeplitz_variant(name):
    """row f3: on equal time steps the first block column T_d = A(d, 0) reproduces every entry
    (A(a, b) = T_{a-b}), the Toeplitz GEMM product equals the dense product, and GMRES with the
    Toeplitz V_h and D_h returns the dense solution (ragged33: odd N_Gamma, unaligned rows of x
    for the cp.async staging, a ragged 128-row tile)"""
    from workloads.edge import edge_workloads
    w = edge_workloads()[name] if name in edge_workloads() else W.get(name)
    m = S.Mesh.from_workload(w)
    x = W.random_vector(w.n)
    mats = {}
    for kind in "VKD":
        T = m.assemble_toeplitz(kind)
        Dn = getattr(m, f"assemble_{kind}")()
        dT, dD = T.dense(), Dn.dense()
        assert relmax(dT, dD) <= 1e-13, (kind, relmax(dT, dD))
        assert relmax(dT, oracle_dense(name, kind) if name == "C1" else dD) <= 1e-11
        yT = torch.empty(w.n, dtype=torch.float64, device="cuda")
        yD = torch.empty_like(yT)
        T.matvec(cuda(x), yT)
        Dn.matvec(cuda(x), yD)
        assert relmax(yT.cpu().numpy(), yD.cpu().numpy()) <= 1e-13
        assert T.stats()["entries"] == w.n_steps * w.n_gamma ** 2
        mats[kind] = (T, Dn)
    g = cuda(W.dirichlet_data(w))
    Mp, Me = m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
    sols = []
    for i in (0, 1):
        b = torch.empty_like(g)
        S.rhs(mats["K"][i], Mp, g, b)
        wv = torch.zeros_like(g)
        rep = S.solve_gmres(mats["V"][i], b, wv, D=mats["D"][i], M=Me, rel_tol=1e-10, max_iter=200, precond=2)
        assert rep["converged"]
        sols.append(wv.cpu().numpy())
    assert relmax(sols[0], sols[1]) <= 1e-9


def test_block_toeplitz_needs_uniform_steps():
    m = S.Mesh.from_workload(W.get("LT"))      # graded steps
    with pytest.raises(S.BemError):
        m.assemble_toeplitz("V")


POT_PTS = np.array([[0.5, 0.5, 0.5], [0.25, 0.5, 1.0], [0.5, 0.75, 0.75], [0.3, 0.3, 0.25],
                    [0.6, 0.35, 0.9], [0.4, 0.65, 0.6], [0.45, 0.5, 0.125], [0.7, 0.7, 0.33]])


@pytest.mark.parametrize("name", ["C1", "S32"])
def test_potential_parity(name):
    """row f2: the representation formula on the GPU against the oracle's (same w, g)"""
    w = W.get(name)
    om = O.OracleMesh(w)
    g = W.dirichlet_data(w)
    wh = W.random_vector(w.n)          # any density: the map (w, g) -> u is what is compared
    m = S.Mesh.from_workload(w)
    got = S.eval_potential(m, cuda(wh), cuda(g), POT_PTS).cpu().numpy()
    ref = om.potential(wh, g, POT_PTS)
    assert relmax(got, ref) <= 1e-11, relmax(got, ref)


def test_potential_after_solve_converges():
    """GPU solve then representation formula: the error against u = U*(x - x*, t) at interior
    points falls under refinement C1 -> C2 -> C3"""
    errs = []
    for name in ("C1", "C2", "C3"):
        wv, rep = solve(name, 2, 1e-10) if name != "C3" else (None, None)
        w = W.get(name)
        if name == "C3":
            m = S.Mesh.from_workload(w)
            V, Dm = m.assemble_V(), m.assemble_D()
            gg = cuda(W.dirichlet_data(w))
            b = torch.empty_like(gg)
            S.rhs_fused(m, m.assemble_M(S.MASS_PRIMAL), gg, b)
            wt = torch.zeros_like(gg)
            S.solve_gmres(V, b, wt, D=Dm, M=m.assemble_M(S.MASS_DUAL), rel_tol=1e-10, max_iter=200, precond=2)
            wv = wt.cpu().numpy()
        m = S.Mesh.from_workload(w)
        u = S.eval_potential(m, cuda(wv), cuda(W.dirichlet_data(w)), POT_PTS).cpu().numpy()
        ex = W.exact_solution(w, POT_PTS[:, :2], POT_PTS[:, 2])
        errs.append(float(np.abs(u - ex).max() / np.abs(ex).max()))
    print("potential errors", errs)
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-4, errs


def test_potential_rejects_boundary_points():
    w = W.get("C1")
    m = S.Mesh.from_workload(w)
    with pytest.raises(S.BemError):
        S.eval_potential(m, cuda(np.zeros(w.n)), cuda(np.zeros(w.n)), np.array([[0.01, 0.5, 0.5]]))


@pytest.mark.parametrize("L,orders", [(2, (4, 4, 12)), (3, (8, 6, 16)), (4, (4, 4, 12)), (5, (4, 4, 12))])
def test_initial_potential_parity(L, orders):
    """row f1: b - M_h^0 u0 on the GPU against the oracle's M_h^0 u0 (paper's Table-1 workload)"""
    import workloads.table1 as T
    w = T.table1(L)
    om = O.OracleMesh(w)
    nodes, tris = T.triangulation(w)
    u0 = T.initial_nodes(w)
    ref = om.initial_rhs(nodes, tris, u0, *orders)
    m = S.Mesh.from_workload(w)
    b = torch.zeros(w.n, dtype=torch.float64, device="cuda")
    S.rhs_initial(m, nodes, tris, cuda(u0), b, *orders)
    got = -b.cpu().numpy()
    assert relmax(got, ref) <= 1e-11, relmax(got, ref)


def test_large_kappa_falls_back_to_legacy_touching_path():
    """kappa = alpha h^2 / (4 min h_t) beyond the records' regime A: the touching pairs go through
    the per-lag singular kernel (fused_sing = 0) and bem_rhs_fused falls back to assemble + GEMV"""
    from workloads.configs import square
    w = square(2, 64, name="K64", tol=1e-10)      # h = 0.5, h_t = 1/64: kappa = 1
    m = S.Mesh.from_workload(w)
    assert m.info.kappa >= 1.0
    om = O.OracleMesh(w)
    rows = np.arange(0, w.n, 7)
    for kind in "VKD":
        A = getattr(m, f"assemble_{kind}")()
        assert A.stats()["fused_sing"] == 0
        cols = (rows // w.n_gamma) * w.n_gamma + (rows * 3) % w.n_gamma    # same test step, varied j
        ref = om.entries(kind, rows, cols)
        got = A.entries(rows, cols)
        assert float(np.abs(got - ref).max() / np.abs(ref).max()) <= MAT_TOL
    g = cuda(W.dirichlet_data(w))
    Mp = m.assemble_M(S.MASS_PRIMAL)
    b1, b2 = torch.empty_like(g), torch.empty_like(g)
    S.rhs(m.assemble_K(), Mp, g, b1)
    st = S.rhs_fused(m, Mp, g, b2, stats=True)
    assert st["fused_sing"] == 0
    assert relmax(b2.cpu().numpy(), b1.cpu().numpy()) <= 1e-14


def test_c4_sampled_entries_block_toeplitz():
    """BJ configs[3] (C4, N = 262 144, the largest): its dense V_h + D_h need 2 x 146 GB, the uniform
    steps let the block-Toeplitz variant hold every entry on one GPU; sampled entries (diagonal,
    near and random cells) against the oracle"""
    w = W.get("C4")
    m = S.Mesh.from_workload(w)
    rng = np.random.default_rng(1811)
    rows, cols = sample_entries(w, rng, n_random=300, rows_per=2)
    om = O.OracleMesh(w)
    for kind in "VKD":
        T = m.assemble_toeplitz(kind)
        r_, c_ = (rows[::4], cols[::4]) if kind == "D" else (rows[::2], cols[::2])
        ref = om.entries(kind, r_, c_)
        got = T.entries(r_, c_)
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        print(f"C4 {kind} sampled rel max-norm error {err:.3e} over {len(r_)} entries")
        assert err <= MAT_TOL
        T.close()


def test_ragged_tiles_and_many_slices():
    """N_Gamma = 40 (a full 32-wide tile and a ragged one of 8) with the maximum number of temporal
    slices (P = N_I): symmetric packed storage, products and the fused RHS against the oracle"""
    from workloads.configs import square
    w = square(10, 12, name="R40", tol=1e-10)
    om = O.OracleMesh(w)
    x = W.random_vector(w.n)
    g = W.dirichlet_data(w)
    for P in (1, 12):
        m = S.Mesh.from_workload(w, n_slices=P)
        for kind in "VKD":
            A = getattr(m, f"assemble_{kind}")()
            ref = om.dense(kind)
            dA = A.dense()
            assert relmax(dA, ref) <= MAT_TOL, (P, kind, relmax(dA, ref))
            y = torch.empty(w.n, dtype=torch.float64, device="cuda")
            A.matvec(cuda(x), y)
            assert relmax(y.cpu().numpy(), dA @ x) <= 1e-13
        b = torch.empty(w.n, dtype=torch.float64, device="cuda")
        S.rhs_fused(m, m.assemble_M(S.MASS_PRIMAL), cuda(g), b)
        assert relmax(b.cpu().numpy(), om.rhs(om.dense("K"), g)) <= 1e-11


def test_api_misuse_reports_errors():
    """the C-ABI's documented error returns (include/stbem.h) surface as BemError, nothing launches
    on bad input: wrong matrix kinds, missing or mismatched preconditioner parts, product mode on
    V_h, out-of-range triangle indices, orders above the tables"""
    import workloads.table1 as T
    w = W.get("T8")
    m = S.Mesh.from_workload(w)
    V, K, D = m.assemble_V(), m.assemble_K(), m.assemble_D()
    Ml, Md = m.assemble_M(S.MASS_DUAL_LUMPED), m.assemble_M(S.MASS_DUAL)
    b = cuda(np.ones(w.n))
    x = torch.zeros_like(b)
    with pytest.raises(S.BemError):
        S.solve_gmres(K, b, x)                              # first matrix must be V_h
    with pytest.raises(S.BemError):
        S.solve_gmres(V, b, x, precond=2)                   # D_h and M missing
    with pytest.raises(S.BemError):
        S.solve_gmres(V, b, x, D=D, M=Ml, precond=2)        # exact precond needs the dual mass
    with pytest.raises(S.BemError):
        S.solve_gmres(V, b, x, D=V, M=Md, precond=2)        # D slot holds V_h
    rep = S.solve_gmres(V, b, x, D=D, M=Md, precond=2, rel_tol=1e-10)
    assert rep["status"] == "OK"
    wt = T.table1(2)
    mt = S.Mesh.from_workload(wt)
    nodes, tris = T.triangulation(wt)
    u0 = cuda(T.initial_nodes(wt))
    bt = torch.zeros(wt.n, dtype=torch.float64, device="cuda")
    bad = tris.copy()
    bad[0, 0] = len(nodes)
    with pytest.raises(S.BemError):
        S.rhs_initial(mt, nodes, bad, u0, bt)
    with pytest.raises(S.BemError):
        S.rhs_initial(mt, nodes, tris, u0, bt, qx=40)
    assert float(bt.abs().max()) == 0.0                     # nothing was written
    from workloads.configs import Workload, uniform_times
    tri = Workload("tri3", [(0.0, 0.0), (1.0, 0.0), (0.3, 0.8)], [1, 1, 1], uniform_times(4), 1.0,
                   (1.5, 1.5), 1e-10)
    with pytest.raises(S.BemError):
        S.Mesh.from_workload(tri).assemble_V()              # N_Gamma >= 6 required


def test_distributed_path_on_a_one_rank_nccl_communicator():
    """the multi-GPU code path (owned blocks, partial products + ncclAllReduce on the stream,
    all-reduced fused RHS) on a real one-rank NCCL communicator against the plain path: same
    matrices, products, RHS and GMRES solution (one GPU: no ranks waiting on each other)"""
    import ctypes
    uid = ctypes.create_string_buffer(128)
    S.check(S.lib().bem_nccl_get_unique_id(uid))
    comm = S.Comm(0, 1, 0, unique_id=bytes(uid.raw))
    w = W.get("C1")
    out = []
    for cm in (comm, None):
        m = S.Mesh.from_workload(w, n_slices=2, comm=cm)
        V, D = m.assemble_V(), m.assemble_D()
        Mp, Md = m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
        g = cuda(W.dirichlet_data(w))
        b = torch.empty_like(g)
        S.rhs_fused(m, Mp, g, b)
        x = cuda(W.random_vector(w.n))
        y = torch.empty_like(x)
        V.matvec(x, y)
        wv = torch.zeros_like(g)
        rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=1e-10)
        assert rep["status"] == "OK"
        out.append((b.cpu().numpy(), y.cpu().numpy(), wv.cpu().numpy(), V.dense()))
    comm.close()
    (b1, y1, w1, V1), (b0, y0, w0, V0) = out
    assert np.array_equal(V1, V0)
    assert relmax(y1, y0) <= 1e-14 and relmax(b1, b0) <= 1e-14
    assert relmax(w1, w0) <= 1e-12


@pytest.mark.parametrize("name", ["triangle6", "onestep", "ragged33", "grade2", "alpha_small", "alpha_large",
                                  "acute", "pentagon", "ratio10", "scaled"])
def test_edge_case_meshes_full_parity(name):
    """degenerate and extreme inputs (minimal boundary, one step, ragged tiles, strong grading,
    alpha extremes): V_h, K_h, D_h in full against the oracle, causality zeros, and V_h's spatial
    blocks symmetric"""
    from workloads.edge import edge_workloads
    w = edge_workloads()[name]
    om = O.OracleMesh(w)
    m = S.Mesh.from_workload(w)
    ng = w.n_gamma
    for kind in "VKD":
        got = getattr(m, f"assemble_{kind}")().dense()
        ref = om.dense(kind)
        err = relmax(got, ref)
        assert err <= MAT_TOL, (name, kind, err)
        for a in range(w.n_steps):
            assert np.all(got[a * ng:(a + 1) * ng, (a + 1) * ng:] == 0.0)
        if kind == "V":
            for a in range(w.n_steps):
                for b in range(a + 1):
                    blk = got[a * ng:(a + 1) * ng, b * ng:(b + 1) * ng]
                    assert np.allclose(blk, blk.T, rtol=0, atol=MAT_TOL * np.abs(got).max())


@pytest.mark.parametrize("name", ["C1", "LT"])
def test_dual_pairing_inf_sup_from_gpu_mass(name):
    """row f4, SPEC's stability surrogate (eq. 5): the pairing block of the first time step
    read back from the GPU dual mass matrix (matvec on unit vectors) gives the oracle's discrete
    inf-sup constant sqrt(3)/2 (equal elements: C1 and LT both have h = 1/4 on every side)"""
    w = W.get(name)
    om = O.OracleMesh(w)
    m = S.Mesh.from_workload(w)
    Md = m.assemble_M(S.MASS_DUAL)
    ng = w.n_gamma
    cols = []
    for k in range(ng):
        e = torch.zeros(w.n, dtype=torch.float64, device="cuda")
        e[k] = 1.0
        y = torch.empty_like(e)
        Md.matvec(e, y)
        cols.append(y[:ng].cpu().numpy())
    Ms = np.stack(cols, 1) / (w.t_breaks[1] - w.t_breaks[0])
    np.testing.assert_allclose(Ms, om.mass_dual()[:ng, :ng] / om.ht[0], rtol=1e-14, atol=1e-16)
    wy, Uy = np.linalg.eigh(om.dual_gram())
    B = (Uy @ np.diag(wy ** -0.5) @ Uy.T) @ Ms @ np.diag(om.seg_h ** -0.5)
    assert np.linalg.svd(B, compute_uv=False).min() == pytest.approx(np.sqrt(3.0) / 2.0, rel=1e-12)


@pytest.mark.parametrize("t", [0.5, 0.05, 0.002])
def test_potential_initial_parity(t):
    """row f2 with u0 != 0: the initial potential (M~_0 u0)(x, t) of the representation formula on
    the GPU against the oracle (the paper's u0 on the Table-1 triangulation, L = 3); small t makes
    the Gaussian narrower than the triangles (composite cells)"""
    import workloads.table1 as T
    w = T.table1(3)
    om = O.OracleMesh(w)
    nodes, tris = T.triangulation(w)
    u0 = T.initial_nodes(w)
    pts = np.array([[0.5, 0.5, t], [0.3, 0.8, t], [0.05, 0.6, t], [0.9, 0.1, t]])
    ref = om.potential_initial(nodes, tris, u0, pts)
    m = S.Mesh.from_workload(w)
    out = torch.zeros(len(pts), dtype=torch.float64, device="cuda")
    S.eval_potential_initial(m, nodes, tris, cuda(u0), cuda(pts), out)
    assert relmax(out.cpu().numpy(), ref) <= 1e-11
    with pytest.raises(S.BemError):
        S.eval_potential_initial(m, nodes, tris, cuda(u0), cuda(np.array([[0.5, 0.5, 0.0]])), out[:1])


def test_representation_formula_with_initial_datum_converges():
    """SPEC's evaluate_interior example on the paper's Table-1 problem: u_h(x, t) =
    (M~_0 u0)(x,t) + (Vt w_h)(x,t) - (W g)(x,t) at x = (0.5, 0.5), t = 0.5 after the solve approaches
    u = e^{-t/alpha} sin(x . d) as L grows"""
    import workloads.table1 as T
    errs = []
    for L in (2, 3, 4, 5):
        w = T.table1(L)
        m = S.Mesh.from_workload(w)
        V, D, Mp, Md = m.assemble_V(), m.assemble_D(), m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
        nodes, tris = T.triangulation(w)
        u0 = cuda(T.initial_nodes(w))
        g = cuda(T.dirichlet_data(w))
        b = torch.empty_like(g)
        S.rhs_fused(m, Mp, g, b)
        S.rhs_initial(m, nodes, tris, u0, b)
        wv = torch.zeros_like(g)
        rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=1e-10, history=False)
        assert rep["status"] == "OK"
        pts = np.array([[0.5, 0.5, 0.5]])
        u = S.eval_potential(m, wv, g, pts)
        S.eval_potential_initial(m, nodes, tris, u0, cuda(pts), u)
        exact = float(T.exact(pts[:, :2], 0.5)[0])
        errs.append(abs(float(u.cpu().numpy()[0]) - exact) / abs(exact))
    assert errs[-1] < 0.25 * errs[0] and all(b < a for a, b in zip(errs, errs[1:])), errs


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_bench_step_configuration_against_golden(name):
    """the step exactly as bench.py launches it -- V_h and D_h assembled on two side streams while
    K_h g runs fused on the main stream, exact dual-mass preconditioning, solve after both streams
    are joined -- against the oracle's golden right-hand side and density (C2: dense oracle
    matrices; C3, N = 65 536: the oracle's first block columns, reading R26), eq. (4)
    P:81-90 solved to the GMRES tolerance of P:182 (BJ: 1e-10)"""
    path = os.path.join(GOLDEN, f"{name}_oracle_w.npy")
    if not os.path.exists(path):
        pytest.skip(f"tests/golden/{name}_oracle_w.npy missing (python -m oracle.gen_golden {name})")
    wd = np.load(path)
    bd = np.load(os.path.join(GOLDEN, f"{name}_oracle_b.npy"))
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    side = (torch.cuda.Stream(), torch.cuda.Stream())
    cur = torch.cuda.current_stream()
    for s_ in side:
        s_.wait_stream(cur)
    V = m.assemble_V(stream=side[0])
    D = m.assemble_D(stream=side[1])
    Mp, Md = m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
    g = cuda(W.dirichlet_data(w))
    b = torch.empty_like(g)
    S.rhs_fused(m, Mp, g, b)
    for s_ in side:
        cur.wait_stream(s_)
    wv = torch.zeros_like(g)
    rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=w.tol, history=False)
    assert rep["status"] == "OK"
    assert relmax(b.cpu().numpy(), bd) <= MAT_TOL
    assert relmax(wv.cpu().numpy(), wd) <= W_TOL
    for A in (V, D, Mp, Md):
        A.close()


def test_c5_leading_steps_against_golden():
    """the headline configuration (C5: L-shape, graded steps, N = 98 304) solved in the bench's
    launch configuration, against the oracle's exact density of the first 24 time steps (block
    forward substitution over the oracle's causal blocks, oracle/gen_golden.py C5; V_h is block
    lower triangular, so those steps depend on nothing else): b and w of those steps"""
    path = os.path.join(GOLDEN, "C5_oracle_w_first24.npy")
    if not os.path.exists(path):
        pytest.skip("tests/golden/C5_oracle_w_first24.npy missing (python -m oracle.gen_golden C5)")
    wd = np.load(path)
    bd = np.load(os.path.join(GOLDEN, "C5_oracle_b_first24.npy"))
    w = W.get("C5")
    k = len(wd)
    m = S.Mesh.from_workload(w)
    side = (torch.cuda.Stream(), torch.cuda.Stream())
    cur = torch.cuda.current_stream()
    for s_ in side:
        s_.wait_stream(cur)
    V = m.assemble_V(stream=side[0])
    D = m.assemble_D(stream=side[1])
    Mp, Md = m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
    g = cuda(W.dirichlet_data(w))
    b = torch.empty_like(g)
    S.rhs_fused(m, Mp, g, b)
    for s_ in side:
        cur.wait_stream(s_)
    wv = torch.zeros_like(g)
    rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=w.tol, history=False)
    assert rep["status"] == "OK"
    assert relmax(b.cpu().numpy()[:k], bd) <= MAT_TOL
    assert relmax(wv.cpu().numpy()[:k], wd) <= W_TOL
    for A in (V, D, Mp, Md):
        A.close()


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_full_size_step_properties(name):
    """BJ configs at full size in the bench's launch configuration, checked through properties
    that hold at any size: GMRES converges within the preconditioned iteration band of §6.2, the
    true preconditioned residual meets the tolerance, and the density approaches the exact
    Neumann datum (first order in h: relative L2(Sigma) error below that of C2)"""
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    side = (torch.cuda.Stream(), torch.cuda.Stream())
    cur = torch.cuda.current_stream()
    for s_ in side:
        s_.wait_stream(cur)
    V = m.assemble_V(stream=side[0])
    D = m.assemble_D(stream=side[1])
    Mp, Md = m.assemble_M(S.MASS_PRIMAL), m.assemble_M(S.MASS_DUAL)
    g = cuda(W.dirichlet_data(w))
    b = torch.empty_like(g)
    S.rhs_fused(m, Mp, g, b)
    for s_ in side:
        cur.wait_stream(s_)
    wv = torch.zeros_like(g)
    rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=w.tol, history=False)
    assert rep["status"] == "OK" and rep["iterations"] <= 16, rep
    assert rep["true_rel_residual"] <= 2.0 * w.tol, rep
    err, nrm = O.OracleMesh(w).l2_error(wv.cpu().numpy(), nq=4)
    assert err / nrm < 0.0798, (err, nrm)          # C2: 0.0798 (P11)
    for A in (V, D, Mp, Md):
        A.close()


@pytest.mark.parametrize("name", ["C1", "S32"])
def test_potential_parity_hard_points(name):
    """row f2 at the hard end of its domain: points at 1.05 h_max from Gamma (the rejection
    distance is h_max) next to each side, times inside the first step, just after a step break
    and at T"""
    w = W.get(name)
    om = O.OracleMesh(w)
    h = max(np.hypot(*(np.asarray(w.vertices[(k + 1) % len(w.vertices)]) - np.asarray(w.vertices[k]))) / n
            for k, n in enumerate(w.segments_per_side))
    t = np.asarray(w.t_breaks)
    d = 1.05 * h
    xs = [(d, 0.3), (0.4, d), (0.5, 1.0 - d), (1.0 - d, 0.6)]
    ts = [0.5 * t[1], t[2] + 1e-3 * (t[3] - t[2]), t[-1]]
    pts = np.array([[x1, x2, tt] for (x1, x2) in xs for tt in ts])
    g = W.dirichlet_data(w)
    wh = W.random_vector(w.n)
    m = S.Mesh.from_workload(w)
    got = S.eval_potential(m, cuda(wh), cuda(g), pts).cpu().numpy()
    ref = om.potential(wh, g, pts)
    assert relmax(got, ref) <= 1e-11, relmax(got, ref)


@pytest.mark.gpu
def test_storage_beyond_device_memory_reports_nomem():
    """maximum sizes: V_h of a 1024-element, 1024-step square needs ~2.2 TB even in symmetric packed
    storage (far beyond one GPU's 180 GB): bem_assemble fails with BEM_E_NOMEM (include/stbem.h)
    before any kernel runs, and the library stays usable -- the same process then assembles and
    checks a small matrix"""
    from workloads.configs import square
    big = S.Mesh.from_workload(square(256, 1024, name="huge", tol=1e-10))
    with pytest.raises(S.BemError) as ei:
        big.assemble_V()
    assert ei.value.status == 2, str(ei.value)             # BEM_E_NOMEM
    big.close()
    w = W.get("C1")
    om = O.OracleMesh(w)
    ref = om.dense("V")
    got = S.Mesh.from_workload(w).assemble_V().dense()
    assert relmax(got, ref) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C3", "C5"])
def test_rhs_fused_full_size_sampled_rows(name):
    """BJ configs C3, C5 at full size in the bench's product mode (bem_rhs_fused: K_h g with K_h
    never stored, one slice): rows of the first, second, middle and last test steps of
    b = (1/2 M_h + K_h) g against the oracle row by row"""
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    g_h = W.dirichlet_data(w)
    Mp = m.assemble_M(S.MASS_PRIMAL)
    b = torch.empty(w.n, dtype=torch.float64, device="cuda")
    S.rhs_fused(m, Mp, cuda(g_h), b)
    got = b.cpu().numpy()
    rng = np.random.default_rng(1811)
    ng, nt = w.n_gamma, w.n_steps
    rows = [a * ng + int(i) for a in (0, 1, nt // 2, nt - 1) for i in rng.choice(ng, 2, replace=False)]
    ref = O.OracleMesh(w).rhs_rows(rows, g_h)
    err = float(np.abs(got[rows] - ref).max() / np.abs(ref).max())
    print(f"{name} fused rhs sampled rows rel error {err:.3e}")
    assert err <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["C3", "C5"])
def test_gemv_full_size_sampled_rows(name):
    """BJ configs C3, C5 at full size: the bench's stored V_h, D_h (symmetric packed, one slice) and
    the fused-reduction SYMV, y = A x for a seeded x, against the oracle on rows of the first,
    second, middle and last test steps"""
    w = W.get(name)
    m = S.Mesh.from_workload(w)
    x_h = np.random.default_rng(1811).standard_normal(w.n)
    x = cuda(x_h)
    rng = np.random.default_rng(7)
    ng, nt = w.n_gamma, w.n_steps
    rows = [a * ng + int(i) for a in (0, 1, nt // 2, nt - 1) for i in rng.choice(ng, 2, replace=False)]
    om = O.OracleMesh(w)
    for kind in "VD":
        A = m.assemble_V() if kind == "V" else m.assemble_D()
        y = torch.empty_like(x)
        A.matvec(x, y)
        got = y.cpu().numpy()[rows]
        A.close()
        ref = om.matvec_rows(kind, rows, x_h)
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        print(f"{name} {kind} product sampled rows rel error {err:.3e}")
        assert err <= 1e-11


@pytest.mark.gpu
def test_c4_toeplitz_products_sampled_rows():
    """C4 at full size through the block-Toeplitz variant the bench times: y = T x (the DMMA GEMM over
    the stacked lags, lag-chunk partials reduced in fixed order) for V_h and D_h, rows of the first,
    second, middle and last test steps against the oracle's row sums"""
    w = W.get("C4")
    m = S.Mesh.from_workload(w)
    x_h = np.random.default_rng(1811).standard_normal(w.n)
    x = cuda(x_h)
    rng = np.random.default_rng(11)
    ng, nt = w.n_gamma, w.n_steps
    rows = [a * ng + int(i) for a in (0, 1, nt // 2, nt - 1) for i in rng.choice(ng, 2, replace=False)]
    om = O.OracleMesh(w)
    for kind in "VD":
        T = m.assemble_toeplitz(kind)
        y = torch.empty_like(x)
        T.matvec(x, y)
        got = y.cpu().numpy()[rows]
        T.close()
        ref = om.matvec_rows(kind, rows, x_h)
        err = float(np.abs(got - ref).max() / np.abs(ref).max())
        print(f"C4 Toeplitz {kind} product sampled rows rel error {err:.3e}")
        assert err <= 1e-11


def test_quadrature_options():
    """bem_quad_opts (include/stbem.h): q_near / near_gap at their defaults reproduce the default
    assembly bitwise; raised near orders keep oracle parity; invalid values are rejected"""
    w = W.get("C1")
    m = S.Mesh.from_workload(w)
    for kind in "VKD":
        A0 = getattr(m, f"assemble_{kind}")()
        A1 = getattr(m, f"assemble_{kind}")(q_near=min(6, A0.stats()["q_bulk"] + 1), near_gap=9)
        A2 = getattr(m, f"assemble_{kind}")(q_near=10, near_gap=3)
        d0, d1, d2 = A0.dense(), A1.dense(), A2.dense()
        assert np.array_equal(d0, d1)
        assert relmax(d2, oracle_dense("C1", kind)) <= MAT_TOL
        assert not np.array_equal(d0, d2)           # the near cells did change order
    for bad in (dict(q_bulk=7), dict(q_near=2), dict(q_near=17), dict(near_gap=-1), dict(q_sing=3)):
        with pytest.raises(S.BemError) as e:
            m.assemble_V(**bad)
        assert e.value.status == S.BEM_E_INVALID


def test_small_boundaries_rejected_everywhere():
    """the touching-pair enumeration needs N_Gamma >= 6: every assembly entry point says INVALID"""
    w = W.Workload("tri3", [(0.0, 0.0), (1.0, 0.0), (0.0, 1.0)], [1, 1, 1], W.configs.uniform_times(4), 1.0,
                   (1.5, 1.5), 1e-10)
    m = S.Mesh.from_workload(w)
    g = cuda(np.ones(w.n))
    b = torch.empty_like(g)
    Mp = m.assemble_M(S.MASS_PRIMAL)
    for call in (lambda: m.assemble_V(), lambda: m.assemble_toeplitz("K"), lambda: S.rhs_fused(m, Mp, g, b)):
        with pytest.raises(S.BemError) as e:
            call()
        assert e.value.status == S.BEM_E_INVALID


def test_cyclic_solve_beyond_shared_memory():
    """N_Gamma = 8000 (4 N_Gamma doubles exceed the 227 KB of shared memory per CTA): the dual-mass
    solves run from global memory and still match a dense solve"""
    w = W.Workload("big", [(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)], [1000, 3000, 1000, 3000],
                   W.configs.uniform_times(2), 1.0, (1.5, 1.5), 1e-10)
    m = S.Mesh.from_workload(w)
    M = m.assemble_M(S.MASS_DUAL)
    x = W.random_vector(w.n)
    ng = w.n_gamma
    h = np.concatenate([np.full(1000, 1e-3), np.full(3000, 1.0 / 3000), np.full(1000, 1e-3), np.full(3000, 1.0 / 3000)])
    hm, hp = np.roll(h, 1), np.roll(h, -1)
    vm, vp = hm / (hm + h), hp / (h + hp)
    for a in range(2):
        ht = 0.5
        Md = np.diag(ht * h * (2 + vm + vp) / 4)
        idx = np.arange(ng)
        Md[idx, (idx - 1) % ng] += ht * hm * vm / 4
        Md[idx, (idx + 1) % ng] += ht * hp * vp / 4
        for tr in (False, True):
            z = M.solve(cuda(x), torch.empty(w.n, dtype=torch.float64, device="cuda"), transpose=tr).cpu().numpy()
            ref = np.linalg.solve(Md.T if tr else Md, x[a * ng:(a + 1) * ng])
            assert relmax(z[a * ng:(a + 1) * ng], ref) <= 1e-12
