"""The multi-rank path with the real kernels on ONE GPU: G emulated ranks (bem_comm_create_group,
one host thread each, SPMD) own the blocks of the cyclic K_P plan with P = 2G temporal slices
 and sum their partial products with the group all-reduce.
Against the single-rank path: products and the fused right-hand side to rounding, the GMRES
solution to the density tolerance with the same iteration count, every rank bitwise identical
(the all-reduce gives all ranks the same sums, so they take identical decisions)."""
import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1811_05224_b200 import stbem as S  # noqa: E402


def relmax(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def step(w, n_slices, comm, x_host):
    """one rank's SPMD sequence: assemble, products, fused rhs, preconditioned solve"""
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        m = S.Mesh.from_workload(w, n_slices=n_slices, comm=comm)
        V, D = m.assemble_V(stream=st), m.assemble_D(stream=st)
        Mp, Md = m.assemble_M(S.MASS_PRIMAL, stream=st), m.assemble_M(S.MASS_DUAL, stream=st)
        x = torch.tensor(x_host, dtype=torch.float64, device="cuda")
        Vx, Dx = torch.empty_like(x), torch.empty_like(x)
        V.matvec(x, Vx, stream=st)
        D.matvec(x, Dx, stream=st)
        g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
        b = torch.empty_like(g)
        S.rhs_fused(m, Mp, g, b, stream=st)
        wv = torch.zeros_like(g)
        rep = S.solve_gmres(V, b, wv, D=D, M=Md, precond=2, rel_tol=w.tol, max_iter=200, history=False, stream=st)
        st.synchronize()
        out = {"Vx": Vx.cpu().numpy(), "Dx": Dx.cpu().numpy(), "b": b.cpu().numpy(), "w": wv.cpu().numpy(),
               "rep": rep, "blocks": m.info.n_owned_blocks, "entries": m.info.entries_owned}
        for A in (V, D, Mp, Md):
            A.close()
        m.close()
    return out


_single = {}


def single(name):
    if name not in _single:
        w = W.get(name)
        _single[name] = step(w, 1, None, W.random_vector(w.n))
    return _single[name]


@pytest.mark.parametrize("name,G", [("S32", 2), ("S32", 4), ("S32", 8), ("C2", 2), ("C2", 4)])
def test_emulated_ranks_match_single_rank(name, G):
    w = W.get(name)
    ref = single(name)
    comms = S.Comm.group(G, 0)
    res, errs = [None] * G, []

    def run(r):
        try:
            res[r] = step(w, 2 * G, comms[r], W.random_vector(w.n))
        except Exception as e:   # noqa: BLE001
            errs.append(repr(e))
    th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    for c in comms:
        c.close()
    assert not errs, errs
    # the cyclic plan gives every rank its share: P(P+1)/2 blocks in total, entries summing to the whole
    P = 2 * G
    assert sum(r["blocks"] for r in res) == P * (P + 1) // 2
    assert sum(r["entries"] for r in res) == w.n_gamma ** 2 * w.n_steps * (w.n_steps + 1) // 2
    for r in range(1, G):                              # identical sums on every rank
        for k in ("Vx", "Dx", "b", "w"):
            assert np.array_equal(res[r][k], res[0][k]), (r, k)
    out = res[0]
    for k in ("Vx", "Dx", "b"):
        assert relmax(out[k], ref[k]) <= 1e-13, k
    assert out["rep"]["status"] == "OK"
    assert out["rep"]["iterations"] == ref["rep"]["iterations"], (out["rep"], ref["rep"])
    assert relmax(out["w"], ref["w"]) <= 1e-10
    assert out["rep"]["seconds_comm"] > 0.0            # the collectives were timed


@pytest.mark.parametrize("name,G", [("S32", 2), ("S32", 4), ("C2", 4)])
def test_solo_rank_partials_sum_to_the_product(name, G):
    """each rank of the cyclic plan alone on the GPU (bem_comm_create_solo, P = 2G): its owned
    blocks' partial products of V_h, D_h and of K_h g sum over the ranks to the single-rank results
    (the verdict's partial-product check, with the real kernels)"""
    w = W.get(name)
    ref = single(name)
    x = torch.tensor(W.random_vector(w.n), dtype=torch.float64, device="cuda")
    g = torch.tensor(W.dirichlet_data(w), dtype=torch.float64, device="cuda")
    sums = {k: np.zeros(w.n) for k in ("Vx", "Dx", "Kg")}
    m0 = S.Mesh.from_workload(w)
    half_mg = torch.zeros_like(g)
    m0.assemble_M(S.MASS_PRIMAL).matvec(g, half_mg, a=0.5)
    for r in range(G):
        c = S.Comm.solo(G, r, 0)
        m = S.Mesh.from_workload(w, n_slices=2 * G, comm=c)
        V, D = m.assemble_V(), m.assemble_D()
        y = torch.empty_like(x)
        V.matvec(x, y)
        sums["Vx"] += y.cpu().numpy()
        D.matvec(x, y)
        sums["Dx"] += y.cpu().numpy()
        b = torch.empty_like(g)
        S.rhs_fused(m, m.assemble_M(S.MASS_PRIMAL), g, b)
        sums["Kg"] += (b - half_mg).cpu().numpy()
        with pytest.raises(S.BemError):
            S.solve_gmres(V, b, torch.zeros_like(g), D=D, M=m.assemble_M(S.MASS_DUAL), precond=2)
        V.close(); D.close(); m.close(); c.close()
    torch.cuda.synchronize()
    assert relmax(sums["Vx"], ref["Vx"]) <= 1e-13
    assert relmax(sums["Dx"], ref["Dx"]) <= 1e-13
    assert relmax(sums["Kg"] + half_mg.cpu().numpy(), ref["b"]) <= 1e-13


@pytest.mark.parametrize("name,G", [("S32", 3), ("C2", 4), ("C2", 8)])
def test_distributed_records_entries_bitwise(name, G):
    """emulated ranks compute 1/G of the pair records each and all-gather them (assemble.cu,
    DESIGN.md section 4.5): every owned entry equals the single-rank entry bit for bit and every
    entry is owned by exactly one rank (the others read 0), so the sum over ranks is exact"""
    w = W.get(name)
    rng = np.random.default_rng(7)
    rows = rng.integers(0, w.n, 40000)
    cols = rng.integers(0, w.n, 40000)
    cols = np.where(cols // w.n_gamma > rows // w.n_gamma, rows, cols)   # causal entries (b <= a)
    m0 = S.Mesh.from_workload(w)
    ref = {}
    for k, f in (("V", m0.assemble_V), ("D", m0.assemble_D)):
        A = f()
        ref[k] = A.entries(rows, cols)
        A.close()
    m0.close()
    comms = S.Comm.group(G, 0)
    got, errs = [None] * G, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                m = S.Mesh.from_workload(w, n_slices=2 * G, comm=comms[r])
                out = {}
                for k, f in (("V", m.assemble_V), ("D", m.assemble_D)):
                    A = f(stream=st)
                    out[k] = A.entries(rows, cols)
                    A.close()
                m.close()
            got[r] = out
        except Exception as e:   # noqa: BLE001
            errs.append(repr(e))
    th = [threading.Thread(target=run, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    for c in comms:
        c.close()
    assert not errs, errs
    for k in ("V", "D"):
        nz = np.stack([got[r][k] != 0.0 for r in range(G)])
        assert np.all(nz.sum(axis=0) <= 1), k                 # one owner per entry
        tot = sum(got[r][k] for r in range(G))
        assert np.array_equal(tot, ref[k]), (k, relmax(tot, ref[k]))
