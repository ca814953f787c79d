"""CPU-only checks of the native library: it loads, exports every C-ABI symbol of
include/stbem.h, validates descriptors before touching CUDA, fails loudly without a GPU, and its
host-side cyclic K_P plan (Fig. 3) satisfies the SPEC invariants."""
import os
import re

import numpy as np
import pytest

from paper_1811_05224_b200 import stbem as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "stbem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bem_[A-Za-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = S.lib()
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(S.symbols())        # the binding covers the whole ABI


def test_version_and_launch_counter():
    assert b"sm_100a" in S.lib().bem_version()
    S.launch_count(reset=True)
    assert S.launch_count() == 0


def _ok_plan(P):
    own = S.plan_build(P)
    blocks = [(i, j) for i in range(P) for j in range(i + 1)]
    assert all(0 <= own[i, j] < P for i, j in blocks)            # tiling: every block owned once
    assert all(own[i, j] == -1 for i in range(P) for j in range(i + 1, P))
    for p in range(P):
        assert own[p, p] == p                                       # one diagonal block each
    for (i, j) in blocks:                                           # rotation symmetry
        p = own[i, j]
        u, v = (i - p) % P, (j - p) % P
        assert own[max(u, v), min(u, v)] == 0 or (P % 2 == 0 and (i - j) == P // 2)
    return np.bincount(own[own >= 0].ravel(), minlength=P)


@pytest.mark.parametrize("P", list(range(1, 65)))
def test_cyclic_plan_invariants(P):
    counts = _ok_plan(P)
    assert counts.sum() == P * (P + 1) // 2
    assert counts.max() - counts.min() <= 1


def test_cyclic_plan_examples():
    assert sorted(_ok_plan(4).tolist()) == [2, 2, 3, 3]             # SPEC S:327 (Fig. 3)
    assert _ok_plan(7).tolist() == [4] * 7
    assert S.plan_generator(7) == [0, 1, 3]
    assert S.plan_generator(8) == [0, 1, 2, 4]
    assert sorted(_ok_plan(8).tolist()) == [4] * 4 + [5] * 4
    assert len(S.plan_generator(16)) == 5


def test_plan_distinct_slices_bound():
    # max distinct slices per worker <= ceil((1 + sqrt(8P+1))/2) + 1
    for P in range(1, 65):
        own = S.plan_build(P)
        bound = int(np.ceil((1 + np.sqrt(8 * P + 1)) / 2)) + 1
        for p in range(P):
            sl = {x for i in range(P) for j in range(i + 1) if own[i, j] == p for x in (i, j)}
            assert len(sl) <= bound


def test_slice_ranges():
    assert S.slice_ranges(8, 4) == [0, 2, 4, 6, 8]
    assert S.slice_ranges(5, 2) == [0, 3, 5]
    with pytest.raises(S.BemError) as e:
        S.slice_ranges(4, 8)
    assert e.value.status == S.BEM_E_INVALID


SQ = [(0, 0), (1, 0), (1, 1), (0, 1)]


@pytest.mark.parametrize("kw,msg", [
    (dict(alpha=0.0), "alpha"),
    (dict(t_breaks=[0.0, 0.5, 0.5, 1.0]), "increasing"),
    (dict(t_breaks=[0.1, 0.5, 1.0]), "t_breaks[0]"),
    (dict(vertices=SQ[::-1]), "counter-clockwise"),
    (dict(vertices=[(0, 0), (3, 0), (3, 3), (1, -1), (0, 3)], segments_per_side=[1, 1, 1, 1, 1]), "simple"),
    (dict(n_slices=9), "n_slices"),
    (dict(segments_per_side=[2, 0, 2, 2]), "segments_per_side"),
])
def test_mesh_descriptor_validation(kw, msg):
    args = dict(vertices=SQ, segments_per_side=[2, 2, 2, 2], t_breaks=np.linspace(0, 1, 5), alpha=1.0, n_slices=1)
    args.update(kw)
    with pytest.raises(S.BemError) as e:
        S.Mesh(**args)
    assert e.value.status == S.BEM_E_INVALID and msg in str(e.value)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(S.BemError) as e:
        S.Mesh(SQ, [2, 2, 2, 2], np.linspace(0, 1, 5), 1.0)
    assert e.value.status == S.BEM_E_CUDA


def test_diag_fp64_rate_rejects_bad_arguments():
    """bem_diag_fp64_rate validates before touching the device (0 < seconds <= 60)"""
    for sec in (0.0, -1.0, 61.0):
        with pytest.raises(S.BemError) as e:
            S.diag_fp64_rate(sec)
        assert e.value.status == S.BEM_E_INVALID
