"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/kde.h declares,
and its host-side pieces (tile map of Eq. 42-43, fixed-point arithmetic) are right.  No compute
call touches a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_1505_01998_b200 as kb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "kde.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kde_[a-zA-Z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = kb.lib()
    decl = _declared()
    assert len(decl) >= 18
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(kb.EXPORTS) == decl


def test_tile_map_matches_enumeration():
    # Eq. 42-43 with the integer fix-up == plain column-major enumeration
    l, q = oracle.tile_enumerate(200_000)
    for bx in list(range(0, 5000)) + list(range(5000, 200_000, 997)):
        assert kb.tile_coords(bx) == (l[bx], q[bx]), bx


@pytest.mark.parametrize("T", [256, 512, 2048])
def test_tile_map_near_perfect_squares_large_ids(T):
    # l(l+1)/2 <= bx < (l+1)(l+2)/2 exactly, including ids past 2^24 where an fp32 sqrt breaks
    # and up to the tile count of n = 2^31 - 1 (reading Z13).
    nb = (2 ** 31 - 1 + T - 1) // T
    last = nb * (nb + 1) // 2 - 1
    ids = [2 ** 24 - 1, 2 ** 24, 2 ** 24 + 1, last - 1, last]
    for L in [4095, 4096, 65535, 1 << 20, nb - 1]:
        s = L * (L + 1) // 2
        ids += [s - 1, s, s + 1, s + L]
    for bx in ids:
        if bx < 0 or bx > last:
            continue
        l, q = kb.tile_coords(bx)
        assert l * (l + 1) // 2 <= bx < (l + 1) * (l + 2) // 2 and q == bx - l * (l + 1) // 2 and 0 <= q <= l


def test_fixed_point_value_and_exact_add():
    S = 60
    a = kb.Fixed(hi=1, mid=3, lo=-5, scale_exp=S)
    b = kb.Fixed(hi=-2, mid=(1 << 40) - 1, lo=7, scale_exp=S)
    va = (2 ** 80 + 3 * 2 ** 40 - 5) * 2.0 ** -S
    vb = (-2 * 2 ** 80 + ((1 << 40) - 1) * 2 ** 40 + 7) * 2.0 ** -S
    assert kb.fixed_value(a) == pytest.approx(va, rel=1e-15)
    c = kb.fixed_add(a, b)
    assert (c.hi, c.mid, c.lo) == (-1, 3 + (1 << 40) - 1, 2)
    assert kb.fixed_value(c) == pytest.approx(va + vb, rel=1e-15)


def test_default_opts_and_workspace_size():
    o = kb.default_opts()
    assert (o.n_grid, o.range_factor, o.max_iter, o.tol_rel, o.penalty, o.speculative) == (150, 4.0, 500, 1e-7, 1e300, 0)
    L = kb.lib()
    assert L.kde_workspace_bytes(1 << 20, 1, 1) >= (1 << 20) * 4
    assert L.kde_workspace_bytes(0, 1, 1) == 0


def test_null_context_is_rejected():
    L = kb.lib()
    out = ctypes.c_double()
    g = ctypes.c_double(1.0)
    assert L.kde_psi_r(None, None, 10, 4, ctypes.byref(g), 1, ctypes.byref(out)) == 1
    assert L.kde_last_error(None) == b"null context"
    # the mode setters reject a null context too (no GPU needed)
    assert L.kde_set_precision(None, 1) == 1
    assert L.kde_set_profiling(None, 1) == 1
    assert L.kde_set_host_allreduce(None, kb.HOST_ALLREDUCE_FN(lambda p, n, u: 0), None) == 1


def test_binding_marshals_host_and_rejects_other_dtypes():
    # host fp64 arrays are passed as host pointers (the library copies them to the GPU inside
    # the call); anything that is not fp64 is refused before the C ABI is reached
    s = kb._samples(np.zeros(4))
    assert s.shape == (1, 4) and s.host and s.ptr.value
    with pytest.raises(TypeError):
        kb._samples(np.zeros((1, 4), dtype=np.float32))
    with pytest.raises(TypeError):
        kb._samples([0.0, 1.0])
