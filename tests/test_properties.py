"""Property-based checks (hypothesis) of the host-side logic of the C ABI and of oracle
invariants.  CPU only."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
import paper_1505_01998_b200 as kb


@settings(max_examples=300, deadline=None)
@given(st.integers(min_value=0, max_value=2 ** 52))
def test_tile_map_inverts_column_major_numbering(bx):
    # Eq. 42-43 + integer fix-up: bx lies in column l, which starts at l(l+1)/2
    l, q = kb.tile_coords(bx)
    assert l * (l + 1) // 2 <= bx < (l + 1) * (l + 2) // 2
    assert q == bx - l * (l + 1) // 2 and 0 <= q <= l


limb = st.integers(min_value=-(2 ** 40), max_value=2 ** 40)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.tuples(limb, limb, limb), min_size=1, max_size=40), st.integers(min_value=0, max_value=120))
def test_fixed_point_addition_is_exact_and_order_free(vals, S):
    fs = [kb.Fixed(hi=a, mid=b, lo=c, scale_exp=S) for a, b, c in vals]
    acc = fs[0]
    for f in fs[1:]:
        acc = kb.fixed_add(acc, f)
    rev = fs[-1]
    for f in reversed(fs[:-1]):
        rev = kb.fixed_add(rev, f)
    assert (acc.hi, acc.mid, acc.lo) == (rev.hi, rev.mid, rev.lo)
    exact = sum(a * 2 ** 80 + b * 2 ** 40 + c for a, b, c in vals)
    assert (acc.hi * 2 ** 80 + acc.mid * 2 ** 40 + acc.lo) == exact
    v = kb.fixed_value(acc)
    assert v == float(exact) * 2.0 ** -S or abs(v - exact * 2.0 ** -S) <= abs(exact * 2.0 ** -S) * 2 ** -52


@settings(max_examples=200, deadline=None)
@given(st.sampled_from([kb.SUM_PSI4, kb.SUM_PSI6, kb.SUM_PSI8, kb.SUM_LSCV_h, kb.SUM_LSCV_H]),
       st.integers(min_value=1, max_value=2 ** 31 - 1), st.integers(min_value=1, max_value=16),
       st.integers(min_value=1, max_value=64))
def test_shard_ranges_partition_the_tile_grid(kind, n, d, world):
    # round-robin chunks: counts add up, balanced to one chunk, and the local -> id map of every rank
    # hits exactly the ids whose chunk index is congruent to the rank (checked at both ends)
    counts = []
    for r in range(world):
        T, tot, cnt, chunk = kb.shard_tiles(kind, n, d, r, world)
        nb = (n + T - 1) // T
        assert tot == nb * (nb + 1) // 2
        counts.append(cnt)
        if world > 1:
            assert chunk == 16
            for i in {0, cnt - 1, cnt // 2} - {-1}:
                if 0 <= i < cnt:
                    t = kb.shard_tile(i, r, world)
                    assert 0 <= t < tot and (t // chunk) % world == r and t % chunk == i % chunk
        else:
            assert cnt == tot and kb.shard_tile(5, 0, 1) == 5
    assert sum(counts) == tot
    assert max(counts) - min(counts) <= 16


@settings(max_examples=40, deadline=None)
@given(st.lists(st.floats(min_value=-5, max_value=5, allow_nan=False), min_size=2, max_size=25),
       st.floats(min_value=0.05, max_value=3.0), st.sampled_from([4, 6, 8]))
def test_oracle_psi_sign_and_permutation(xs, g, r):
    x = np.array(xs)
    v = oracle.psi_r(x, r, g)
    assert (v > 0) == (r % 4 == 0)                                   # reading Z11
    assert abs(oracle.psi_r(x[::-1].copy(), r, g) - v) <= 1e-12 * abs(v) + 1e-300
