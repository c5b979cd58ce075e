"""The native payload-tape encoder (csrc/tapes_py.cpp, TapeArena.add_many)
== the Python encoder (TapeArena.add, tape.py): byte-identical nodes, data,
refs, key tables and kept objects, over random JSON payloads (big ints,
integral / huge / subnormal / NaN / inf floats, -0.0, NFC-changing and
non-NFC-changing Unicode, lone surrogates, nesting) and payloads outside its
subset (tuples, dict / str / int subclasses, non-str keys) that it hands to
the Python path."""

import collections
import enum
import math
import random

import numpy as np
import pytest

from paper_2603_18897_b200 import tape
from paper_2603_18897_b200.tape import KeyTable, TapeArena

pytestmark = pytest.mark.skipif(tape._native_tapes is None, reason="extension not built")


class Color(enum.IntEnum):
    RED = 1


SCALARS = [None, True, False, 0, -7, 2 ** 80, -(2 ** 70), 1.5, -0.0, 0.0, 1e300, 1e16, 3.0,
           2.5e-320, float("nan"), float("inf"), -float("inf"), 0.1 + 0.2, 1 / 3, "", "x",
           "ünï", "é", "Å", "Å", "\ud800x", "a\x00b", "日本語"]


def rand_payload(rng, depth=0):
    r = rng.random()
    if depth > 4 or r < 0.4:
        return rng.choice(SCALARS)
    if r < 0.75:
        return {rng.choice(["k", "url", "é", "é", "x y", ""]) + str(i): rand_payload(rng, depth + 1)
                for i in range(rng.randint(0, 5))}
    return [rand_payload(rng, depth + 1) for _ in range(rng.randint(0, 5))]


def both(payloads, keep):
    ka, kb = KeyTable(), KeyTable()
    a, b = TapeArena(ka, keep_objects=keep), TapeArena(kb, keep_objects=keep)
    ia = [a.add(p) for p in payloads]
    ib = b.add_many(payloads)
    return a, b, ia, ib


def same(a, b):
    na, da, ra = a.arrays()
    nb, db, rb = b.arrays()
    assert np.array_equal(ra, rb)
    assert na.tobytes() == nb.tobytes()
    assert da.tobytes() == db.tobytes()
    assert a.keys.names == b.keys.names and a.keys.ids == b.keys.ids


@pytest.mark.parametrize("seed,keep", [(s, k) for s in range(8) for k in (False, True)])
def test_native_encoder_equals_python(seed, keep):
    rng = random.Random(seed)
    payloads = [rand_payload(rng) for _ in range(300)]
    a, b, ia, ib = both(payloads, keep)
    assert ia == ib
    same(a, b)
    if keep:
        assert len(a._objs) == len(b._objs)
        assert all(x is y or (isinstance(x, float) and math.isnan(x) and x is y)
                   for x, y in zip(a._objs, b._objs))


def test_outside_the_native_subset_takes_the_python_path():
    odd = [(1, 2), {"a": (1,)}, collections.OrderedDict(a=1), Color.RED, {"k": Color.RED},
           [1, [2, (3,)]], {"s": type("S", (str,), {})("v")}]
    good = [{"a": 1}, [1, 2.5], "ü"]
    payloads = [x for pair in zip(good * 3, odd) for x in pair]
    # the Python path raises for tuples: add_many raises the same error
    with pytest.raises(TypeError):
        TapeArena(keep_objects=False).add_many(payloads)
    ok = [p for p in payloads if not _has_tuple(p)]
    assert len(ok) > len(good)
    for keep in (False, True):
        a, b, ia, ib = both(ok, keep)
        assert ia == ib
        same(a, b)


def _has_tuple(p):
    if isinstance(p, tuple):
        return True
    if isinstance(p, dict):
        return any(_has_tuple(v) for v in p.values())
    if isinstance(p, list):
        return any(_has_tuple(v) for v in p)
    return False


def test_non_str_keys_raise_like_the_python_path():
    arena = TapeArena(keep_objects=False)
    with pytest.raises(TypeError):
        arena.add_many([{1: "x"}])
