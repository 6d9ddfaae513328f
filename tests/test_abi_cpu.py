"""The C-ABI library loads, exports every symbol include/evox.h declares, and
validates arguments synchronously -- all without a GPU (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2301_12457_b200 as ev
from paper_2301_12457_b200 import evox as E

HEADER = os.path.join(ROOT, "include", "evox.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(evox_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = ev.lib()
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), f"libevox.so does not export {n}"
    # the binding declares a signature for every entry point of the header
    assert set(names) == set(E.SIGNATURES), set(names) ^ set(E.SIGNATURES)


def test_version_and_abi():
    assert "evox" in ev.version()
    assert ev.lib().evox_abi_version() == 2


@pytest.mark.parametrize("pop,world", [(100, 4), (10, 4), (7, 3), (1, 1), (5, 8), (1000003, 8)])
def test_shard_rows(pop, world):
    """P=100,W=4 -> (25,25,25,25); P=10,W=4 -> (3,3,2,2); contiguous, sizes differ <= 1."""
    parts = [ev.shard_rows(pop, world, r) for r in range(world)]
    sizes = [n for _, n in parts]
    assert sum(sizes) == pop and max(sizes) - min(sizes) <= 1
    assert parts[0][0] == 0
    for (r0, n), (r1, _) in zip(parts, parts[1:]):
        assert r1 == r0 + n
    if (pop, world) == (100, 4):
        assert sizes == [25, 25, 25, 25]
    if (pop, world) == (10, 4):
        assert sizes == [3, 3, 2, 2]


def test_shard_rows_invalid():
    with pytest.raises(E.InvalidArgument):
        ev.shard_rows(10, 0, 0)
    with pytest.raises(E.InvalidArgument):
        ev.shard_rows(10, 2, 2)


def _init(pop=10, dim=3, lb=None, ub=None, w=0.6, opts=None):
    lb = np.full(dim, -1, np.float32) if lb is None else np.asarray(lb, np.float32)
    ub = np.full(dim, 1, np.float32) if ub is None else np.asarray(ub, np.float32)
    h = ctypes.c_void_p()
    st = ev.lib().evox_pso_init(pop, dim, lb.ctypes.data, ub.ctypes.data, w, 2.5, 0.8, 0,
                                ctypes.byref(opts) if opts is not None else None, ctypes.byref(h))
    return st, h.value


def test_pso_init_validation_before_device_work():
    assert _init(pop=0)[0] == E.INVALID_ARGUMENT
    assert _init(dim=0, lb=np.zeros(1), ub=np.ones(1))[0] == E.INVALID_ARGUMENT
    assert _init(lb=[0, 0, 1], ub=[1, 1, 1])[0] == E.INVALID_ARGUMENT  # lb == ub
    assert _init(lb=[0, np.nan, 0], ub=[1, 1, 1])[0] == E.INVALID_ARGUMENT
    assert _init(lb=[0, 0, 0], ub=[1, np.inf, 1])[0] == E.INVALID_ARGUMENT
    assert _init(w=float("nan"))[0] == E.INVALID_ARGUMENT
    assert "finite" in ev.evox.last_error()
    o = E.EvoxOpts()
    o.world, o.rank = 2, 2
    assert _init(opts=o)[0] == E.INVALID_ARGUMENT
    assert _init(pop=1 << 33)[0] == E.SHAPE


def test_cso_init_validation():
    lb, ub = np.full(4, -1, np.float32), np.full(4, 1, np.float32)
    h = ctypes.c_void_p()
    L = ev.lib()
    assert L.evox_cso_init(1, 4, lb.ctypes.data, ub.ctypes.data, 0.0, 0, 0, None,
                           ctypes.byref(h)) == E.INVALID_ARGUMENT
    assert L.evox_cso_init(10, 4, lb.ctypes.data, ub.ctypes.data, 0.0, 1, 0, None,
                           ctypes.byref(h)) == E.INVALID_ARGUMENT
    o = E.EvoxOpts()
    o.world, o.rank = 2, 0
    nid = (ctypes.c_uint8 * 128)()
    o.nccl_id = ctypes.addressof(nid)
    # blocks straddling shards need peer connection: not with world > 8 or a workspace
    o.world = 9
    assert L.evox_cso_init(90, 4, lb.ctypes.data, ub.ctypes.data, 0.0, 90, 0, ctypes.byref(o),
                           ctypes.byref(h)) == E.CONFIG


def test_eval_validation():
    L = ev.lib()
    assert L.evox_eval(9, None, 1, 1, 4, None, None) == E.INVALID_ARGUMENT
    assert L.evox_eval(0, None, 1, 5, 6, None, None) == E.SHAPE
    assert L.evox_eval(0, None, 1, 5, 4, None, None) == E.SHAPE
    assert L.evox_eval(0, None, 0, 5, 8, None, None) == E.OK  # empty population: no-op
    assert L.evox_eval(0, None, 3, 5, 8, None, None) == E.INVALID_ARGUMENT


def test_null_handles():
    L = ev.lib()
    assert L.evox_pso_destroy(None) == E.OK
    assert L.evox_cso_destroy(None) == E.OK
    assert L.evox_pso_step(None, 0, 1) == E.INVALID_ARGUMENT
    assert L.evox_pso_sync(None) == E.INVALID_ARGUMENT
    assert L.evox_cso_step(None, 0, 1) == E.INVALID_ARGUMENT
    assert L.evox_pso_tell(None, None) == E.INVALID_ARGUMENT


def test_workspace_bytes():
    b1 = ev.PSO.workspace_bytes(1000, 10)
    assert b1 >= 3 * 1000 * 12 * 4
    b2 = ev.PSO.workspace_bytes(1000, 10, world=4, rank=1)
    assert b2 < b1
    assert ev.CSO.workspace_bytes(1000, 10) < b1
    with pytest.raises(E.ShapeError):
        ev.PSO.workspace_bytes(0, 10)


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle and has no CPU compute path."""
    pkg = os.path.join(ROOT, "paper_2301_12457_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(Exception):
            ev.evaluate("sphere", torch.zeros(4, 4))
