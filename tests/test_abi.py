"""The C-ABI library loads, exports every symbol include/*.h declares, and its
host-only entry points (seeding, jump-ahead, argument validation) behave --
no GPU needed."""

import ctypes
import glob
import json
import os
import re

import numpy as np
import pytest

from paper_1207_6365_b200 import _lib
from paper_1207_6365_b200.sketch import derived_seed, pcg64_state, seed_words

from .conftest import GOLDEN, ROOT


def declared_symbols():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(hdr).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(skt_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    decl = declared_symbols()
    assert decl, "no declarations found"
    assert decl == set(_lib.EXPORTS)
    for name in decl:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.skt_version()


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_seedseq_and_pcg64_seed_match_numpy():
    for row in json.load(open(os.path.join(GOLDEN, "seeds.json"))):
        ent = seed_words(row["seed"])
        key = np.asarray(row["key"], dtype=np.uint32)
        out = np.zeros(4, dtype=np.uint32)
        assert _lib.lib().skt_seedseq_generate(
            ent.ctypes.data, len(ent), key.ctypes.data if len(key) else None, len(key), out.ctypes.data, 4
        ) == 0
        assert out.tolist() == row["gen4"]
        st = pcg64_state(row["seed"], row["key"])
        assert (st.state_hi << 64 | st.state_lo) == int(row["state"])
        assert (st.inc_hi << 64 | st.inc_lo) == int(row["inc"])


@pytest.mark.parametrize("delta", [0, 1, 2, 31, 32, 1000, 2**40 + 3])
def test_pcg64_advance_matches_numpy(delta):
    st = pcg64_state(7, (0, 0))
    g = np.random.PCG64(np.random.SeedSequence(7, spawn_key=(0, 0)))
    g.advance(delta)
    assert _lib.lib().skt_pcg64_advance(ctypes.byref(st), delta) == 0
    want = g.state["state"]
    assert (st.state_hi << 64 | st.state_lo) == want["state"]


def test_derived_seed():
    for seed, key in [(0, (1,)), (5, (3,)), (2**70, (100, 2))]:
        assert derived_seed(seed, *key) == int(np.random.SeedSequence(seed, spawn_key=key).generate_state(1)[0])


def test_negative_seed_rejected():
    with pytest.raises(ValueError):
        seed_words(-1)


def test_device_entry_points_validate_before_touching_cuda():
    L = _lib.lib()
    st = _lib.SktPcg64()
    # t = 0 and t > 2^32 are EINVAL
    assert L.skt_hash_signs(ctypes.byref(st), ctypes.byref(st), 0, 10, 0, None, None, None, 0, None) == _lib.SKT_EINVAL
    assert L.skt_hash_signs(ctypes.byref(st), ctypes.byref(st), 0, 10, 2**32 + 1, None, None, None, 0, None) == _lib.SKT_EINVAL
    assert "bad arguments" in _lib.last_error()
    nb = ctypes.c_size_t()
    assert L.skt_plan_workspace(2**31, 10, 0, ctypes.byref(nb)) == _lib.SKT_EINVAL
    assert L.skt_plan_workspace(1000, 10, 9, ctypes.byref(nb)) == _lib.SKT_EINVAL
    assert L.skt_plan_workspace(1000, 1 << 16, 0, ctypes.byref(nb)) == 0 and nb.value > 0
    assert L.skt_plan_workspace(1000, 1, 0, ctypes.byref(nb)) == 0 and nb.value == 0
    assert L.skt_plan_workspace(1000, 256, 8, ctypes.byref(nb)) == 0 and nb.value == 0
    # lda < d
    assert L.skt_apply_dense(None, None, 4, 10, None, 0, 8, 4, None, 1, 8, None, None) == _lib.SKT_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.SKT_EINVAL)
    with pytest.raises(_lib.SketchError):
        _lib.check(_lib.SKT_ECUDA)


def test_no_cuda_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1207_6365_b200 import SparseEmbedding

    with pytest.raises(Exception):
        SparseEmbedding(10, 4, seed=0)
