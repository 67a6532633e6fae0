"""CPU: the in-tree sm_100a library builds, loads without a GPU, and exports
every entry point declared in include/sutradhara_b200.h."""
import ctypes
import os
import re

from paper_2601_12967_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sutradhara_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares a signature for each of them
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_host_hash_matches_oracle():
    import numpy as np
    from oracle import oracle as O

    L = _lib.lib()
    assert L.sb_kv_root_hash() == O.root_hash()
    rng = np.random.default_rng(1)
    for n in (0, 1, 16, 33):
        t = rng.integers(0, 2**63, n, dtype=np.uint64)
        assert L.sb_kv_chain_hash_host(O.root_hash(), t.ctypes.data_as(_lib.U64P), n) == O.chain_hash(O.root_hash(), t)


def test_no_oracle_in_product():
    """The product never imports or links the CPU oracle (it is the checker)."""
    pkg = os.path.join(ROOT, "paper_2601_12967_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f
                assert "kvcache_oracle" not in src and "libkvoracle" not in src and "agentsim_ref" not in src, f
