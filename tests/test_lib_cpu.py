"""C-ABI library checks that need no GPU: it loads, exports every symbol the header
declares, its host topology is bit-exact with the oracle, and it validates arguments."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import topology as T

import __graft_entry__ as entry

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "crossover_sgd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(cs_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol():
    syms = _header_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(cs.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(cs.exported_symbols()) == syms


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", cs.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n", list(range(2, 17)) + [31, 32, 33, 63, 64, 65, 100, 257])
def test_host_topology_bit_exact_vs_oracle(n):
    k = 4 if n > 64 else 8
    cs.cs_init(n, 1, k, 0xDEADBEEF12345678)
    for step in [0, 1, 2, 7, 100, 4_000_000_000]:
        assert np.array_equal(cs.cs_topology(step, n, k), T.topology(0xDEADBEEF12345678, step, n, k)), (n, step)


def test_host_topology_many_steps_bit_exact():
    # P5: 10^4 (step, segment) pairs across sizes
    total = 0
    for n, k, seed in [(8, 32, 0), (16, 8, 1), (64, 4, 2**63 + 5), (3, 16, 7)]:
        cs.cs_init(n, 1, k, seed)
        steps = 2500 // k + 1
        for step in range(0, steps * 3, 3):
            assert np.array_equal(cs.cs_topology(step, n, k), T.topology(seed, step, n, k))
            total += k
    assert total >= 10_000


def test_host_hier_topology_bit_exact():
    cs.cs_init(16, 4, 5, 99)
    for step in range(20):
        assert np.array_equal(cs.cs_topology_hier(step, 4, 5), T.topology(99, step, 4, 5, T.TAG_HIER))
    cs.cs_init(8, 2, 3, 1)
    assert np.all(cs.cs_topology_hier(5, 2, 3) == np.array([[1, 0]] * 3))


def test_segment_bounds_match_oracle():
    for d, k in [(1_000_000, 4), (11_689_512, 8), (25_557_032, 16), (97, 3), (32, 1)]:
        cs.cs_init(2, 2, k, 0)
        assert np.array_equal(cs.cs_segment_bounds(d, k), T.segment_bounds(d, k))


@pytest.mark.parametrize("args,code", [((1, 1, 1, 0), -1), ((1025, 1, 1, 0), -1), ((6, 4, 1, 0), -2),
                                       ((6, 0, 1, 0), -2), ((4, 2, 0, 0), -3)])
def test_init_errors(args, code):
    with pytest.raises(cs.CSError) as e:
        cs.cs_init(*args)
    assert e.value.code == code


def test_uninitialised_and_unbound_errors():
    cs.cs_finalize()
    with pytest.raises(cs.CSError) as e:
        cs.cs_topology(0, 4, 1)
    assert e.value.code == -7
    cs.cs_init(4, 4, 2, 0)
    with pytest.raises(cs.CSError) as e:
        cs.cs_gossip_step(16, 16, 16, 0.1, 0.9)
    assert e.value.code == -8
    with pytest.raises(cs.CSError) as e:
        cs.cs_test_set_topology(np.zeros((2, 4), np.int32))
    assert e.value.code == -8
    with pytest.raises(cs.CSError) as e:
        cs.cs_topology(2**32, 4, 2)
    assert e.value.code == -11


def test_bind_layout_validation_before_any_cuda_call():
    cs.cs_init(4, 4, 2, 0)
    for d, ld, ptr, code in [(100, 102, 256, -4), (100, 96, 256, -4), (100, 100, 8, -4),
                             (0, 4, 256, -4), (32, 32, 256, -3)]:
        with pytest.raises(cs.CSError) as e:
            cs.cs_bind(ptr, d, ld)
        assert e.value.code == code, (d, ld, ptr)
    with pytest.raises(cs.CSError) as e:
        cs.cs_bind(256, 64, 64, proc_rank=0, nprocs=3)
    assert e.value.code == -1


def test_segment_bounds_errors():
    cs.cs_init(4, 4, 3, 0)
    with pytest.raises(cs.CSError) as e:
        cs.cs_segment_bounds(64, 3)
    assert e.value.code == -3


def test_host_segment_plan_matches_oracle():
    # C++ cs_segment_plan (binary search + greedy) vs oracle/lars.segment_plan (bit-exact)
    from oracle.lars import segment_plan
    import synth
    rng = np.random.default_rng(7)
    for _ in range(200):
        L = int(rng.integers(1, 30))
        sizes = [int(v) for v in rng.integers(1, 50, size=L) * 4]
        for k in sorted({1, L, int(rng.integers(1, L + 1))}):
            assert cs.cs_segment_plan(sizes, k).tolist() == segment_plan(sizes, k), (sizes, k)
    sizes, _ = synth.resnet50_layers()
    for k in (2, 8, 18, 161):
        assert cs.cs_segment_plan(sizes, k).tolist() == segment_plan(sizes, k), k
    for bad_k in (0, 162):
        with pytest.raises(cs.CSError):
            cs.cs_segment_plan(sizes, bad_k)


def test_host_exponential_topology_matches_oracle():
    from oracle.sgp import exponential_topology
    for n, k in [(2, 1), (8, 3), (64, 1), (1024, 2)]:
        cs.cs_init(n, n, k, 5)
        cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
        for t in [0, 1, 2, 9, 2**32 - 1]:
            assert np.array_equal(cs.cs_topology(t, n, k), exponential_topology(t, n, k))
        cs.cs_set_topology_kind(cs.TOPO_CROSSOVER)
        assert np.array_equal(cs.cs_topology(3, n, k), T.topology(5, 3, n, k))
    cs.cs_init(12, 12, 1, 0)
    with pytest.raises(cs.CSError) as e:
        cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
    assert e.value.code == -12
    with pytest.raises(cs.CSError):
        cs.cs_set_topology_kind(7)


def test_abi_version():
    assert cs.cs_version() == 300  # 0.3.0


def test_build_id_matches_sources():
    # the library in the tree was built from exactly these sources (build()
    # used to trust file times): __graft_entry__.build() rebuilds on any mismatch
    import __graft_entry__ as entry
    assert cs.cs_build_id() == entry.source_hash() == entry.built_id()


def test_binding_constants_match_header():
    """Every status code and constant the binding names equals the header's #define."""
    txt = open(os.path.join(ROOT, "include", "crossover_sgd.h")).read()
    defs = {k: int(v) for k, v in re.findall(r"^#define\s+(CS_\w+)\s+(-?\d+)", txt, flags=re.M)}
    for code, name in cs.STATUS.items():
        assert defs[name] == code, name
    assert set(cs.STATUS.values()) == {k for k in defs if k == "CS_OK" or k.startswith("CS_E")}
    for name in ("CS_MAX_WORLD", "CS_QUANTUM", "CS_IPC_HANDLE_BYTES", "CS_TAG_FLAT", "CS_TAG_HIER",
                 "CS_PATH_AUTO", "CS_PATH_REG", "CS_PATH_TMA", "CS_PATH_PEER"):
        assert getattr(cs, name) == defs[name], name
    for name in ("TOPO_CROSSOVER", "TOPO_EXPONENTIAL", "WIRE_FP32", "WIRE_BF16"):
        assert getattr(cs, name) == defs["CS_" + name], name


def test_nccl_group_id_and_h1_setters_need_a_binding():
    # cs_nccl_unique_id is the host half of the NCCL h1 setup (reading B-8): NCCL loaded at run
    # time, a fresh 128-byte id per call; the setters that join or register a group need a
    # bound library (and so a GPU)
    try:
        a, b = cs.cs_nccl_unique_id(), cs.cs_nccl_unique_id()
    except cs.CSError as e:  # no usable libnccl on this host
        pytest.skip(f"NCCL unavailable: {e}")
    assert len(a) == cs.CS_NCCL_ID_BYTES == 128 and a != b
    cs.cs_finalize()
    for call in (lambda: cs.cs_set_hier_nccl(a), lambda: cs.cs_set_multicast(0, 0, 0), cs.cs_multicast_bytes):
        with pytest.raises(cs.CSError) as e:
            call()
        assert e.value.code == -7  # CS_ENOTINIT
    cs.cs_init(4, 2, 2, 0)
    for call in (lambda: cs.cs_set_hier_nccl(a), lambda: cs.cs_set_multicast(0, 0, 0), cs.cs_multicast_bytes):
        with pytest.raises(cs.CSError) as e:
            call()
        assert e.value.code == -8  # CS_ENOTBOUND
    cs.cs_finalize()
