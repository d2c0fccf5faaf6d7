"""C-ABI library: loads, exports every symbol include/spfom.h declares, and its
host-only logic (partition, validation, workspace sizing) works without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_22421_b200 import build as b
    b.build()
    import paper_2602_22421_b200 as pkg
    return pkg.load_library()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "spfom.h")).read()
    return sorted(set(re.findall(r"\b(spfom_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_are_exported(lib):
    import paper_2602_22421_b200 as pkg
    decl = declared_symbols()
    assert decl, "no declarations parsed"
    assert set(decl) == set(pkg.EXPORTED)
    for name in decl:
        assert hasattr(lib, name), name


def test_built_for_sm100a():
    so = os.path.join(ROOT, "paper_2602_22421_b200", "libspfom.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _ref_partition(seg_ptr, world):
    nnz = seg_ptr[-1]
    b = [0]
    for r in range(1, world):
        target = -(-nnz * r // world)
        k = int(np.searchsorted(seg_ptr, target, side="left"))
        if 0 < k <= len(seg_ptr) - 1 and (target - seg_ptr[k - 1]) < (seg_ptr[k] - target):
            k -= 1
        b.append(min(max(k, b[-1]), len(seg_ptr) - 1))
    b.append(len(seg_ptr) - 1)
    return np.array(b)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_balanced_contiguous(lib, world):
    from paper_2602_22421_b200 import partition
    rng = np.random.default_rng(world)
    ks = rng.integers(20, 201, size=5000)
    seg_ptr = np.concatenate([[0], np.cumsum(ks)])
    b = partition(seg_ptr, world)
    assert b[0] == 0 and b[-1] == 5000 and np.all(np.diff(b) >= 0)
    assert np.array_equal(b, _ref_partition(seg_ptr, world))
    nnz_r = seg_ptr[b[1:]] - seg_ptr[b[:-1]]
    assert np.all(np.abs(nnz_r - seg_ptr[-1] / world) <= ks.max())


def test_partition_more_ranks_than_segments(lib):
    from paper_2602_22421_b200 import partition
    b = partition(np.array([0, 3, 5]), 4)
    assert b[0] == 0 and b[-1] == 2 and np.all(np.diff(b) >= 0)


def test_workspace_bytes_host_only(lib):
    from paper_2602_22421_b200.spfom import Params, _Instance
    from spfom_inputs import generate
    inst = generate("small", m=100, N=50, k=(1, 40))
    sp = np.ascontiguousarray(inst.seg_ptr)
    ci = _Instance(inst.m, inst.N, inst.nnz, 0, inst.m, sp.ctypes.data, *([None] * 7))
    p, _ = Params()._c()
    nb = C.c_size_t()
    assert lib.spfom_workspace_bytes(C.byref(ci), C.byref(p), C.byref(nb)) == 0
    nq = int(np.sum((np.diff(inst.seg_ptr) + 3) // 4))
    assert nb.value >= nq * (16 + 3 * 32)


def _create_status(lib, inst, params=None):
    from paper_2602_22421_b200.spfom import Params, _Instance
    arrs = [np.ascontiguousarray(a) for a in (inst.seg_ptr, inst.prod_idx.astype(np.int32), inst.attract,
                                              inst.shadow, inst.no_purchase, inst.arrival, inst.price,
                                              inst.capacity)]
    ci = _Instance(inst.m, inst.N, inst.nnz, 0, inst.m, *[a.ctypes.data for a in arrs])
    p, _b = (params or Params())._c()
    h = C.c_void_p()
    st = lib.spfom_create(C.byref(ci), C.byref(p), None, None, None, 0, C.byref(h))
    return st, lib.spfom_last_error(None).decode()


@pytest.mark.parametrize("breaker,needle", [
    (lambda I: I.shadow.__setitem__(3, I.attract[3]), "0 <= w < v"),
    (lambda I: I.attract.__setitem__(5, -1.0), "0 <= w < v"),
    (lambda I: I.no_purchase.__setitem__(2, 0.0), "no_purchase[2]"),
    (lambda I: I.arrival.__setitem__(1, -3.0), "arrival[1]"),
    (lambda I: I.capacity.__setitem__(4, np.nan), "capacity[4]"),
    (lambda I: I.prod_idx.__setitem__(1, I.prod_idx[0]), "strictly increasing"),
])
def test_create_rejects_invalid_instances(lib, breaker, needle):
    """Validation (S:L34-36 + GAM rules) is host logic: EDATA naming the offender."""
    from spfom_inputs import generate
    inst = generate("small", m=20, N=30, k=5)
    breaker(inst)
    st, msg = _create_status(lib, inst)
    assert st == 2 and needle in msg, (st, msg)


def test_create_rejects_bad_params(lib):
    from paper_2602_22421_b200 import Params
    from spfom_inputs import generate
    inst = generate("small", m=20, N=30, k=5)
    for p in (Params(theta=0.0), Params(tau=-1.0), Params(extrapolation=1.5), Params(tau_mode=0, tau=1.0, mu=2.0),
              Params(blocks=np.array([[3, 2]], dtype=np.int32)), Params(blocks=np.array([[0, 99]], dtype=np.int32))):
        st, _ = _create_status(lib, inst, p)
        assert st == 1


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without the shared library the binding raises instead of computing anything."""
    import paper_2602_22421_b200.spfom as s
    monkeypatch.setattr(s, "LIB_PATH", "/nonexistent/libspfom.so")
    monkeypatch.setattr(s, "_lib", None)
    with pytest.raises(ImportError):
        s.load_library()


def test_product_never_imports_oracle():
    """The CUDA path and the oracle share no code (grep of the package sources)."""
    pkg = os.path.join(ROOT, "paper_2602_22421_b200")
    for dirpath, _d, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "spfom_oracle" not in text, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            text = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"(import|from)\s+paper_2602_22421_b200", text), f
            assert '#include "spfom.h"' not in text and "spfom_kernels" not in text, f


def test_ctypes_mirrors_match_the_header_structs(lib):
    """The binding's ctypes structs have the C sizes (a mismatch would let the
    library write past the Python buffers)."""
    import ctypes as C
    from paper_2602_22421_b200 import spfom as B
    out = (C.c_size_t * 5)()
    lib.spfom_abi_sizes(out)
    assert list(out) == [C.sizeof(B._Instance), C.sizeof(B._Params), C.sizeof(B._Info), C.sizeof(B._Residuals),
                         C.sizeof(B._Dist)]


def test_binding_checks_array_lengths_before_native_code():
    """The C ABI trusts the sizes it is given: the binding rejects short arrays
    (SPFOM_EINVAL) before any pointer reaches the library (no GPU needed)."""
    import copy
    from paper_2602_22421_b200 import Solver, SpfomError
    from spfom_inputs import generate
    inst = generate("tiny")
    for field, cut in (("attract", 1), ("shadow", 1), ("no_purchase", 1), ("arrival", 1), ("capacity", 1)):
        bad = copy.copy(inst)
        setattr(bad, field, np.asarray(getattr(inst, field))[:-cut])
        with pytest.raises(SpfomError) as ei:
            Solver(bad)
        assert ei.value.status == 1, (field, ei.value)
