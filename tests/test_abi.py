"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/topo.h declares, and its pure host entry points work
(element stiffness vs the oracle's, error paths that fail before any device
work)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "topo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(topo_[a-z_0-9A-Z]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2504_05604_b200 import topo
    lib = ctypes.CDLL(topo.LIB_PATH)
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(topo.EXPORTS)


def test_library_is_sm100a():
    """The fatbin carries sm_100a code (cuobjdump lists it)."""
    import subprocess
    from paper_2504_05604_b200 import topo
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", topo.LIB_PATH],
                       capture_output=True, text=True)
    assert "sm_100a" in r.stdout


@pytest.mark.parametrize("nu", [0.0, 0.3, 0.45])
def test_element_stiffness_matches_oracle(nu):
    """Library KE (C++ quadrature) vs oracle KE (numpy quadrature): independent
    implementations of S:117."""
    from paper_2504_05604_b200 import element_stiffness
    from oracle import element_stiffness as oracle_ke
    assert np.max(np.abs(element_stiffness(nu) - oracle_ke(nu))) < 1e-15


def test_init_rejects_bad_inputs_before_device_work():
    from paper_2504_05604_b200.topo import Problem, TopoError, TOPO_EINVAL, TOPO_EUNCONSTRAINED
    from workloads import make_problem
    p, f, fx, _ = make_problem(0)
    with pytest.raises(TopoError) as e:
        Problem(dict(p, nelx=0), f, fx)
    assert e.value.code == TOPO_EINVAL
    with pytest.raises(TopoError) as e:
        Problem(dict(p, volfrac=1.5), f, fx)
    assert e.value.code == TOPO_EINVAL
    with pytest.raises(TopoError) as e:
        Problem(p, f, np.zeros_like(fx))
    assert e.value.code == TOPO_EUNCONSTRAINED
    bad = f.copy()
    bad[0] = 1.0                       # node 0 is on the fixed x = 0 face
    with pytest.raises(TopoError) as e:
        Problem(p, bad, fx)
    assert e.value.code == TOPO_EINVAL


def test_strerror_and_version():
    from paper_2504_05604_b200 import topo
    assert topo._lib.topo_strerror(0) == b"ok"
    assert b"sm_100a" in topo._lib.topo_version()
