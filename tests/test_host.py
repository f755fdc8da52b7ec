"""CPU: host-side logic of the product package (no GPU needed)."""
import glob
import os
import re

import numpy as np
import pytest

from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200.mesh import FaceBc, build_uniform

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_mesh_mirror_matches_reference_topology(path):
    """mesh.py rebuilds the reference's block table, level lists and
    neighbour tables (mesh.hpp:157-320, 429-469; harness.hpp:295-321)."""
    gold = np.load(path)
    case = cfgs.get_case(os.path.basename(path)[:-4].replace("_L", "@"))
    t = case.build_mesh().topology_arrays()
    for k in ("level", "coords", "parent", "nbr", "cnbr"):
        assert np.array_equal(t[k], gold["topo_" + k]), k


def test_amr_config3_block_counts():
    """Config 3: blocks per level 1/8/64/512/1664/5120/12160,
    8,749,056 leaf cells."""
    case = cfgs.get_case("cfg3")
    m = case.build_mesh()
    assert [len(m.level_blocks(l)) for l in range(1, m.n_levels + 1)] == \
        [1, 8, 64, 512, 1664, 5120, 12160]
    assert case.leaf_cells(m) == 8749056


def test_splitmix64_known_values():
    # public splitmix64 stream: the first outputs for seed 0 are well known
    z = cfgs.splitmix64(0, np.arange(3, dtype=np.uint64))
    assert [int(x) for x in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    u = cfgs.uniform01(123, np.arange(1000, dtype=np.uint64))
    assert np.all((u >= 0) & (u < 1))


def test_config_inputs_are_deterministic_and_in_range():
    c2 = cfgs.get_case("cfg2@3")
    m = c2.build_mesh()
    a, b = c2.rhs_fields(m), c2.rhs_fields(m)
    assert np.array_equal(a, b)
    leaf = np.array([m.is_leaf(x) for x in range(m.n_blocks)])
    assert np.all(np.abs(a[leaf]) <= 1e-2) and np.all(a[~leaf] == 0)
    s = cfgs.spheres32()
    assert len(s.children) == 32
    for ch in s.children:
        assert all(0.15 <= v <= 0.85 for v in ch.center) and 0.01 <= ch.radius <= 0.06
    c5 = cfgs.get_case("cfg5@3")
    g = c5.rhs_fields(c5.build_mesh())
    assert abs(np.std(g[g != 0]) - 1e-3) < 1e-4


def test_vcycle_byte_model():
    """about 171.4 algorithmic bytes per unknown at 256^3, L=5."""
    import bench
    case = cfgs.get_case("cfg2")
    m = case.build_mesh()
    B = bench.vcycle_bytes(m, case.N, case.dim)
    assert abs(B / case.leaf_cells(m) - 171.39) < 0.01


def test_face_bc_values_follow_fill_positions():
    """x_f = cell_center(b, i1) + 0.5 dx sign(dir) e_axis (mesh.hpp:538-552)."""
    m = build_uniform(2, (0, 0), (1, 1), 4, 2)
    m.face_bc[1] = FaceBc(0, lambda x: x[:, 0] + 2 * x[:, 1])
    vals = m.face_bc_values(1)
    # blocks with a physical +x face: ids of level-2 blocks with coords x == 1
    ids = [b for b in range(m.n_blocks) if m.nbr[b][1] < 0 and m.cnbr[b][1] < 0]
    assert vals.size == 4 * len(ids)
    b = ids[0]
    y = m.origin[b][1] + (np.arange(4) + 0.5) * m.dx[b]
    assert np.array_equal(vals[:4], 1.0 + 2 * y)


def test_abi_library_exports_every_declared_symbol():
    """The C-ABI library loads without a GPU and exports what include/ declares."""
    import ctypes
    from paper_2205_09411_b200 import _lib
    lib = _lib.load()
    hdr = open(os.path.join(ROOT, "include", "pmg_b200.h")).read()
    names = sorted(set(re.findall(r"\b(pmg_b200_[a-z_0-9]+)\s*\(", hdr)))
    assert len(names) >= 35
    for n in names:
        assert hasattr(lib, n), n
    assert set(_lib.EXPORTS) <= set(names)
    # without a device the context reports an error instead of crashing
    lo = np.zeros(3)
    hi = np.ones(3)
    h = lib.pmg_b200_create(3, 16, lo, hi, 0)
    assert h
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert b"CUDA" in lib.pmg_b200_last_error(h) or lib.pmg_b200_last_error(h)
    lib.pmg_b200_destroy(h)
    assert ctypes.sizeof(_lib.LsfT) == 4 + 4 + 24 + 8 + 24 + 24 + 8 * 4


def test_abi_argument_errors_without_gpu():
    from paper_2205_09411_b200 import _lib
    lib = _lib.load()
    h = lib.pmg_b200_create(4, 16, np.zeros(3), np.ones(3), 0)
    assert b"dim must be 2 or 3" in lib.pmg_b200_last_error(h)
    lib.pmg_b200_destroy(h)
    h = lib.pmg_b200_create(3, 12, np.zeros(3), np.ones(3), 0)
    assert b"power of two" in lib.pmg_b200_last_error(h)
    lib.pmg_b200_destroy(h)


def _cbrt_restated(x):
    """numpy restatement of the device libm_cbrt (stencil_build.cuh): glibc's
    dbl-64 s_cbrt algorithm, which the reference's std::cbrt runs."""
    xm, xe = np.frexp(np.abs(x))
    u = (0.354895765043919860 + ((1.50819193781584896 + ((-2.11499494167371287 + (
        (2.44693122563534430 + ((-1.83469277483613086 + (0.784932344976639262
                                                         - 0.145263899385486377 * xm) * xm) * xm))
        * xm)) * xm)) * xm))
    t2 = u * u * u
    c2, s2 = 1.2599210498948731648, 1.5874010519681994748
    fac = np.array([1.0 / s2, 1.0 / c2, 1.0, c2, s2])
    idx = 2 + np.fmod(xe, 3)  # C's truncating %
    ym = u * (t2 + 2.0 * xm) / (2.0 * t2 + xm) * fac[idx]
    q = np.trunc(xe / 3).astype(np.int64)  # C's truncating /
    out = np.ldexp(np.where(x > 0, ym, -ym), q)
    return np.where(x == 0, x + x, out)


def test_cbrt_restatement_matches_host_libm():
    """The heart/astroid level sets call std::cbrt (levelset.hpp:114-120); the
    GPU reproduces the host libm's (not correctly rounded) cbrt bit for bit."""
    import ctypes
    import ctypes.util
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.cbrt.restype = ctypes.c_double
    libm.cbrt.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(0, 64, 40000) ** 2, rng.uniform(-1e-3, 1e3, 20000),
                        np.exp(rng.uniform(-700, 700, 20000)), [0.0, 1.0, 8.0, 27.0, 5e-324]])
    ref = np.array([libm.cbrt(float(v)) for v in x])
    assert np.array_equal(_cbrt_restated(x).view(np.uint64), ref.view(np.uint64))
