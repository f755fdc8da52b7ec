"""Post-solve field kernels against the reference.

pmg::face_gradient (proj/include/pmg/fields.hpp:149-232) runs on the
unmodified reference build (oracle/_ref/libpmgref.so) after a few cycles;
its PHI (every level: coarse-fine ghosts read the parent level) is uploaded
to the GPU and the device kernels must reproduce every face value and the
cell-centred magnitude bit for bit -- regular faces, faces cut by the level
set, faces inside objects, physical and (AMR) coarse-fine ghosts.
"""
import os

import numpy as np
import pytest

from oracle.oc import REF_SO
from paper_2205_09411_b200 import configs as cfgs
from paper_2205_09411_b200 import face_gradient
from paper_2205_09411_b200.mesh import VAR_PHI
from paper_2205_09411_b200.solver import LAYOUT_INTERIOR

from helpers import interior, setup_pair

pytestmark = pytest.mark.gpu

VAR_AUX = 4  # the reference's post-processing scratch (mesh.hpp:19)


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference build missing (make -C oracle ref)")
@pytest.mark.parametrize("name", ["cfg1@4", "cfg2@3", "cfg3@5", "cfg4@3"])
def test_face_gradient_bit_exact(name):
    case = cfgs.get_case(name)
    o, dev, sol, mesh, st = setup_pair(case)
    o.fmg_cycle()
    for _ in range(2):
        o.v_cycle()
    phi = interior(o, VAR_PHI, case.dim, case.N)
    dev.set_field(VAR_PHI, phi, layout=LAYOUT_INTERIOR)
    ref_ids, ref_faces = o.face_gradient(VAR_PHI, VAR_AUX)
    ids, faces, mag = face_gradient(dev)
    assert np.array_equal(ids, ref_ids)
    assert faces.shape == ref_faces.shape
    bad = np.flatnonzero(faces.reshape(-1) != ref_faces.reshape(-1))
    assert bad.size == 0, (bad.size, bad[:8], faces.reshape(-1)[bad[:4]], ref_faces.reshape(-1)[bad[:4]])
    # some faces of each kind were exercised
    assert np.count_nonzero(ref_faces) > 0
    ref_mag = interior(o, VAR_AUX, case.dim, case.N)[ref_ids]
    assert np.array_equal(mag, ref_mag.reshape(mag.shape))
