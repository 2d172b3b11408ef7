"""GPU: GFNCKPT1 checkpoints written by libgfnx load in the reference's load_checkpoint and
vice versa (checkpoint.cpp:11-107), so device-trained policies can be evaluated by the CPU
reference (run_eval, train.cpp:268-292) and reference checkpoints resume on the device."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kw", [
    ("hypergrid_tb_b16", {}), ("dag_mdb_b8192", dict(batch=64)),
    # narrower MLPs run zero-padded on the device; files carry the user's widths
    ("hypergrid_tb_b16", dict(hidden=[64, 48])), ("ising_tb_b32768", dict(batch=32, hidden=[128, 96])),
])
def test_checkpoint_round_trip_with_reference(tmp_path, name, kw):
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    e, t = abi.config(name, **kw)
    d = engine.Trainer(e, t)
    for it in range(3):  # non-trivial parameters and Adam moments
        d.iteration(it)
    p, z = d.params()
    m, v, at, zm, zv, zt = d.adam_state()
    path = tmp_path / "dev.ckpt"
    d.save_checkpoint(path, step=3)
    ref = O.RefLib(e, t)
    assert ref.load_checkpoint(path) == 3
    rp, rz = ref.params()
    assert np.array_equal(rp, p) and rz == z
    # reference -> device: the reference's own writer, read back by libgfnx
    path2 = tmp_path / "ref.ckpt"
    ref.save_checkpoint(path2, 7)
    d2 = engine.Trainer(e, t)
    assert d2.load_checkpoint(path2) == 7
    p2, z2 = d2.params()
    m2, v2, at2, zm2, zv2, zt2 = d2.adam_state()
    assert np.array_equal(p2, p) and z2 == z  # fp32 masters round-trip exactly through fp64
    assert np.array_equal(m2, m) and np.array_equal(v2, v) and (at2, zt2) == (at, zt)
    assert zm2 == zm and zv2 == zv
    # and the bytes agree: device save of the same state == reference save
    path3 = tmp_path / "dev2.ckpt"
    d2.save_checkpoint(path3, 7)
    assert path3.read_bytes() == path2.read_bytes()
    d.close()
    d2.close()
