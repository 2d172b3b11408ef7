"""CPU: the C-ABI library loads, exports every symbol include/gfnx.h declares, and its
struct layouts / defaults agree with the Python mirror (no compute calls: no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2511_16592_b200 import abi, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gfnx.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gfnx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = engine.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 30
    nm = subprocess.run(["nm", "-D", "--defined-only", engine.LIB_PATH], capture_output=True, text=True)
    exported = set(re.findall(r" T (gfnx_\w+)", nm.stdout))
    assert set(declared_symbols()) <= exported


def test_struct_layouts_match_header(tmp_path):
    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "gfnx.h"\nint main(){'
                 'printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(gfnx_env_desc), sizeof(gfnx_train_desc),'
                 'sizeof(gfnx_schedule), sizeof(gfnx_env_shape), sizeof(gfnx_host_batch),'
                 'offsetof(gfnx_train_desc, explore), offsetof(gfnx_env_desc, dag_data_seed));'
                 'printf("%zu %zu\\n", sizeof(gfnx_eb_desc), offsetof(gfnx_eb_desc, coupling_lr_end));return 0;}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I" + os.path.dirname(HEADER), str(c), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(abi.EnvDesc), C.sizeof(abi.TrainDesc), C.sizeof(abi.Schedule),
            C.sizeof(abi.EnvShape), C.sizeof(abi.HostBatch), abi.TrainDesc.explore.offset,
            abi.EnvDesc.dag_data_seed.offset, C.sizeof(abi.EbDesc), abi.EbDesc.coupling_lr_end.offset]
    assert got == want


@pytest.mark.parametrize("kind", [abi.HYPERGRID, abi.BITSEQ, abi.ISING, abi.DAG])
def test_defaults_match_reference_drivers(kind):
    L = engine.lib()
    e, t = abi.EnvDesc(), abi.TrainDesc()
    assert L.gfnx_default_env_desc(kind, C.byref(e)) == 0
    assert L.gfnx_default_train_desc(kind, C.byref(t)) == 0
    pe, pt = abi.env_desc(kind), abi.train_desc(kind)
    assert bytes(e) == bytes(pe)
    assert bytes(t) == bytes(pt)


def test_env_shapes_of_baseline_configs():
    want = {"hypergrid_tb_b16": (5, 5, 80, 77), "bitseq_tb_b16384": (3840, 15, 3856, 15),
            "ising_tb_b32768": (200, 100, 300, 100), "dag_mdb_b8192": (21, 21, 25, 11)}
    for name, (A, Ab, O, T) in want.items():
        e, _ = abi.config(name)
        s = engine.env_shape(e)
        assert (s.num_actions, s.num_backward_actions, s.obs_dim, s.max_traj_len) == (A, Ab, O, T)


def test_config_errors_without_gpu():
    with pytest.raises(engine.config_error, match="r0 must be positive"):
        engine.env_shape(abi.env_desc(abi.HYPERGRID, hg_r0=0.0))
    with pytest.raises(engine.config_error, match="k must divide"):
        engine.env_shape(abi.env_desc(abi.BITSEQ, bs_n_bits=12, bs_k=5))


def test_eb_defaults_and_host_gibbs_sampler_match_reference():
    """run_eb_gfn's defaults (train.cpp:899-913) and the host Gibbs data sampler used by
    gfnx_eb_init (gibbs_data_sampler ising.cpp:185-220, key fold_in(make_key(seed), 0x919B))
    against the compiled reference: identical spins, with and without parallel tempering."""
    d = engine.eb_desc()
    assert (d.data_samples, d.k, d.gibbs_burn_in, d.gibbs_thinning, d.gibbs_chains, d.data_batch) == \
        (2000, 0, 2000, 10, 1, 0)
    assert (d.gibbs_hottest_beta, d.alpha, d.coupling_lr, d.coupling_lr_end) == (0.2, 0.5, 0.05, 0.05)
    from oracle import oracle as O
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    for side, sigma, seed, chains in ((3, 0.2, 5, 1), (4, 0.35, 1, 3)):
        d = engine.eb_desc(gibbs_burn_in=200, gibbs_thinning=3, gibbs_chains=chains)
        dev = engine.ising_gibbs_data(side, sigma, seed, 150, d)
        ref = O.ref_gibbs_data(side, sigma, seed, 150, burn_in=200, thinning=3, chains=chains)
        assert np.array_equal(dev, ref), (side, chains)
