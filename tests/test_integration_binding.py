"""The reference-side drop-in: include/gfnx_device.hpp compiled against the reference's own
headers (/root/reference/proj/include) and objects, linked with libgfnx.so, driven from a
gfnkit program (tests/integration/binding_driver.cpp, built by oracle/Makefile).

CPU: the binding compiles and links, and bad descriptors surface as the reference's own
exception types (gfn::config_error, errors.hpp:6-16) through the C ABI.
GPU: the reference's mlp_init parameters go to the device, three iterations train there,
and the parameters come back into the reference's MlpParams.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "binding_driver")
REF = "/root/reference/proj/include/gfn/nn.hpp"


def _driver():
    if os.path.exists(REF):
        r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/binding_driver"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    if not os.path.exists(DRIVER):
        pytest.skip("reference headers absent and no prebuilt oracle/_ref/binding_driver")
    return DRIVER


def test_binding_compiles_links_and_maps_errors():
    r = subprocess.run([_driver(), "errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("config_error: hypergrid: r0 must be positive")
    assert lines[1].startswith("config_error:")


@pytest.mark.gpu
def test_binding_trains_reference_params_on_device():
    r = subprocess.run([_driver(), "train"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "roundtrip_maxdiff" in r.stdout


@pytest.mark.gpu
def test_binding_runs_eb_gfn_loop_on_device():
    """run_eb_gfn's loop through DeviceTrainer::eb_*: reference Gibbs data in, the learned
    coupling back in the reference's IsingCoupling; its neg_log_rmse (computed by the
    reference) equals the device's metric."""
    r = subprocess.run([_driver(), "eb"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    vals = dict(zip(r.stdout.split()[1::2], map(float, r.stdout.split()[2::2])))
    assert vals["final_nlr"] > vals["init_nlr"], vals
