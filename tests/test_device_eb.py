"""GPU: EB-GFN on the device (gfnx_eb_*; run_eb_gfn train.cpp:875-1018).

* fp64 check mode reproduces the reference's run_eb_gfn: the same Gibbs data, the same mixed
  sampler batches (on-policy rows + data-backed backward walks), back-and-forth proposals, MH
  decisions and CD updates, so the learned coupling after 30 iterations and the metrics.csv
  rows (loss, logZ, neg_log_rmse, acceptance rate) agree with the compiled reference to
  ~1e-12 (the device exp/log differ from glibc by <= 1 ulp).
* The reference's acceptance criterion 5, EB part (acceptance.cpp:365-385: side 3, batch 16,
  MLP 2x128, data batch 64, coupling lr 0.02, seed 5, 1200 iterations): the device run must
  gain >= 1.0 in neg-log-RMSE of the coupling.
* The bf16 path (lockstep Ising rollout with teacher-forced data rows on the tensor cores)
  runs the same loop and learns the coupling.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu


def _ctx(side, sigma, batch, hidden, iterations, seed, check=True, learned=0):
    e = abi.env_desc(abi.ISING, is_side=side, is_sigma=sigma)
    t = abi.train_desc(abi.ISING, batch=batch, hidden=hidden, iterations=iterations, seed=seed)
    t.learned_backward = learned
    if check:
        t.precision = abi.PREC_FP64_CHECK
    return engine.Trainer(e, t)


@pytest.mark.parametrize("learned", [0, 1])
def test_eb_check_mode_matches_reference_run(learned):
    """test_config_train.cpp:344-361's configuration (k = 4, data batch 16) on the device; with
    learned = 1 the sampler's learned backward head drives the data walks, the training log P_B
    and the back-and-forth proposals (objective.learned_backward)."""
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    kv = {"env.side": 2, "env.sigma": 0.3, "env.data_samples": 100, "gibbs.burn_in": 100,
          "train.iterations": 30, "train.batch_size": 8, "mlp.hidden": "16", "eval.interval": 10,
          "eb.k": 4, "eb.data_batch": 16, "objective.learned_backward": "true" if learned else "false"}
    out = tempfile.mkdtemp(prefix="ebref_")
    res, J_ref, rows = O.ref_eb_gfn(kv, out)
    tr = _ctx(2, 0.3, 8, (16,), 30, 0, learned=learned)
    tr.eb_init(engine.eb_desc(data_samples=100, gibbs_burn_in=100, k=4, data_batch=16))
    m = tr.eb_run(0, 30)
    jm, jt, init_nlr = tr.eb_coupling()
    tr.close()
    assert abs(init_nlr - res["init_nlr"]) <= 1e-12
    err = np.max(np.abs(jm - J_ref))
    print(f"EB-GFN 30 iterations: max |J_device - J_reference| = {err:.2e}")
    assert err <= 1e-10, err
    for step, loss, logz, nlr, rate in rows:
        i = int(step) - 1
        assert abs(m[i, 0] - loss) <= 1e-8 * max(1.0, abs(loss)), (step, m[i, 0], loss)
        assert abs(m[i, 1] - logz) <= 1e-8 * max(1.0, abs(logz)), (step, m[i, 1], logz)
        assert abs(m[i, 2] - nlr) <= 1e-8, (step, m[i, 2], nlr)
        lo = int(step) - 10
        assert abs(m[lo:int(step), 3].sum() / (10 * 16) - rate) <= 1e-12, (step, rate)
    assert abs(m[-1, 0] - res["final_loss"]) <= 1e-8 * max(1.0, abs(res["final_loss"]))


def test_eb_acceptance_criterion5_coupling_gain():
    """acceptance.cpp:365-385 (reference: gain >= 1.0 in neg-log-RMSE within 1200 iterations)."""
    tr = _ctx(3, 0.2, 16, (128, 128), 1200, 5)
    tr.eb_init(engine.eb_desc(data_samples=2000, data_batch=64, coupling_lr=0.02, coupling_lr_end=0.02))
    m = tr.eb_run(0, 1200)
    _, _, init_nlr = tr.eb_coupling()
    tr.close()
    best = float(np.max(m[:, 2]))
    print(f"EB-GFN criterion 5: neg-log-rmse {init_nlr:.3f} -> {best:.3f} (gain {best - init_nlr:.2f}), "
          f"acceptance {m[-200:, 3].sum() / (200 * 64):.3f}")
    assert np.all(np.isfinite(m[:, :3]))
    assert best - init_nlr >= 1.0, (init_nlr, best)


def test_eb_bf16_lockstep_path_learns_coupling():
    """The sampler batch (on-policy + data-backed rows) on the bf16 lockstep Ising rollout."""
    tr = _ctx(3, 0.2, 128, (256, 256), 400, 5, check=False)
    tr.eb_init(engine.eb_desc(data_samples=2000, data_batch=64, coupling_lr=0.02, coupling_lr_end=0.02))
    m = tr.eb_run(0, 400)
    _, _, init_nlr = tr.eb_coupling()
    tr.close()
    best = float(np.max(m[:, 2]))
    print(f"EB-GFN bf16: neg-log-rmse {init_nlr:.3f} -> {best:.3f}")
    assert np.all(np.isfinite(m[:, :3])) and np.all((m[:, 3] >= 0) & (m[:, 3] <= 64))
    assert best - init_nlr >= 0.5, (init_nlr, best)


def test_eb_rejects_non_ising_and_bad_k():
    e = abi.env_desc(abi.HYPERGRID)
    t = abi.train_desc(abi.HYPERGRID)
    tr = engine.Trainer(e, t)
    with pytest.raises(engine.config_error):
        tr.eb_init()
    tr.close()
    tr = _ctx(2, 0.3, 8, (16,), 10, 0)
    with pytest.raises(engine.config_error):
        tr.eb_init(engine.eb_desc(k=5))  # k must lie in [0, D]
    with pytest.raises(engine.contract_violation):
        tr.eb_run(0, 1)  # no EB state
    tr.close()
