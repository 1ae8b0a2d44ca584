"""Device-side instance synthesis (hcran_b200_synth_gamma, the loader of
scenarios.py:84-153 on the GPU; config[3]'s inputs).  The numbers differ from
the reference's numpy streams, the distributions must not: two-sample KS tests
of the device draws against the host generator (the reference's own
build_config / gen_channel restated, test_loader.py pins it bit-identical),
plus determinism and shard independence."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from scipy.stats import ks_2samp  # noqa: E402

from paper_1803_07772_b200 import synth_gamma  # noqa: E402
from paper_1803_07772_b200.scenarios import workload_batch, workload_instance  # noqa: E402


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_synth_matches_host_distribution(name):
    host = workload_batch(name, range(400, 600))
    cfg = host.cfg
    dev = synth_gamma(cfg, 400, 200).cpu().numpy()
    assert dev.shape == host.gamma.shape and np.all(dev > 0)
    # independent samples only (the cells of one user share its position):
    # the path loss of each (draw, user) per head, through the mean log gain over
    # subcarriers, and the fading alone through the ratio of two subcarriers of
    # one (RRH, user) (the distance cancels)
    for m in range(cfg.n_rrh):
        a = np.log(dev[:, m]).mean(axis=-1).ravel()
        b = np.log(host.gamma[:, m]).mean(axis=-1).ravel()
        assert ks_2samp(a, b).pvalue > 1e-3, m
    ra = np.log(dev[..., 0] / dev[..., 1]).ravel()
    rb = np.log(host.gamma[..., 0] / host.gamma[..., 1]).ravel()
    assert ks_2samp(ra, rb).pvalue > 1e-3


def test_synth_deterministic_and_shard_free():
    cfg, _, _ = workload_instance("c3", 0)
    a = synth_gamma(cfg, 0, 8).cpu().numpy()
    b = synth_gamma(cfg, 4, 4).cpu().numpy()
    c = synth_gamma(cfg, 0, 8).cpu().numpy()
    assert np.array_equal(a, c)
    assert np.array_equal(a[4:], b)
    assert a.shape == (8, 16, 128, 256)
