"""Device CloudSource sampler (csrc/sample.cu) vs numpy's Generator stream.

CPU: the pure-Python Philox/Lemire model (oracle/philox.py) reproduces
numpy's integers() and the bit-generator state.  GPU: the device sampler's
indices, gathered signals and advanced state are bit-identical to numpy's
over consecutive batches, including the pending-half and buffered-word
states, tiny and huge N (heavy rejection), and N == 1.
"""

import numpy as np
import pytest

from oracle.philox import PhiloxModel


def _state_tuple(st):
    # numpy leaves a stale uinteger behind once the pending half is used
    has = int(st["has_uint32"])
    return (tuple(int(x) for x in st["state"]["counter"]), tuple(int(x) for x in st["buffer"]),
            int(st["buffer_pos"]), has, int(st["uinteger"]) if has else 0)


@pytest.mark.parametrize("seed", [7, 1, 2026])
def test_python_model_matches_numpy(seed):
    rng = np.random.Generator(np.random.Philox(seed))
    rng.integers(0, 5, size=3)  # leave a pending half and a partly used block
    model = PhiloxModel(rng.bit_generator.state)
    for n_excl, m in ((1_000_000, 5000), (7, 3001), (2**31 + 12345, 2000), (1, 9), (100_000, 7)):
        assert list(rng.integers(0, n_excl, size=m)) == model.integers(n_excl, m)
    st = rng.bit_generator.state
    assert (tuple(model.ctr), tuple(model.buf), model.pos, model.has) == _state_tuple(st)[:4]


def _device_indices(sampler, m):
    import torch

    d = torch.empty(max(m, 1), dtype=torch.int64, device="cuda")
    sampler.draw_indices(m, d.data_ptr())
    torch.cuda.synchronize()
    return d[:m].cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("n_excl", [1, 2, 3, 1000, 1_000_000, 2**31 + 1, 2**32 - 1])
def test_device_indices_match_numpy(n_excl):
    from paper_1503_08294_b200.device_sampling import DeviceCloudSampler

    rng = np.random.Generator(np.random.Philox(11))
    rng.integers(0, 3, size=1)
    s = DeviceCloudSampler(None, rng, npts=n_excl)
    for m in (1, 5, 8191, 8192, 8193, 100_000, 3):
        want = rng.integers(0, n_excl, size=m)
        assert np.array_equal(_device_indices(s, m), want), (n_excl, m)
        w = s.state_words()
        st = rng.bit_generator.state
        assert (tuple(int(x) for x in w[0:4]), tuple(int(x) for x in w[6:10]), int(w[10]),
                int(w[11]), int(w[12]) if int(w[11]) else 0) == _state_tuple(st)
    s.close()


@pytest.mark.gpu
def test_device_signals_match_cloudsource():
    import torch

    from paper_1503_08294_b200 import CloudSource
    from paper_1503_08294_b200.device_sampling import DeviceCloudSampler

    pts = np.random.Generator(np.random.Philox(3)).random((123_457, 3))
    src = CloudSource(pts)
    rng_host = np.random.Generator(np.random.Philox(9))
    rng_dev = np.random.Generator(np.random.Philox(9))
    src.sample(rng_host, 2)
    src.sample(rng_dev, 2)
    s = DeviceCloudSampler(pts, rng_dev)
    out = torch.empty((70_000, 3), dtype=torch.float64, device="cuda")
    for m in (64, 1024, 4097, 65_536):
        want = src.sample(rng_host, m)
        s.draw(m, out.data_ptr())
        torch.cuda.synchronize()
        got = out[:m].cpu().numpy()
        assert np.array_equal(got.view(np.int64), want.view(np.int64)), m
    s.store_state(rng_dev)  # the host generator continues where the device stopped
    assert np.array_equal(src.sample(rng_dev, 100), src.sample(rng_host, 100))
    s.close()
