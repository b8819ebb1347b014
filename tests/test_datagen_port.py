"""The numpy port of the device generator (oracle/datagen_port.py) pinned to
Philox4x32-10's published known-answer vectors (Random123 kat_vectors), and
its transforms' distributions (CPU)."""
import numpy as np

from oracle import datagen_port as port


def _raw(c, k):
    out = port.philox_raw(*[np.array([x], dtype=np.uint64) for x in c], *k)
    return [int(x[0]) for x in out]


def test_philox4x32_10_known_answers():
    assert _raw((0, 0, 0, 0), (0, 0)) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert _raw((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF)) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert _raw((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0)) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_uniforms_open_interval_and_normals():
    x0, x1, x2, x3 = port.philox(np.arange(200000, dtype=np.uint64), 1, 11)
    u = port.u53(x0, x1)
    assert u.min() > 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.005
    z = port.normal01(np.arange(200000, dtype=np.uint64), 1, 11)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01


def test_slices_are_rows_of_the_full_instance():
    full = port.latent(0, 6, 40, 8, 1, 0.5, 5)
    part = port.latent(2, 3, 40, 8, 1, 0.5, 5)
    assert np.array_equal(full[2:5], part)
    s = port.sparse(0, 3, 60, 5, 1.1, 1e-4, 2)
    assert np.all((s > 2e-4).sum(axis=1) == 5)
