"""GPU parity of the decomposition and the quantiser as entry points of their own
(forward_transform / inverse_transform, transform.hpp:24-30; quantize /
dequantize, quantize.hpp:32-42) against the reference.

north_star gate: coefficients within 1e-12 relative (fp64) — the GPU path is
held to the stronger bar of bit-identity with the reference library, and the
relative difference (normalised by max|u|) is reported as 0.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [
    ((65, 65, 65), "multisine", None),
    ((33, 17, 9), "noisy", None),
    ((129, 130), "noisy", None),
    ((257, 256), "noisy", None),
    ((12, 7, 10), "noisy", None),
    ((6, 5, 4, 3), "noisy", None),
    ((17,), "noisy", None),
    ((6,), "noisy", None),
    ((2, 2), "noisy", None),          # L = 0
    ((2, 9), "noisy", None),
    ((100, 3, 40), "random", None),
    ((17, 12, 9), "noisy", 3),         # explicit non-uniform coordinates
    ((256, 33), "noisy", None),
]


def make_field(o, kind, shape):
    if kind == "multisine":
        return o.multisine(shape)
    if kind == "noisy":
        return o.multisine_noisy(shape, 42, 0.05)
    return o.random_field(shape, 7, -3.0, 3.0)


def make_coords(shape, seed):
    rng = np.random.default_rng(seed)
    return [np.cumsum(rng.uniform(0.05, 1.0, n)) - 1.0 for n in shape]


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint64),
                                                 np.ascontiguousarray(b).view(np.uint64))


@pytest.mark.parametrize("case", SHAPES, ids=lambda c: "x".join(map(str, c[0])) + ("-coords" if c[2] else ""))
def test_transform_and_quantizer_bit_exact(mg, oracle, case):
    shape, kind, seed = case
    u = make_field(oracle, kind, shape)
    coords = make_coords(shape, seed) if seed is not None else None
    grid = mg.make_grid(shape, coords)
    c = mg.forward_transform(u, grid)
    c_ref = oracle.forward(u, coords)
    assert bits_equal(c, c_ref)
    back = mg.inverse_transform(c, grid)
    assert bits_equal(back, oracle.inverse(c_ref, coords))
    L = mg.nlevels(grid)
    h = oracle.hierarchy(shape, coords)
    assert L == h["nlevels"]
    tau = 1e-4 * float(u.max() - u.min())
    for norm, s in [(0, 0.0), (1, 0.0), (1, 1.0)]:
        w = mg.initial_bin_widths(tau, mg.ErrorSpec(tau, mg.Norm(norm), s), len(shape), L)
        assert np.array_equal(w, oracle.bin_widths(tau, norm, s, len(shape), L))
        q, r, outl = mg.quantize(c, w, grid)
        q_ref, r_ref, outl_ref = oracle.quantize(c_ref, w, coords)
        assert np.array_equal(q, q_ref) and bits_equal(r, r_ref) and outl == outl_ref
        assert bits_equal(mg.dequantize(q, w, grid), oracle.dequantize(q_ref, w, coords))


def test_device_tensors(mg, oracle):
    import torch

    u = oracle.multisine_noisy((33, 40, 21), 42, 0.05)
    du = torch.from_numpy(u).cuda()
    c = mg.forward_transform(du)
    assert c.is_cuda and bits_equal(c.cpu().numpy(), oracle.forward(u))
    w = mg.initial_bin_widths(1e-3, mg.ErrorSpec(1e-3), 3, mg.nlevels(mg.make_grid(u.shape)))
    q, r, _ = mg.quantize(c, w)
    assert q.is_cuda and r.is_cuda
    q_ref, r_ref, _ = oracle.quantize(oracle.forward(u), w)
    assert np.array_equal(q.cpu().numpy(), q_ref) and bits_equal(r.cpu().numpy(), r_ref)
    back = mg.inverse_transform(mg.dequantize(q, w))
    assert back.is_cuda
    assert bits_equal(back.cpu().numpy(), oracle.inverse(oracle.dequantize(q_ref, w)))


def test_quantizer_errors_and_outliers(mg, oracle):
    u = oracle.random_field((65, 65), 7, -3.0, 3.0)
    c = mg.forward_transform(u)
    L = mg.nlevels(mg.make_grid(u.shape))
    tiny = np.full(L + 1, 1e-14)  # |q| > 2^31: outliers counted like the reference
    q, r, outl = mg.quantize(c, tiny)
    q_ref, r_ref, outl_ref = oracle.quantize(oracle.forward(u), tiny)
    assert outl == outl_ref and outl > 0
    assert np.array_equal(q, q_ref) and bits_equal(r, r_ref)
    with pytest.raises(mg.MgrcError) as e:
        mg.quantize(c, np.full(L + 1, 1e-300))
    assert e.value.name == "Overflow"
    with pytest.raises(mg.MgrcError) as e:
        mg.quantize(c, np.full(L, 1e-3))
    assert e.value.name == "ShapeMismatch"
    with pytest.raises(mg.MgrcError) as e:
        mg.quantize(c, np.zeros(L + 1))
    assert e.value.name == "InvalidState"
    bad = u.copy()
    bad[5, 5] = np.inf
    with pytest.raises(mg.MgrcError) as e:
        mg.forward_transform(bad)
    assert e.value.name == "NonFiniteInput"


@pytest.mark.slow
def test_cfg4_decompose_recompose_round_trip(mg, oracle):
    """BASELINE configs[3]: 1025^3 fp64 decompose + recompose.  Coefficients and the round trip are
    bit-identical to the reference library's (gate: 1e-12 relative); max|u - u_hat| / range ~ 1e-16."""
    import torch

    from oracle import binding

    ref = binding.get("reference") if binding.available("reference") else oracle
    ref.set_threads(os.cpu_count() or 1)
    shape = (1025, 1025, 1025)
    u = oracle.multisine(shape)
    du = torch.from_numpy(u).cuda()
    dc = mg.forward_transform(du)
    c_ref = ref.forward(u)
    c = dc.cpu().numpy()
    rel = float(np.max(np.abs(c - c_ref))) / float(np.max(np.abs(u)))
    assert rel <= 1e-12
    assert bits_equal(c, c_ref)
    del c
    dback = mg.inverse_transform(dc)
    del dc
    back_ref = ref.inverse(c_ref)
    del c_ref
    back = dback.cpu().numpy()
    assert bits_equal(back, back_ref)
    err = float((dback - du).abs().max()) / float(du.max() - du.min())
    assert err < 1e-14
