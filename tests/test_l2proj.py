"""The L²-projection correction: the CPU oracle
(oracle/l2proj.py) pinned by the properties of the projection, and the
sm_100a kernels (mass-matrix multiply, restriction, batched tridiagonal solve;
paper_2401_05994_b200/csrc/transform.cu) against the oracle.

The reference has no correction, so there is no reference
output to compare with; the oracle is pinned instead by
  * its interpolation part reproducing the reference transform bit for bit,
  * the Galerkin orthogonality of the corrected coarse level (the defining
    property of the L² projection): R_l M_l (u_l - I z) = 0 for every coarse
    basis function,
  * exact reproduction of the coarse space (multilinear fields: zero
    coefficients), and an inverse exact up to rounding.
Gate for the GPU (north_star): coefficients within 1e-12 relative (fp64);
the kernels follow the oracle's operation order and are checked bit for bit.
"""
import numpy as np
import pytest

from oracle import binding, l2proj

SHAPES = [(17,), (33, 17), (12, 7, 10), (6, 5, 4, 3), (65, 65), (2, 9), (2, 2), (40, 21, 9)]


def field(o, shape):
    return o.multisine_noisy(shape, 42, 0.05)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_oracle_interpolation_part_is_the_reference(oracle, shape):
    u = field(oracle, shape)
    L, tab = l2proj._level_tables(u.shape, None)
    v = u.copy()
    for lvl in range(L, 0, -1):
        l2proj._interp_level(v, tab, u.ndim, lvl, -1.0)
    assert np.array_equal(v.view(np.uint64), oracle.forward(u).view(np.uint64))


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_oracle_round_trip(oracle, shape):
    u = field(oracle, shape)
    back = l2proj.inverse_l2(l2proj.forward_l2(u))
    assert np.max(np.abs(back - u)) <= 1e-14 * max(1.0, float(np.max(np.abs(u))))


def test_oracle_reproduces_the_coarse_space(oracle):
    """Multilinear fields lie in every coarse space: all coefficients vanish, the coarsest values are u."""
    shape = (17, 9, 5)
    g = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    u = 0.5 + 0.25 * g[0] - 0.125 * g[1] + 0.0625 * g[2]
    c = l2proj.forward_l2(u)
    L, tab = l2proj._level_tables(shape, None)
    coarse = np.ix_(*[tab[a, 0]["idx"] for a in range(3)])
    mask = np.ones(shape, bool)
    mask[coarse] = False
    assert np.max(np.abs(c[mask])) <= 1e-13
    assert np.allclose(c[coarse], u[coarse], rtol=0, atol=1e-13)


@pytest.mark.parametrize("shape,coords", [((33,), None), ((17, 9), None), ((9, 7, 5), None),
                                          ((12, 10), "random")], ids=["1d", "2d", "3d", "2d-coords"])
def test_oracle_galerkin_orthogonality(oracle, shape, coords):
    """One level: with the corrected coarse values w = u|coarse + z, the error u - I(w) on the level-L grid is
    M-orthogonal to every coarse hat function: R M (u - I w) = 0 (the L² projection's defining property)."""
    rng = np.random.default_rng(5)
    cs = None if coords is None else [np.cumsum(rng.uniform(0.3, 1.0, n)) for n in shape]
    u = rng.standard_normal(shape)
    d = len(shape)
    L, tab = l2proj._level_tables(shape, cs)
    v = u.copy()
    l2proj._interp_level(v, tab, d, L, -1.0)          # level-L coefficients
    z = l2proj._correction(v, tab, d, L)
    cb = np.ix_(*[tab[a, L - 1]["idx"] for a in range(d)])
    w = np.zeros(shape)
    w[cb] = u[cb] + z                                  # corrected coarse values
    l2proj._interp_level(w, tab, d, L, +1.0)           # I w on the level-L grid
    e = u - w
    # R M e along every axis (the level-L mass matrix and restriction of the oracle, without the solve)
    C = e
    for a in range(d):
        tl = tab[a, L]
        if not tl["fresh"].any():
            continue
        vv = np.moveaxis(C, a, -1)
        f = tl["di"] * vv
        f[..., 1:] = tl["lo"][1:] * vv[..., :-1] + f[..., 1:]
        f[..., :-1] = f[..., :-1] + tl["up"][:-1] * vv[..., 1:]
        kq = np.nonzero(~tl["fresh"])[0]
        r = f[..., kq].copy()
        for q, k in enumerate(kq):
            if k > 0 and tl["fresh"][k - 1]:
                r[..., q] += tl["wr"][k - 1] * f[..., k - 1]
            if k + 1 < len(tl["fresh"]) and tl["fresh"][k + 1]:
                r[..., q] += tl["wl"][k + 1] * f[..., k + 1]
        C = np.moveaxis(r, -1, a)
    assert np.max(np.abs(C)) <= 1e-12 * float(np.max(np.abs(u)))


def test_projection_beats_interpolation_in_l2(oracle):
    """The corrected coarse approximation has the smaller L² (mass-norm) error than the interpolant."""
    rng = np.random.default_rng(9)
    u = np.cumsum(rng.standard_normal(65))
    L, tab = l2proj._level_tables(u.shape, None)
    t = tab[0, L]
    v = u.copy()
    l2proj._interp_level(v, tab, 1, L, -1.0)
    z = l2proj._correction(v, tab, 1, L)
    kq = np.nonzero(~t["fresh"])[0]

    def mass_norm(e):
        f = t["di"] * e
        f[1:] = t["lo"][1:] * e[:-1] + f[1:]
        f[:-1] = f[:-1] + t["up"][:-1] * e[1:]
        return float(e @ f)

    def err(coarse_vals):
        w = np.zeros_like(u)
        w[t["idx"][kq]] = coarse_vals
        l2proj._interp_level(w, tab, 1, L, +1.0)
        return mass_norm(u - w)

    assert err(u[kq] + z) < err(u[kq])


@pytest.mark.gpu
@pytest.mark.parametrize("shape", SHAPES + [(129, 65, 33)], ids=lambda s: "x".join(map(str, s)))
def test_gpu_l2_transform_matches_oracle(mg, oracle, shape):
    u = field(oracle, shape)
    c = mg.forward_transform(u, l2=True)
    want = l2proj.forward_l2(u)
    rel = float(np.max(np.abs(c - want))) / max(1e-300, float(np.max(np.abs(u))))
    assert rel <= 1e-12  # north_star gate
    assert np.array_equal(c.view(np.uint64), want.view(np.uint64))  # same operation order: bit for bit
    back = mg.inverse_transform(c, l2=True)
    assert np.array_equal(back.view(np.uint64), l2proj.inverse_l2(want).view(np.uint64))
    assert np.max(np.abs(back - u)) <= 1e-14 * max(1.0, float(np.max(np.abs(u))))


@pytest.mark.gpu
def test_gpu_l2_transform_coords_and_device(mg, oracle):
    import torch

    rng = np.random.default_rng(3)
    shape = (17, 12, 9)
    cs = [np.cumsum(rng.uniform(0.05, 1.0, n)) - 1.0 for n in shape]
    u = field(oracle, shape)
    c = mg.forward_transform(torch.from_numpy(u).cuda(), mg.make_grid(shape, cs), l2=True)
    assert c.is_cuda
    want = l2proj.forward_l2(u, cs)
    assert np.array_equal(c.cpu().numpy().view(np.uint64), want.view(np.uint64))
    back = mg.inverse_transform(c, mg.make_grid(shape, cs), l2=True)
    assert np.max(np.abs(back.cpu().numpy() - u)) <= 1e-14


# ---------------------------------------------------------------------------
# containers of the corrected decomposition (header flag 0x04)

L2_CASES = [  # (shape, dtype, tol, norm, s, mode, codec, coords seed)
    ((33, 17, 9), np.float32, 1e-4, 0, 0.0, 1, 2, None),
    ((65, 65, 65), np.float64, 1e-3, 0, 0.0, 1, 2, None),
    ((129, 130), np.float64, 1e-3, 1, 1.0, 1, 2, None),
    ((129, 130), np.float64, 1e-3, 1, 0.0, 1, 2, None),
    ((40, 33, 17), np.float32, 1e-3, 1, 0.0, 1, 2, None),
    ((6, 5, 4, 3), np.float64, 1e-2, 0, 0.0, 0, 2, None),
    ((17, 12, 9), np.float64, 1e-3, 0, 0.0, 0, 2, 3),
    ((33, 20), np.float64, 1e-3, 0, 0.0, 1, 1, None),
    ((33, 20), np.float32, 1e-3, 0, 0.0, 1, 0, None),
    ((2, 9), np.float64, 1e-3, 0, 0.0, 0, 2, None),
]


def test_l2_container_rejected_by_reference_parser(oracle):
    u = field(oracle, (33, 17)).astype(np.float64)
    blob = l2proj.compress_l2(u, 1e-3, 0, 0.0, 1, 2)
    with pytest.raises(binding.OracleError) as e:
        oracle.decompress(blob)
    assert e.value.name == "CorruptStream"  # unknown header flags (container.cpp:143)


@pytest.mark.gpu
@pytest.mark.parametrize("case", L2_CASES, ids=lambda c: "x".join(map(str, c[0])) + f"-{c[1].__name__}-n{c[3]}s{c[4]}c{c[6]}")
def test_gpu_l2_container_matches_oracle(mg, oracle, case):
    shape, dt, tol, norm, s, mode, codec, seed = case
    coords = None
    if seed is not None:
        rng = np.random.default_rng(seed)
        coords = [np.cumsum(rng.uniform(0.05, 1.0, n)) - 1.0 for n in shape]
    u = field(oracle, shape).astype(dt)
    want = l2proj.compress_l2(u, tol, norm, s, mode, codec, coords)
    spec = mg.ErrorSpec(tol, mg.Norm(norm), s, mg.Mode(mode))
    got = mg.compress(u, mg.make_grid(shape, coords), spec, mg.Codec(codec), l2=True)
    assert got == want
    info = mg.inspect(got)
    assert info.l2_projection and "l2_projection: 1" in mg.describe(got)
    back = mg.decompress(got)
    ref = l2proj.decompress_l2(want, coords)
    assert np.array_equal(back.view(np.uint8), ref.view(np.uint8))
    err = back.astype(np.float64) - u.astype(np.float64)
    tau = oracle.absolute_tolerance(u, tol, norm, s, mode)
    if norm == 0:
        assert np.max(np.abs(err)) <= tau
    elif s == 0.0:
        assert np.sqrt(np.mean(err * err)) <= tau


@pytest.mark.gpu
def test_gpu_l2_constant_and_device_buffers(mg, oracle):
    import torch

    u = np.full((9, 33), 2.5)
    assert mg.compress(u, l2=True) == oracle.compress(u, 1e-3, 0, 0.0, 0, 2)  # constant: the reference container
    v = field(oracle, (40, 21, 9))
    du = torch.from_numpy(v).cuda()
    spec = mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel)
    n = mg.compress_to(du, None, mg.make_grid(v.shape), spec, l2=True)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    mg.compress_to(du, dst, mg.make_grid(v.shape), spec, l2=True)
    blob = bytes(dst.cpu().numpy())
    assert blob == l2proj.compress_l2(v, 1e-4, 0, 0.0, 1, 2)
    out = torch.empty_like(du)
    mg.decompress_into(dst, out)
    assert np.array_equal(out.cpu().numpy(), l2proj.decompress_l2(blob))
