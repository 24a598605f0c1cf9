"""MDR refactor / recompose on the GPU (row f2) against the reference library's
own refactor / request / reconstruct (refactor.hpp:81-117; oracle/_ref, the
reference compiled unmodified): segments byte-identical, the same greedy
plans, progressive reconstructions bit-identical."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # (shape, field, planes, coords seed)
    ((33, 17, 9), "multisine", 32, None),
    ((65, 65), "noisy", 32, None),
    ((17,), "noisy", 8, None),
    ((6, 5, 4, 3), "noisy", 16, None),
    ((17, 12, 9), "noisy", 60, 3),
    ((40, 21, 9), "random", 24, None),
]


def _field(o, kind, shape):
    if kind == "multisine":
        return o.multisine(shape)
    if kind == "noisy":
        return o.multisine_noisy(shape, 42, 0.05)
    return o.random_field(shape, 7, -3.0, 3.0)


def _coords(shape, seed):
    if seed is None:
        return None
    rng = np.random.default_rng(seed)
    return [np.cumsum(rng.uniform(0.05, 1.0, n)) - 1.0 for n in shape]


@pytest.fixture(scope="module")
def refmdr():
    from oracle import binding

    if not binding.available("reference"):
        pytest.skip("oracle/_ref not built")
    return binding


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])) + f"-B{c[2]}")
def test_refactor_request_reconstruct_match_reference(mg, oracle, refmdr, case):
    from paper_2401_05994_b200 import mdr

    shape, kind, B, seed = case
    cs = _coords(shape, seed)
    u = _field(oracle, kind, shape)
    store = mdr.refactor(u, mg.make_grid(shape, cs), planes=B)
    ref = refmdr.mdr_refactor(u, B, coords=cs)
    rj = json.loads(ref.manifest_json)
    m = store.manifest
    assert list(m.shape) == rj["shape"] and m.nlevels == rj["nlevels"] and m.planes == rj["planes"]
    assert m.level_exponents == rj["level_exponents"]
    assert m.level_counts == rj["level_counts"]
    assert (m.value_min, m.value_max, m.value_rms) == (rj["stats"]["min"], rj["stats"]["max"], rj["stats"]["rms"])
    for s in rj["segments"]:
        g = m.segments[s["level"]][s["plane"]]
        assert (g.byte_size, g.raw_bits, g.checksum) == (s["bytes"], s["bits"], s["crc32"]), s
        assert store.segments[s["level"]][s["plane"]] == ref.segment(s["level"], s["plane"]), s
    # plans and progressive reconstructions (two rounds on one state)
    rng = float(u.max() - u.min())
    for norm, sm in [(mg.Norm.inf, 0.0), (mg.Norm.s, 0.0), (mg.Norm.s, 1.0)]:
        st = mdr.make_initial_state(m)
        sess = refmdr.RefSession(ref, u.size)
        fetched = [0] * (m.nlevels + 1)
        for tol in (1e-2 * rng, 1e-5 * rng):
            req = mdr.request(m, tol, norm, sm, st)
            want = refmdr.mdr_request(ref.manifest_json, tol, int(norm), sm, fetched)
            assert req.segments == want[0] and req.total_bytes == want[1]
            assert req.predicted == want[2] and req.satisfiable == want[3]
            got = mdr.reconstruct(m, lambda l, p: store.segments[l][p], req, st, norm, sm)
            wv, wacc = sess.reconstruct(want[0], int(norm), sm)
            assert np.array_equal(got.ravel().view(np.uint64), wv.view(np.uint64))
            assert st.accrued == wacc
            for lv, _ in req.segments:
                fetched[lv] += 1
            assert st.planes_fetched == fetched
            if norm == mg.Norm.inf and req.satisfiable:
                assert float(np.max(np.abs(got - u))) <= tol


def test_store_persistence_and_errors(mg, oracle, refmdr, tmp_path):
    from paper_2401_05994_b200 import mdr

    u = oracle.multisine_noisy((33, 20), 42, 0.05)
    store = mdr.refactor(u, planes=16)
    mdr.write_store(store, tmp_path)
    m = mdr.read_manifest(tmp_path)
    assert m == store.manifest
    # the reference's manifest document reads back into the same manifest
    ref = refmdr.mdr_refactor(u, 16)
    assert mdr.manifest_from_json(ref.manifest_json) == store.manifest
    src = mdr.directory_source(tmp_path, m)
    req = mdr.request(m, 1e-4, mg.Norm.inf)
    st = mdr.make_initial_state(m)
    full = mdr.reconstruct(m, src, req, st)
    assert float(np.max(np.abs(full - u))) <= 1e-4
    # per-level prefix order (PrefixViolation) and checksums (ChecksumMismatch)
    st2 = mdr.make_initial_state(m)
    lv = next(l for l in range(m.nlevels + 1) if m.level_exponents[l] is not None)
    with pytest.raises(mg.MgrcError) as e:
        mdr.reconstruct(m, src, mdr.SegmentRequest([(lv, 1)], 0.0, True, 0), st2)
    assert e.value.name == "PrefixViolation"
    bad = lambda l, p: bytes([store.segments[l][p][0] ^ 1]) + store.segments[l][p][1:]  # noqa: E731
    with pytest.raises(mg.MgrcError) as e:
        mdr.reconstruct(m, bad, mdr.SegmentRequest([(lv, 0)], 0.0, True, 0), mdr.make_initial_state(m))
    assert e.value.name == "ChecksumMismatch"
    with pytest.raises(mg.MgrcError) as e:
        mdr.refactor(u, planes=7)
    assert e.value.name == "PlaneCountOutOfRange"
