"""Op-level GPU parity: every libdfc operator against the oracle (which is
pinned bit-for-bit to the reference) on the golden inputs plus random grids.
Selection ops must be bit-exact; blurs within 1e-4 (fast) or bit-exact-ish
(exact fp64 mode, 1 float32 ulp)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import depthfill_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1802_00036_b200 import ops as _ops

    return _ops


@pytest.fixture(scope="module")
def golden(golden_dir):
    return np.load(golden_dir / "ops_small.npz")


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def _eq(a, b):
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    return a.shape == b.shape and np.array_equal(_bits(a), _bits(b))


def _keys(golden):
    return [k[3:] for k in golden.files if k.startswith("in_")]


def _dev(v):
    return torch.from_numpy(np.ascontiguousarray(v)).cuda()


def test_box_minmax_golden(ops, golden):
    for key in _keys(golden):
        v = _dev(golden[f"in_{key}"])
        for r in (1, 2, 3, 15):
            assert _eq(ops.box_max(v, r).cpu().numpy(), golden[f"box_max_r{r}_{key}"]), (key, r)
            assert _eq(ops.box_min(v, r).cpu().numpy(), golden[f"box_min_r{r}_{key}"]), (key, r)


def test_offsets_golden(ops, golden):
    for key in _keys(golden):
        v = _dev(golden[f"in_{key}"])
        for shape in O.KernelShape:
            for size in (3, 5, 7):
                offs = O.kernel_offsets(O.make_kernel(shape, size))
                assert _eq(ops.offsets_max(v, offs).cpu().numpy(), golden[f"offs_max_{shape.value}{size}_{key}"])
                assert _eq(ops.offsets_min(v, offs).cpu().numpy(), golden[f"offs_min_{shape.value}{size}_{key}"])


def test_median_golden(ops, golden):
    for key in _keys(golden):
        v = _dev(golden[f"in_{key}"])
        for size in (3, 5, 7):
            assert _eq(ops.median(v, size).cpu().numpy(), golden[f"median{size}_{key}"]), (key, size)


def test_gaussian_golden(ops, golden):
    for key in _keys(golden):
        v = _dev(golden[f"in_{key}"])
        for (size, sigma) in ((5, 1.1), (3, 0.8), (7, 2.0)):
            w = O.gaussian_weights(size, sigma)
            ref = golden[f"gauss{size}_{sigma}_{key}"]
            fast = ops.gaussian_separable(v, w).cpu().numpy()
            assert np.abs(fast - ref).max() <= 1e-4, (key, size)
            exact = ops.gaussian_separable(v, w, exact=True).cpu().numpy()
            assert _eq(exact, ref), (key, size)  # fp64, reference operation order


def test_bilateral_golden(ops, golden):
    for key in _keys(golden):
        v = _dev(golden[f"in_{key}"])
        for (size, sv, ss) in ((5, 1.5, 2.0), (3, 0.5, 1.0), (7, 3.0, 1.5)):
            ref = golden[f"bilat{size}_{sv}_{ss}_{key}"]
            fast = ops.bilateral(v, size, sv, ss).cpu().numpy()
            assert np.abs(fast - ref).max() <= 1e-4, (key, size, np.abs(fast - ref).max())
            exact = ops.bilateral(v, size, sv, ss, exact=True).cpu().numpy()
            # device exp() is not glibc's: allow 1 float32 ulp
            assert np.abs(_bits(exact).astype(np.int64) - _bits(ref).astype(np.int64)).max() <= 1


def test_batched_ops_match_per_frame(ops):
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 90, size=(5, 37, 53)).astype(np.float32)
    x[rng.random(x.shape) < 0.6] = 0
    t = _dev(x)
    bm = ops.box_max(t, 3).cpu().numpy()
    md = ops.median(t, 5).cpu().numpy()
    for i in range(5):
        assert _eq(bm[i], O.box_max(x[i], 3))
        assert _eq(md[i], O.median_filter(x[i], 5))


def test_stage_kernels(ops, golden_dir):
    z = np.load(golden_dir / "stages_small.npz")
    for key in [k[3:] for k in z.files if k.startswith("in_")]:
        v = z[f"in_{key}"]
        inv, st = ops.invert(_dev(v), 100.0)
        assert _eq(inv.cpu().numpy(), z[f"invert_{key}"])
        assert int(st.cpu()[0]) == 0
        back, _ = ops.invert(inv, 100.0)
        assert _eq(back.cpu().numpy(), z[f"invert_back_{key}"])
        assert _eq(ops.extend_to_top(inv).cpu().numpy(), z[f"extend_{key}"])
        for size in (3, 7, 31):
            k = f"mfill{size}_{key}"
            if k in z.files:
                got = ops.masked_fill(inv, ops.box_max(inv, size // 2)).cpu().numpy()
                assert _eq(got, z[k])


def test_invert_range_and_validate(ops):
    x = np.zeros((3, 4, 5), np.float32)
    x[0, 1, 1] = 100.0
    x[1, 2, 2] = 5.0
    _, st = ops.invert(_dev(x), 100.0)
    assert st.cpu().tolist() == [8, 0, 0]
    x[1, 0, 0] = -1.0
    x[2, 0, 0] = np.inf
    st, nv = ops.validate(_dev(x))
    st = st.cpu().tolist()
    assert st[0] == 0 and st[1] == 2 and st[2] == 1  # inf > 0.1 counts as "valid" (pipeline.py:138)
    assert nv.cpu().tolist() == [1, 1, 1]
    st, nv = ops.validate(_dev(np.zeros((2, 3, 3), np.float32)))
    assert st.cpu().tolist() == [4, 4] and nv.cpu().tolist() == [0, 0]


def test_count_empty_and_reimpose(ops):
    x = np.array([[[0.0, 0.1, 0.2], [5.0, 0.05, 7.0]]], np.float32)
    assert ops.count_empty(_dev(x)).cpu().tolist() == [3]
    b = np.full_like(x, 9.0)
    got = ops.reimpose(_dev(b), _dev(x)).cpu().numpy()
    assert _eq(got, np.where(x > np.float32(0.1), b, np.float32(0)))


def test_random_grids_bit_exact(ops):
    """SPEC.md:587 acceptance: selection ops bit-exact on many random grids."""
    rng = np.random.default_rng(11)
    for _ in range(60):
        h, w = rng.integers(1, 65, size=2)
        v = rng.uniform(0, 99, size=(h, w)).astype(np.float32)
        v[rng.random((h, w)) < rng.uniform(0.2, 0.9)] = 0
        t = _dev(v)
        shape = O.KernelShape(rng.choice([s.value for s in O.KernelShape]))
        size = int(rng.choice([3, 5, 7]))
        offs = O.kernel_offsets(O.make_kernel(shape, size))
        assert _eq(ops.offsets_max(t, offs).cpu().numpy(), O.offsets_max(v, offs))
        assert _eq(ops.offsets_min(t, offs).cpu().numpy(), O.offsets_min(v, offs))
        assert _eq(ops.box_max(t, 15).cpu().numpy(), O.box_max(v, 15))
        assert _eq(ops.median(t, 5).cpu().numpy(), O.median_filter(v, 5))
