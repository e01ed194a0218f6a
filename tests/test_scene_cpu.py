"""Host-side semantics of the drop-in containers (no kernels run; storage on the CPU device).

The reference's callers assign to these objects:
* ``scene.capacity = args.budget`` (io_cli.py:339-343);
* ``scene.positions = (...).astype(f32)`` and the other columns every iteration (splat2d.py:382-391);
* ``stats.edge_score = sample_scores(...)`` (splat2d.py:397).
The device scene must keep the value its kernels see within its allocation and copy assigned
columns into the storage the kernels read."""

import numpy as np
import pytest
import torch

from paper_2603_08661_b200.core import Scene2, Scene3
from paper_2603_08661_b200.densify_controller import DensifyStats


def _scene3(n=5, cap=8, k=16):
    rng = np.random.default_rng(0)
    return Scene3(rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 4)),
                  rng.normal(size=n), rng.random((n, k, 3)), capacity=cap, device="cpu")


def _scene2(n=5, cap=8):
    rng = np.random.default_rng(1)
    return Scene2(rng.normal(size=(n, 2)), rng.normal(size=(n, 2)), rng.normal(size=n),
                  rng.normal(size=n), rng.random((n, 3)), capacity=cap, device="cpu")


@pytest.mark.parametrize("make", [_scene3, _scene2])
def test_capacity_assignment_reserves_storage(make):
    s = make()
    before = {c: getattr(s, c).clone() for c in s._columns}
    s.capacity = 100                      # io_cli.py:339-343
    assert s.capacity == 100 and s.reserved_rows >= 100
    for attr in s._buffers:
        assert getattr(s, attr).shape[0] >= 100, attr
    for c, v in before.items():
        assert torch.equal(getattr(s, c), v), c
    s.capacity = 6                        # shrinking keeps the storage, lowers the budget
    assert s.capacity == 6 and s.reserved_rows >= 100
    s.capacity = 3                        # below count: allowed, validate() raises (core.py:135)
    with pytest.raises(ValueError):
        s.validate()
    with pytest.raises(ValueError):
        s.capacity = 0
    with pytest.raises(ValueError):
        s._set_count(4 + s.reserved_rows)


def test_scene3_column_assignment_copies_into_storage():
    s = _scene3()
    ptr = s._pos.data_ptr()
    new = np.arange(15, dtype=np.float64).reshape(5, 3)
    s.positions = new.astype(np.float32)
    assert s._pos.data_ptr() == ptr
    assert torch.equal(s._pos[:5], torch.from_numpy(new).float())
    s.colors = np.full((5, 3), 0.5)
    assert torch.equal(s._sh[:5, 0, :], torch.full((5, 3), 0.5))
    s.opacity_logits = torch.zeros(5, dtype=torch.float64)
    assert torch.equal(s._op[:5], torch.zeros(5))
    with pytest.raises(ValueError):
        s.positions = np.zeros((4, 3), np.float32)
    with pytest.raises(ValueError):
        s.rotations = np.zeros((5, 3), np.float32)


def test_scene2_column_assignment_is_not_shadowed():
    s = _scene2()
    s.positions = np.ones((5, 2), np.float32)
    s.thetas = np.full(5, 0.25, np.float32)
    assert "positions" not in s.__dict__
    assert torch.equal(s._cols["positions"][:5], torch.ones(5, 2))
    assert torch.equal(s._cols["thetas"][:5], torch.full((5,), 0.25))
    assert torch.equal(s.positions, torch.ones(5, 2))


def test_edge_score_assignment_checks_and_converts():
    st = DensifyStats(4, device="cpu")
    buf = st.edge_score.data_ptr()
    st.edge_score = np.array([0.1, 0.2, 0.3, 0.4], dtype=np.float32)   # numpy, float32
    assert st.edge_score.dtype == torch.float64 and st.edge_score.data_ptr() == buf
    assert torch.equal(st.edge_score, torch.tensor([0.1, 0.2, 0.3, 0.4], dtype=torch.float32)
                       .double())
    st.edge_score = torch.arange(4)                                      # integer tensor
    assert torch.equal(st.edge_score, torch.arange(4).double())
    with pytest.raises(ValueError):
        st.edge_score = np.zeros(3)
    with pytest.raises(ValueError):
        st.edge_score = np.zeros((4, 1))
    with pytest.raises(TypeError):
        st.edge_score = np.ones(4, bool)
    st.reset(6)
    assert len(st) == 6 and st.edge_score.shape == (6,)
    st.set_edge_score(np.ones(6))
    assert float(st.edge_score.sum()) == 6.0


def test_stats_reset_writes_nothing_and_reads_zeros():
    """DensifyStats.reset gives fresh statistics without a fill: stale buffer contents never
    leak (pending rows read as zeros), old tensors keep their values (new buffers, as the
    reference's new arrays), and assignments / accumulations see zeros underneath."""
    from paper_2603_08661_b200.densify_controller import accumulate_grads
    st = DensifyStats(5, device="cpu")
    accumulate_grads(st, np.arange(5.0))
    old = st._grad_sum
    st.reset(7)
    st._buf.fill_(float("nan"))                  # whatever the allocator hands back
    assert torch.equal(old, torch.arange(5.0, dtype=torch.float64))
    assert len(st) == 7 and st._accum_count == 0
    assert torch.equal(st.grad_norm, torch.zeros(7, dtype=torch.float64))
    st.edge_score = np.full(7, 0.5)
    assert torch.equal(st.edge_score, torch.full((7,), 0.5, dtype=torch.float64))
    assert torch.equal(st._grad_sum, torch.zeros(7, dtype=torch.float64))
    st.reset()
    st._buf.fill_(float("nan"))
    accumulate_grads(st, np.full(7, 2.0))
    assert torch.equal(st.grad_norm, torch.full((7,), 2.0, dtype=torch.float64))
    assert torch.equal(st.edge_score, torch.zeros(7, dtype=torch.float64))
