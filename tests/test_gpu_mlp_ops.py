"""GPU: mlp.hpp's generic-net building blocks through the C ABI (lann_mlp_forward, lann_mse_loss,
lann_mse_gradient, lann_adam_update) against the reference library itself (oracle/_ref):
bit-identical (==) results for Mlp::forward, mse_loss, mse_gradient + LossGrad and
AdamState::update on random nets of 1-3 hidden layers (mlp.hpp:27-60, mlp.cpp:36-154)."""
import numpy as np
import pytest

from paper_2003_07497_b200.abi import ROW

pytestmark = pytest.mark.gpu


def random_nets(seed, count):
    rng = np.random.default_rng(seed)
    nets = []
    for k in range(count):
        depth = 1 + k % 3
        dims = [int(rng.integers(1, ROW + 1))] + [int(rng.integers(1, 17)) for _ in range(depth)] + [1]
        P = sum((dims[i] + 1) * dims[i + 1] for i in range(len(dims) - 1))
        params = rng.uniform(-1, 1, P)
        n = int(rng.integers(1, 300))
        X = np.zeros((n, ROW))
        X[:, : dims[0]] = rng.uniform(-1, 1, (n, dims[0]))
        y = rng.uniform(0, 1, n)
        nets.append((dims, params, X, y))
    return nets


def test_mse_gradient_is_the_reference(engine, reference):
    nets = random_nets(1, 24)
    loss, grads = engine.mse_gradient([(d, p, X[:, : d[0]], y) for d, p, X, y in nets])
    for k, (d, p, X, y) in enumerate(nets):
        st, rl, rg = reference.mse_gradient(d, p, X, y)
        assert st == 0
        assert loss[k] == rl
        assert np.array_equal(grads[k], rg), k


def test_mse_loss_and_forward_are_the_reference(engine, reference):
    nets = random_nets(2, 12)
    loss = engine.mse_loss([(d, p, X[:, : d[0]], y) for d, p, X, y in nets])
    fwd = engine.mlp_forward([(d, p, X[:, : d[0]]) for d, p, X, y in nets])
    off = 0
    for k, (d, p, X, y) in enumerate(nets):
        st, rl = reference.mse_loss(d, p, X, y)
        assert st == 0 and loss[k] == rl
        st, rf = reference.mlp_forward(d, p, X)
        assert st == 0 and np.array_equal(fwd[off: off + len(X)], rf)
        off += len(X)


def test_adam_update_is_the_reference(engine, reference):
    rng = np.random.default_rng(3)
    n, steps = 300, 40
    p0 = rng.uniform(-1, 1, n)
    grads = rng.normal(0, 1e-2, (steps, n))
    grads[:, :5] = 0.0  # never-active units
    grads[10:, 5:10] = 0.0  # units that stop being active
    p, m, v = p0.copy(), np.zeros(n), np.zeros(n)
    for k in range(steps):
        engine.adam_update(p, grads[k], m, v, k + 1, 1e-2)
    st, rp, rm, rv = reference.adam_steps(p0, grads, 1e-2)
    assert st == 0
    assert np.array_equal(p, rp) and np.array_equal(m, rm) and np.array_equal(v, rv)


def test_gradient_errors(engine):
    from paper_2003_07497_b200 import engine as E

    with pytest.raises(E.ParamError):  # two outputs: mse_gradient needs one
        engine.mse_gradient([([2, 3, 2], np.zeros(17), np.zeros((4, 2)), np.zeros(4))])
    with pytest.raises(E.ParamError):  # width over 64
        engine.mse_gradient([([2, 65, 1], np.zeros(3 * 65 + 66), np.zeros((4, 2)), np.zeros(4))])
