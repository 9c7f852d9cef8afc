"""Head training on the GPU (training.train_head -> k_train.cu) against the
reference's own training run (tests/golden/make_golden_train.py) and the
reference's training tests (pkg/tests/test_flow.py:253-292).

Bars: with the reference's features, the trained weights equal the
reference's within 1e-8 (float64, same RNG stream, only the summation order
differs); through the GPU encoder (precision f64) within 1e-6."""

import numpy as np
import pytest

from conftest import has_cuda, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("GPU tests need a CUDA device")


def _pkg():
    import paper_2504_19417_b200 as pkg
    return pkg


def _cfg(g):
    pkg = _pkg()
    return pkg.TrainConfig(hidden=int(g["hidden"]), epochs=int(g["epochs"]), batch_size=int(g["batch_size"]),
                           learning_rate=float(g["lr"]), seed=int(g["seed"]))


def test_training_matches_reference_run_on_reference_features():
    pkg = _pkg()
    g = load_golden("train_small")
    b = pkg.generate_bases(int(g["D"]))
    w = pkg.train_head(None, int(g["width"]), int(g["height"]), int(g["dx"]), int(g["dy"]), float(g["delta_t"]),
                       int(g["D"]), _cfg(g), b, features=(g["feats"], g["u"]))
    for k in ("w1", "b1", "w2", "b2"):
        np.testing.assert_allclose(getattr(w, k), g[k], rtol=0, atol=1e-8, err_msg=k)


def test_training_through_gpu_encoder_matches_reference_run():
    """NormalFlowRegressor.fit without weights (estimators.py:171-190): the
    GPU encoder (f64) feeds the GPU trainer."""
    pkg = _pkg()
    g = load_golden("train_small")
    reg = pkg.NormalFlowRegressor(delta_t=float(g["delta_t"]), delta_x=int(g["dx"]), delta_y=int(g["dy"]),
                                  embed_dim=int(g["D"]), width=int(g["width"]), height=int(g["height"]),
                                  precision="f64", hidden=int(g["hidden"]), epochs=int(g["epochs"]),
                                  batch_size=int(g["batch_size"]), learning_rate=float(g["lr"]),
                                  random_state=int(g["seed"]))
    reg.fit([g["X0"], g["X1"]], [g["u0"], g["u1"]])
    for k in ("w1", "b1", "w2", "b2"):
        np.testing.assert_allclose(getattr(reg.weights_, k), g[k], rtol=0, atol=1e-6, err_msg=k)
    flows = reg.predict(g["X0"])
    assert flows.shape == (len(g["X0"]), 2) and np.isfinite(flows).all()


def test_constant_dataset_reaches_near_zero_residual():
    """pkg/tests/test_flow.py:254-276: one repeated embedding and one target;
    b2 alone can satisfy the constraint."""
    pkg = _pkg()
    u = np.array([3.0, 1.0])
    X = np.array([[0.0, 8.0, 8.0]])
    ds = [(X, u[None, :]) for _ in range(8)]
    b = pkg.generate_bases(4)
    w = pkg.train_head(ds, 16, 16, 2, 2, 0.016, 4, pkg.TrainConfig(hidden=8, epochs=400, batch_size=8,
                                                                   learning_rate=3e-2, seed=0), b, precision="f64")
    reg = pkg.NormalFlowRegressor(delta_x=2, delta_y=2, embed_dim=4, width=16, height=16, precision="f64", weights=w)
    n_hat = reg.predict(X)[0]
    assert abs(n_hat @ (u - n_hat)) / np.linalg.norm(n_hat) < 1e-3


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_divergence_and_empty_dataset():
    """pkg/tests/test_flow.py:278-292."""
    pkg = _pkg()
    b = pkg.generate_bases(4)
    ds = [(np.array([[0.0, 8.0, 8.0]]), np.array([[1e300, 0.0]]))]
    with pytest.raises((pkg.TrainingDivergedError, ValueError)):
        pkg.train_head(ds, 16, 16, 2, 2, 0.016, 4, pkg.TrainConfig(hidden=4, epochs=5, learning_rate=1e200), b,
                       precision="f64")
    with pytest.raises(ValueError, match="empty"):
        pkg.train_head([], 16, 16, 2, 2, 0.016, 4, pkg.TrainConfig(epochs=1), b)


def test_fit_then_predict_shapes_and_pipeline():
    """pkg/tests/test_estimators.py:97-115: fit on three slices then predict
    (training on the GPU), and the encoder inside an sklearn Pipeline."""
    from sklearn.pipeline import Pipeline
    pkg = _pkg()
    rng = np.random.default_rng(5)

    def make_events(n):
        t = np.sort(rng.uniform(0, 0.03, n))
        return np.stack([t, rng.integers(0, 64, n), rng.integers(0, 64, n)], 1).astype(np.float64)

    slices = [make_events(30) for _ in range(3)]
    targets = [np.tile([20.0, 0.0], (30, 1)) for _ in range(3)]
    reg = pkg.NormalFlowRegressor(delta_t=0.016, delta_x=4, delta_y=4, embed_dim=8, width=64, height=64,
                                  hidden=8, epochs=5)
    reg.fit(slices, targets)
    flows = reg.predict(slices[0])
    assert flows.shape == (30, 2) and np.all(np.isfinite(flows))
    pipe = Pipeline([("encode", pkg.LocalEventEncoder(delta_t=0.016, delta_x=4, delta_y=4, embed_dim=8,
                                                       width=64, height=64))])
    feats = pipe.fit_transform(make_events(12))
    assert feats.shape == (12, 16)
