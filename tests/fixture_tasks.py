"""A training task for the run_training parity tests (test infrastructure).

It follows the reference's task protocol (tasks.py: parameter_count,
batch_size, metric_name, initial_weights, gradient, evaluate) and takes the
gradient-vector type as a factory, so the same task drives the reference's
run_training (golden fixtures, tests/golden/make_golden.py) and this
package's (tests/test_gpu_training.py).
"""
import numpy as np


class NoisyBowl:
    """0.5 * sum(c * (w - w*)^2) with per-sample Gaussian gradient noise averaged
    over the batch; the data stream is rng.split(0, worker, iteration), as the
    reference's tasks draw it (tasks.py:82-90)."""

    def __init__(self, size: int, make_vector, noise_std: float = 0.5, batch_size: int = 4, seed: int = 0):
        rs = np.random.default_rng(seed)
        self.size = size
        self.make_vector = make_vector
        self.noise_std = noise_std
        self.batch_size = batch_size
        self.curvature = rs.uniform(0.5, 2.0, size)
        self.w_star = rs.standard_normal(size)

    @property
    def parameter_count(self) -> int:
        return self.size

    @property
    def metric_name(self) -> str:
        return "loss"

    def initial_weights(self, rng):
        del rng
        return self.w_star + 1.0

    def loss(self, w) -> float:
        d = np.asarray(w, dtype=np.float64) - self.w_star
        return float(0.5 * np.dot(self.curvature * d, d))

    def gradient(self, w, worker: int, iteration: int, rng):
        d = np.asarray(w, dtype=np.float64) - self.w_star
        noise = rng.split(0, worker, iteration).generator.standard_normal((self.batch_size, self.size))
        grad = self.curvature * d + self.noise_std * noise.mean(axis=0)
        return self.make_vector(grad.astype(np.float32)), self.loss(w)

    def evaluate(self, w, rng, n_samples: int = 0) -> dict:
        del rng, n_samples
        return {"loss": self.loss(w)}


# the run_training cases of tests/golden/training.npz:
# (mode, compressor, static_cf, theta_min, epsilon, workers, size, iterations, lr, momentum)
TRAINING_CASES = [
    ("gravac", "topk", None, 4.0, 0.3, 2, 20_000, 12, 0.05, 0.9),
    ("gravac", "redsync", None, 4.0, 0.2, 3, 12_000, 10, 0.05, 0.0),
    ("static-cf", "topk", 8.0, None, None, 2, 20_000, 12, 0.05, 0.9),
    ("static-cf", "redsync", 4.0, None, None, 2, 10_000, 8, 0.05, 0.0),
    ("dense", None, None, None, None, 2, 10_000, 6, 0.05, 0.5),
]
TRACE_COLUMNS = ("iter", "cf", "gain_min", "gain_c", "t_o", "t_compress", "t_s", "t_iter", "tsys", "tcomp",
                 "loss", "floats_sent", "words_sent", "theta_min")
CHOICES = {"candidate": 0, "minimum": 1, "dense": 2, "static": 3}
