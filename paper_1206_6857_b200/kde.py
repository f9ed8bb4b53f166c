"""One-call KDE entry point and torch custom ops over the device engine.

``kde(queries, references, weights, bandwidth(s), epsilon)`` is the
convenience form of the reference's per-bandwidth loop (build_tree,
refresh_moments, dito_run; cli_harness.py:246-283): it builds the trees once,
runs every bandwidth in one device sweep and returns G for each query in
original order.  ``torch.ops.fastgauss_b200.*`` expose the exhaustive sum and
the sweep to torch code (CUDA float64 tensors in and out, on the current
stream), as SURVEY.md 8(b) proposes.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .spatial_index import PointStore, build_tree, build_tree_device
from .summation_engine import RunConfig, naive_sum, sweep_run


def kde(queries, references, weights=None, bandwidth=None, epsilon: float = 0.01,
        algorithm: str = "dito", leaf_threshold: int = 25, out=None):
    """G(x_q) = sum_r w_r exp(-|x_q - x_r|^2 / 2h^2) within relative error
    ``epsilon`` for every query and every bandwidth.

    ``queries`` may be ``None`` or the references themselves (monochromatic:
    one tree).  ``bandwidth`` is a scalar (returns shape (M,)) or a sequence
    (returns (len, M)).  ``algorithm`` is one of naive, dfd, dfdo, dito.
    Inputs may be NumPy arrays or CUDA float64 tensors; with CUDA inputs (or a
    CUDA ``out``) the result stays on the device.
    """
    if bandwidth is None:
        raise ValueError("bandwidth is required")
    hs = np.atleast_1d(np.asarray(bandwidth, dtype=float))
    if hs.size == 0 or np.any(hs <= 0.0):
        raise ValueError("bandwidths must be positive")
    mono = queries is None or queries is references
    on_device = _lib._is_torch(references) and references.is_cuda
    if algorithm == "naive":
        q = references if mono else queries
        vals = naive_sum(q, references, weights if weights is not None else
                         _ones_like(references), hs, out=out).values
        return vals[0] if np.ndim(bandwidth) == 0 and out is None else vals
    if on_device:
        rt = build_tree_device(references, weights, leaf_threshold)
        qt = rt if mono else build_tree_device(queries, None, leaf_threshold)
    else:
        rt = build_tree(PointStore(references, weights), leaf_threshold)
        qt = rt if mono else build_tree(PointStore(queries), leaf_threshold)
    if out is None and on_device:
        import torch

        out = torch.empty((hs.size, qt.n), dtype=torch.float64, device=references.device)
    cfg = RunConfig(bandwidth=float(hs[0]), epsilon=epsilon, algorithm=algorithm,
                    leaf_threshold=leaf_threshold)
    res = sweep_run(cfg, qt, rt, hs, out=out)
    vals = out if out is not None else np.stack([r.values for r in res])
    return vals[0] if np.ndim(bandwidth) == 0 else vals


def _ones_like(references):
    if _lib._is_torch(references):
        import torch

        return torch.ones(references.shape[0], dtype=torch.float64, device=references.device)
    return np.ones(np.asarray(references).shape[0])


def register_torch_ops() -> bool:
    """Register ``torch.ops.fastgauss_b200.{naive_sum, kde_sweep}`` (idempotent).
    Work runs on torch's current CUDA stream."""
    import torch

    if hasattr(torch.ops, "fastgauss_b200") and hasattr(torch.ops.fastgauss_b200, "kde_sweep"):
        return True

    def _on_current_stream(fn):
        # the engine runs on torch's current stream; the thread's previous
        # engine stream is restored afterwards
        def wrapped(*args):
            with _lib.torch_stream(torch.empty(0, device="cuda")):
                return fn(*args)
        return wrapped

    @torch.library.custom_op(
        "fastgauss_b200::naive_sum", mutates_args=(),
        schema="(Tensor queries, Tensor references, Tensor weights, float[] bandwidths) -> Tensor")
    def _naive(queries: torch.Tensor, references: torch.Tensor, weights: torch.Tensor,
               bandwidths: list[float]) -> torch.Tensor:
        out = torch.empty((len(bandwidths), queries.shape[0]), dtype=torch.float64,
                          device=queries.device)
        _on_current_stream(lambda: naive_sum(queries, references, weights, bandwidths,
                                             out=out))()
        return out

    @_naive.register_fake
    def _(queries, references, weights, bandwidths):
        return queries.new_empty((len(bandwidths), queries.shape[0]))

    @torch.library.custom_op(
        "fastgauss_b200::kde_sweep", mutates_args=(),
        schema="(Tensor points, Tensor weights, float[] bandwidths, float epsilon, "
               "int leaf_threshold) -> Tensor")
    def _sweep(points: torch.Tensor, weights: torch.Tensor, bandwidths: list[float],
               epsilon: float, leaf_threshold: int) -> torch.Tensor:
        out = torch.empty((len(bandwidths), points.shape[0]), dtype=torch.float64,
                          device=points.device)
        _on_current_stream(lambda: kde(None, points, weights, list(bandwidths), epsilon,
                                       "dito", leaf_threshold, out=out))()
        return out

    @_sweep.register_fake
    def _(points, weights, bandwidths, epsilon, leaf_threshold):
        return points.new_empty((len(bandwidths), points.shape[0]))

    return True
