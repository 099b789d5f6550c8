"""Exact inner solvers, GPU-backed: bottleneck matching value and the
open-loop TSP over the coarsened stage graph.

Mirrors hetsched/combinatorics.py's public surface (``bottleneck_value``
:128-131, ``open_loop_tsp`` :232-251, ``path_cost`` :68-79, the result
records :38-51) with the same validation messages.  The solvers run in the
sm_100a library (hs_bottleneck_batch / hs_path_batch); batched variants
take [B, m, m] / [B, k, k] stacks.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N

MAX_EXACT_TSP = 16
MAX_GPU_PATH_K = 16
MAX_GPU_MATCH_M = 64


@dataclass(frozen=True)
class MatchingResult:
    pairs: tuple[int, ...]
    bottleneck: float


@dataclass(frozen=True)
class PathResult:
    order: tuple[int, ...]
    total: float


def _checked_square(a, what: str) -> np.ndarray:
    m = np.asarray(a, dtype=float)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ValueError(f"{what} must be a square matrix, got shape {m.shape}")
    if m.shape[0] == 0:
        raise ValueError(f"{what} must be non-empty")
    if not np.all(np.isfinite(m)):
        raise ValueError(f"{what} must be finite")
    if np.any(m < 0):
        raise ValueError(f"{what} must be nonnegative")
    return m


def _checked_symmetric(a) -> np.ndarray:
    w = _checked_square(a, "weight matrix")
    if not np.array_equal(w, w.T):
        raise ValueError("weight matrix must be symmetric")
    return w


def path_cost(weights, order) -> float:
    """Right-to-left accumulated cost of a vertex sequence (combinatorics.py:68-79)."""
    w = np.asarray(weights, dtype=float)
    total = 0.0
    for i in range(len(order) - 2, -1, -1):
        total = float(w[order[i], order[i + 1]]) + total
    return total


def bottleneck_values(stack) -> np.ndarray:
    """bottleneck_value of each [m, m] matrix in a [B, m, m] stack (GPU)."""
    a = np.ascontiguousarray(stack, dtype=np.float64)
    if a.ndim != 3 or a.shape[1] != a.shape[2] or a.shape[1] == 0:
        raise ValueError(f"expected a [B, m, m] stack, got shape {a.shape}")
    if not np.all(np.isfinite(a)) or np.any(a < 0):
        raise ValueError("cost matrix must be finite and nonnegative")
    if a.shape[1] > MAX_GPU_MATCH_M:
        raise ValueError(f"GPU bottleneck search supports m <= {MAX_GPU_MATCH_M}, got {a.shape[1]}")
    torch = N.torch_cuda()
    dev = N.current_device()
    B, m = a.shape[0], a.shape[1]
    if B == 0:
        return np.empty(0)
    w = torch.from_numpy(a).to(f"cuda:{dev}")
    out = torch.empty(B, dtype=torch.float64, device=f"cuda:{dev}")
    N.check(N.lib().hs_bottleneck_batch(w.data_ptr(), m, B, out.data_ptr(), dev, N.stream_ptr(dev)),
            "hs_bottleneck_batch")
    return out.cpu().numpy()


def bottleneck_value(costs) -> float:
    """Smallest entry v such that entries <= v admit a perfect matching."""
    w = _checked_square(costs, "cost matrix")
    return float(bottleneck_values(w[None])[0])


def bottleneck_matchings(stack) -> tuple[np.ndarray, np.ndarray]:
    """Optimal bottleneck [B] and lexicographically smallest optimal pairing
    [B, m] (row -> column) of each matrix in a [B, m, m] stack (GPU)."""
    a = np.ascontiguousarray(stack, dtype=np.float64)
    if a.ndim != 3 or a.shape[1] != a.shape[2] or a.shape[1] == 0:
        raise ValueError(f"expected a [B, m, m] stack, got shape {a.shape}")
    if not np.all(np.isfinite(a)) or np.any(a < 0):
        raise ValueError("cost matrix must be finite and nonnegative")
    if a.shape[1] > MAX_GPU_MATCH_M:
        raise ValueError(f"GPU bottleneck search supports m <= {MAX_GPU_MATCH_M}, got {a.shape[1]}")
    B, m = a.shape[0], a.shape[1]
    if B == 0:
        return np.empty(0), np.empty((0, m), dtype=np.int64)
    torch = N.torch_cuda()
    dev = N.current_device()
    w = torch.from_numpy(a).to(f"cuda:{dev}")
    val = torch.empty(B, dtype=torch.float64, device=f"cuda:{dev}")
    pairs = torch.empty((B, m), dtype=torch.int8, device=f"cuda:{dev}")
    N.check(N.lib().hs_bottleneck_match_batch(w.data_ptr(), m, B, val.data_ptr(), pairs.data_ptr(), dev,
                                              N.stream_ptr(dev)), "hs_bottleneck_match_batch")
    return val.cpu().numpy(), pairs.cpu().numpy().astype(np.int64)


def bottleneck_perfect_matching(costs) -> MatchingResult:
    """Perfect matching minimizing the largest selected entry; among the
    optimal ones, the lexicographically smallest pairing
    (combinatorics.py:134-189)."""
    w = _checked_square(costs, "cost matrix")
    val, pairs = bottleneck_matchings(w[None])
    return MatchingResult(tuple(int(x) for x in pairs[0]), float(val[0]))


MAX_BRUTE_FORCE = 10


def _brute_force(w: np.ndarray, kind: int) -> tuple[tuple[int, ...], float]:
    k = w.shape[0]
    if k > MAX_BRUTE_FORCE:
        raise ValueError(f"brute force is limited to k <= {MAX_BRUTE_FORCE}, got {k}")
    torch = N.torch_cuda()
    dev = N.current_device()
    t = torch.from_numpy(np.ascontiguousarray(w)).to(f"cuda:{dev}")
    val = torch.empty(1, dtype=torch.float64, device=f"cuda:{dev}")
    perm = torch.empty(k, dtype=torch.int8, device=f"cuda:{dev}")
    N.check(N.lib().hs_brute_force(t.data_ptr(), k, kind, val.data_ptr(), perm.data_ptr(), dev, N.stream_ptr(dev)),
            "hs_brute_force")
    return tuple(int(x) for x in perm.cpu().numpy()), float(val.item())


def brute_force_bottleneck_matching(costs) -> MatchingResult:
    """All k! pairings on the GPU; the first (itertools order) optimum
    (combinatorics.py:192-207)."""
    w = _checked_square(costs, "cost matrix")
    perm, val = _brute_force(w, 0)
    return MatchingResult(perm, val)


def brute_force_open_loop_tsp(weights) -> PathResult:
    """Every directed vertex sequence on the GPU; the first optimum
    (combinatorics.py:345-361)."""
    w = _checked_symmetric(weights)
    if w.shape[0] > MAX_BRUTE_FORCE:
        raise ValueError(f"brute force is limited to k <= {MAX_BRUTE_FORCE}, got {w.shape[0]}")
    if w.shape[0] == 1:
        return PathResult((0,), 0.0)
    perm, val = _brute_force(w, 1)
    return PathResult(perm, val)


def open_loop_tsps(stack) -> tuple[np.ndarray, np.ndarray]:
    """Exact Held-Karp totals [B] and orders [B, k] of a [B, k, k] stack (GPU, k <= 8)."""
    a = np.ascontiguousarray(stack, dtype=np.float64)
    B, k = a.shape[0], a.shape[1]
    if k > MAX_GPU_PATH_K:
        raise NotImplementedError(f"GPU Held-Karp currently covers k <= {MAX_GPU_PATH_K}, got {k}")
    torch = N.torch_cuda()
    dev = N.current_device()
    w = torch.from_numpy(a).to(f"cuda:{dev}")
    tot = torch.empty(B, dtype=torch.float64, device=f"cuda:{dev}")
    order = torch.empty((B, k), dtype=torch.int8, device=f"cuda:{dev}")
    N.check(N.lib().hs_path_batch(w.data_ptr(), k, B, tot.data_ptr(), order.data_ptr(), dev, N.stream_ptr(dev)),
            "hs_path_batch")
    return tot.cpu().numpy(), order.cpu().numpy().astype(np.int64)


def heuristic_paths(stack) -> tuple[np.ndarray, np.ndarray]:
    """Nearest neighbour + 2-opt (combinatorics.py:299-342) on a [B, k, k]
    stack, k <= 64, one GPU thread per matrix."""
    a = np.ascontiguousarray(stack, dtype=np.float64)
    B, k = a.shape[0], a.shape[1]
    torch = N.torch_cuda()
    dev = N.current_device()
    w = torch.from_numpy(a).to(f"cuda:{dev}")
    tot = torch.empty(B, dtype=torch.float64, device=f"cuda:{dev}")
    order = torch.empty((B, k), dtype=torch.int8, device=f"cuda:{dev}")
    N.check(N.lib().hs_path_heuristic_batch(w.data_ptr(), k, B, tot.data_ptr(), order.data_ptr(), dev,
                                            N.stream_ptr(dev)), "hs_path_heuristic_batch")
    return tot.cpu().numpy(), order.cpu().numpy().astype(np.int64)


def open_loop_tsp(weights, heuristic: bool = False) -> PathResult:
    """Minimum-cost Hamiltonian path, endpoints free (exact up to 16 vertices)."""
    w = _checked_symmetric(weights)
    k = w.shape[0]
    if k == 1:
        return PathResult((0,), 0.0)
    if k > MAX_EXACT_TSP:
        if not heuristic:
            raise ValueError(
                f"exact path search is limited to {MAX_EXACT_TSP} vertices, got {k}; "
                "pass heuristic=True to accept an approximate tour")
        tot, order = heuristic_paths(w[None])
        return PathResult(tuple(int(x) for x in order[0]), float(tot[0]))
    tot, order = open_loop_tsps(w[None])
    return PathResult(tuple(int(x) for x in order[0]), float(tot[0]))
