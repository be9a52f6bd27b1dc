"""Seeded schedules for the asynchronous mode (DIGEST-A).

Input generation only (no DIGEST arithmetic): which worker finishes its next local
epoch when.  Both the oracle and the GPU path consume the same event list, so an
asynchronous run is reproducible and can be compared element by element.

* `straggler_delays`: SPEC's inject_delay -- the straggler part draws a
  delay U[low, high] per local epoch (the paper's 8-10 s), the others 0.
* `async_events`: a discrete-event clock (SPEC "Time model"): worker m's k-th local
  epoch ends at sum of (cost_m + delay_m,j) for j <= k; events are ordered by end
  time, ties by worker id.  Returns the worker id of every event.
"""
import numpy as np


def straggler_delays(num_parts, epochs, straggler, low, high, seed):
    """delays[m][k] for worker m's k-th local epoch; only `straggler` (or None) is delayed."""
    if low > high:
        raise ValueError("delay range: low > high")
    rng = np.random.default_rng(seed)
    d = np.zeros((num_parts, epochs))
    if straggler is not None:
        d[straggler] = rng.uniform(low, high, epochs)
    return d


def async_events(epochs, costs, delays=None):
    """Order of the M * epochs local-epoch completions (worker ids)."""
    costs = np.asarray(costs, np.float64)
    M = costs.size
    delays = np.zeros((M, epochs)) if delays is None else np.asarray(delays, np.float64)
    ends = np.cumsum(costs[:, None] + delays, axis=1)          # [M, epochs]
    keys = [(ends[m, k], m, k) for m in range(M) for k in range(epochs)]
    keys.sort()
    return [m for _, m, _ in keys]
