"""CPU oracle for the batched bootstrap filter -- TEST INFRASTRUCTURE ONLY.

Restates the reference's test-data generator and its closed-form filtering
oracle (``/root/reference/pkg/src/pfresample/pf.py``):

* ``simulate_observations`` -- pf.py:99-108, the reference's own draws
  (RngStream(seed, (4,)).generator(), standard normals), so tests see the
  same observation sequences the reference's tests do;
* ``exact_filter`` -- pf.py:207-229, the Kalman recursion the particle
  filter's estimates are checked against.

Only ``tests/`` (and developer scripts) import this module; the product
package ``paper_1301_4019_b200`` never does.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from oracle.pfr_oracle import generator

_NS_SIMULATE = 4  # pf.py:38


@dataclass
class ExactFilterResult:
    means: np.ndarray
    variances: np.ndarray
    log_likelihood: float


def simulate_observations(model, steps: int, seed: int) -> np.ndarray:
    """Synthetic observations y_1..y_T from the model, drawn exactly as the
    reference does (pf.py:99-108; host test-data helper)."""
    g = generator(seed, (_NS_SIMULATE,))
    x = model.initial_mean + model.initial_std * g.standard_normal()
    ys = np.empty(steps)
    for t in range(steps):
        x = model.coeff * x + model.trans_std * g.standard_normal()
        ys[t] = x + model.obs_std * g.standard_normal()
    return ys


def exact_filter(model, observations) -> ExactFilterResult:
    """Closed-form Gaussian filtering recursion (pf.py:207-229): the oracle the
    particle filter is validated against."""
    observations = np.asarray(observations, dtype=np.float64)
    m, p = model.initial_mean, model.initial_std ** 2
    means = np.empty(observations.size)
    variances = np.empty(observations.size)
    loglik = 0.0
    for t, y in enumerate(observations):
        m_pred = model.coeff * m
        p_pred = model.coeff ** 2 * p + model.trans_std ** 2
        s = p_pred + model.obs_std ** 2
        loglik += -0.5 * (math.log(2.0 * math.pi * s) + (y - m_pred) ** 2 / s)
        gain = p_pred / s
        m = m_pred + gain * (y - m_pred)
        p = (1.0 - gain) * p_pred
        means[t] = m
        variances[t] = p
    return ExactFilterResult(means, variances, loglik)
