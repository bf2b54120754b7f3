"""Bias-corrected Adam — oracle, fp64.

Paper: the optimiser is never named.  Alg. 1 P:1051 writes a plain gradient step
"(phi, psi) <- (phi, psi) - alpha grad"; Table 2 P:938-939 gives only the learning rates
(critic_lr 3e-4, policy_lr 6e-4).  north_star fixes "the fused Adam update"; reading A-15:
beta1 0.9, beta2 0.999, eps 1e-8 outside the square root, bias correction, decoupled
weight decay default 0 (App. E P:1012 lists weight decay among failed experiments).

  t <- t + 1
  m <- b1 m + (1 - b1) g
  v <- b2 v + (1 - b2) g^2
  p <- p - lr ( (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps) + wd p )

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np


def adam_step(p, g, m, v, t, lr=3e-4, b1=0.9, b2=0.999, eps=1e-8, wd=0.0):
    """Returns (p', m', v', t') — t is the number of steps taken BEFORE this one."""
    p = np.asarray(p, np.float64); g = np.asarray(g, np.float64)
    m = np.asarray(m, np.float64); v = np.asarray(v, np.float64)
    if not np.all(np.isfinite(g)):
        raise FloatingPointError("non-finite gradient")
    t = t + 1
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mhat = m / (1.0 - b1 ** t)
    vhat = v / (1.0 - b2 ** t)
    p_new = p - lr * (mhat / (np.sqrt(vhat) + eps) + wd * p)
    return p_new, m, v, t
