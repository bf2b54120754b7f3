"""Contrastive critic losses over the logits matrix — oracle, fp64.

Paper: §3.1 P:197-199 (symmetric InfoNCE, the default critic objective); App. A.2
P:619-630 (InfoNCE-fwd Eq. P:621-622, InfoNCE-bwd P:624-625, InfoNCE-sym = fwd + bwd
P:628-630); logsumexp regulariser with coefficient 0.1: §5.3, Table 2, Alg. 1
P:1052-1053 ("L_Critic + beta L_logsumexp").
Readings: A-02 the denominator runs over the whole batch, j = 1..N,
positive included; A-03 mean (1/N), not sum; A-04 sym = fwd + bwd; A-05 penalty
P = beta * mean_i LSE_i^2 over ROWS only, for every loss kind.

  LSE_i  = log sum_j exp(l_ij)      (row logsumexp, max-shifted)
  LSE'_j = log sum_i exp(l_ij)      (column logsumexp)
  L_fwd  = (1/N) sum_i (LSE_i  - l_ii)
  L_bwd  = (1/N) sum_j (LSE'_j - l_jj)
  P      = beta (1/N) sum_i LSE_i^2
  L      = c_f L_fwd + c_b L_bwd + P,   (c_f, c_b) = (1,0) fwd, (0,1) bwd, (1,1) sym
  dL/dl_ij = (1/N)[c_f (p_ij - delta_ij) + c_b (q_ij - delta_ij)] + (2 beta/N) LSE_i p_ij,
      p_ij = exp(l_ij - LSE_i),  q_ij = exp(l_ij - LSE'_j)

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

LOSS_COEF = {"fwd": (1.0, 0.0), "bwd": (0.0, 1.0), "sym": (1.0, 1.0)}


def lse_rows(l):
    l = np.asarray(l, np.float64)
    m = l.max(axis=1)
    return m + np.log(np.exp(l - m[:, None]).sum(axis=1))


def lse_cols(l):
    return lse_rows(np.asarray(l, np.float64).T)


def loss_and_grad(l, kind="sym", beta=0.1):
    """Returns (dict of components, G = dL/dl)."""
    l = np.asarray(l, np.float64)
    N = l.shape[0]
    cf, cb = LOSS_COEF[kind]
    lse = lse_rows(l)
    lsec = lse_cols(l)
    diag = np.diag(l)
    L_fwd = np.mean(lse - diag)
    L_bwd = np.mean(lsec - diag)
    P = beta * np.mean(lse ** 2)
    total = cf * L_fwd + cb * L_bwd + P
    p = np.exp(l - lse[:, None])
    q = np.exp(l - lsec[None, :])
    I = np.eye(N)
    G = (cf * (p - I) + cb * (q - I)) / N + (2.0 * beta / N) * lse[:, None] * p
    comps = dict(L_fwd=L_fwd, L_bwd=L_bwd, penalty=P, total=total, lse_row=lse, lse_col=lsec)
    return comps, G
