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

LOSS_COEF = {"fwd": (1.0, 0.0), "bwd": (0.0, 1.0), "sym": (1.0, 1.0),
             "flatnce_fwd": (1.0, 0.0), "flatnce_bwd": (0.0, 1.0)}
FLAT = ("flatnce_fwd", "flatnce_bwd")


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
    if kind in PAIRWISE:
        # pair / FB objectives (F3) + the same row logsumexp penalty (reading A-05)
        lse = lse_rows(l)
        P = beta * np.mean(lse ** 2)
        Lp = pairwise_loss(l, kind)
        p = np.exp(l - lse[:, None])
        G = pairwise_grad(l, kind) + (2.0 * beta / N) * lse[:, None] * p
        comps = dict(L_fwd=Lp, L_bwd=0.0, penalty=P, total=Lp + P, lse_row=lse, lse_col=lse_cols(l))
        return comps, G
    cf, cb = LOSS_COEF[kind]
    lse = lse_rows(l)
    lsec = lse_cols(l)
    diag = np.diag(l)
    G = grad_rows(l, np.arange(N), lse, lsec, kind, beta)
    L_fwd = np.mean(lse - diag)
    L_bwd = np.mean(lsec - diag)
    P = beta * np.mean(lse ** 2)
    total = cf * L_fwd + cb * L_bwd + P
    if kind in FLAT:
        # FlatNCE (reading A-24): L = (1/N) sum_i log(S_i / sg[S_i]) with
        # S_i = sum_j exp(l_ij - l_ii): value 0; its gradient, written out,
        #   dL/dl_ij = (1/N) exp(l_ij - l_ii) / S_i = p_ij / N (j != i),
        #   dL/dl_ii = -(1/N) (S_i - 1) / S_i = (p_ii - 1) / N,
        # is the InfoNCE gradient above (bwd: the same with columns)
        L_fwd = 0.0
        L_bwd = 0.0
        total = P
    comps = dict(L_fwd=L_fwd, L_bwd=L_bwd, penalty=P, total=total, lse_row=lse, lse_col=lsec)
    return comps, G


def grad_rows(l_rows, row_ids, lse, lsec, kind="sym", beta=0.1):
    """Rows `row_ids` of dL/dl (InfoNCE family) from those logits rows and the statistics:
    G_ij = (1/N)[c_f (p_ij - delta_ij) + c_b (q_ij - delta_ij)] + (2 beta / N) LSE_i p_ij,
    p = exp(l_ij - LSE_i), q = exp(l_ij - LSE'_j).  loss_and_grad uses it for the whole
    matrix; the full-size GPU tests use it for sampled rows (statistics from blockwise passes)."""
    l_rows = np.asarray(l_rows, np.float64)
    row_ids = np.asarray(row_ids)
    N = l_rows.shape[1]
    cf, cb = LOSS_COEF[kind]
    li = lse[row_ids][:, None]
    p = np.exp(l_rows - li)
    q = np.exp(l_rows - np.asarray(lsec)[None, :])
    D = np.zeros_like(l_rows)
    D[np.arange(len(row_ids)), row_ids] = 1.0
    return (cf * (p - D) + cb * (q - D)) / N + (2.0 * beta / N) * li * p


PAIRWISE = ("fb", "dpo", "ipo", "sppo")


def pairwise_loss(l, kind):
    """The pair / FB objectives of App. A.2 P:643-658 written out, mean over the N positives
    (reading A-03: 1/N for the double sums as for InfoNCE; reading A-34: the printed j-range,
    j = 1..N including j = i, except FB's j != i).  d_i = l_ii.
      FB  : (1/N) [ -sum_i e^{d_i} + (1/(2(N-1))) sum_i sum_{j!=i} e^{2 l_ij} ]
      DPO : (1/N) sum_i sum_j -log sigmoid(d_i - l_ij)
      IPO : (1/N) sum_i sum_j ((d_i - l_ij) - 1)^2
      SPPO: (1/N) sum_i sum_j [(d_i - 1)^2 + (l_ij + 1)^2]"""
    l = np.asarray(l, np.float64)
    N = l.shape[0]
    d = np.diag(l)
    off = ~np.eye(N, dtype=bool)
    if kind == "fb":
        return (-np.exp(d).sum() + (np.exp(2.0 * l)[off]).sum() / (2.0 * max(N - 1, 1))) / N
    if kind == "dpo":
        return np.logaddexp(0.0, l - d[:, None]).sum() / N             # -log sigmoid(x) = log(1 + e^-x)
    if kind == "ipo":
        return (((d[:, None] - l) - 1.0) ** 2).sum() / N
    if kind == "sppo":
        return (N * ((d - 1.0) ** 2).sum() + ((l + 1.0) ** 2).sum()) / N
    raise ValueError(kind)


def pairwise_grad(l, kind):
    """dL/dl of pairwise_loss, derived by hand (pinned by finite differences in the tests):
      off-diagonal g_ij = h(l_ij, d_i) / N, diagonal g_ii = D_i / N with
      FB  : h = e^{2l} / (N-1),        D_i = -e^{d_i}
      DPO : h = sigmoid(l - d),        D_i = -sum_{j!=i} h_ij
      IPO : h = 2 (l - d + 1),         D_i = -sum_{j!=i} h_ij
      SPPO: h = 2 (l + 1),             D_i = 2 (d_i + 1) + 2 N (d_i - 1)"""
    l = np.asarray(l, np.float64)
    N = l.shape[0]
    d = np.diag(l)
    off = ~np.eye(N, dtype=bool)
    if kind == "fb":
        h = np.exp(2.0 * l) / max(N - 1, 1)
        D = -np.exp(d)
    elif kind == "dpo":
        h = 1.0 / (1.0 + np.exp(-(l - d[:, None])))
        D = -np.where(off, h, 0.0).sum(1)
    elif kind == "ipo":
        h = 2.0 * (l - d[:, None] + 1.0)
        D = -np.where(off, h, 0.0).sum(1)
    elif kind == "sppo":
        h = 2.0 * (l + 1.0)
        D = 2.0 * (d + 1.0) + 2.0 * N * (d - 1.0)
    else:
        raise ValueError(kind)
    G = np.where(off, h, 0.0)
    G[np.arange(N), np.arange(N)] = D
    return G / N


def flatnce_literal(l, l_detached, kind="flatnce_fwd"):
    """The printed FlatNCE objective with an explicit stop-gradient argument (A-24 sign):
    (1/N) sum_i log(S_i(l) / S_i(l_detached)), S_i = sum_j exp(l_ij - l_ii); columns for bwd.
    Used by the tests to pin the gradient above by finite differences."""
    l = np.asarray(l, np.float64); l0 = np.asarray(l_detached, np.float64)
    if kind == "flatnce_bwd":
        l, l0 = l.T, l0.T
    d = np.diag(l)[:, None]; d0 = np.diag(l0)[:, None]
    S = np.exp(l - d).sum(1); S0 = np.exp(l0 - d0).sum(1)
    return float(np.mean(np.log(S / S0)))
