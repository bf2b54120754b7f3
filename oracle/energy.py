"""Critic energies f(phi_i, psi_j) and their vector-Jacobian products — oracle, fp64.

Paper: App. A.2 P:607-617 ("The full list of evaluated energy functions"):
  f_cos = <phi,psi> / (||phi||_2 ||psi||_2)
  f_dot = <phi,psi>
  f_L2  = -||phi - psi||_2                       (sign per A-01, the main text P:201
                                                  prints it without the minus)
  f_L1  = -||phi - psi||_1           [§8(f) F3]
  f_L2sq = -||phi - psi||_2^2                    ("L2 w/o sqrt") [§8(f) F3]
Readings: A-06 eps2 = 1e-12 inside the L2 square root; cosine norms clamped at 1e-8;
A-33 the L1 derivative at a tie (phi_k = psi_k) is 0 (np.sign), a subgradient.

The logits are computed in *difference form* (sum over k of (phi_ik - psi_jk)^2), never
as ||phi||^2 + ||psi||^2 - 2 phi.psi, so the oracle has no cancellation.

VJPs, given G = dL/dl (N x N), written out:
  dot: dPhi = G Psi,  dPsi = G^T Phi
  L2sq: dphi_i = 2 sum_j G_ij (psi_j - phi_i),  dpsi_j = 2 sum_i G_ij (phi_i - psi_j)
  L1 : dphi_ik = -sum_j G_ij sign(phi_ik - psi_jk),  dpsi_jk = -sum_i G_ij sign(psi_jk - phi_ik)
  L2 : r_ij = sqrt(d_ij^2 + eps2),  W = G / r;
       dphi_i = sum_j W_ij (psi_j - phi_i),  dpsi_j = sum_i W_ij (phi_i - psi_j)
  cos: u = phi / n_phi, v = psi / n_psi (n = max(||.||, 1e-8));  du = G v,  dv = G^T u;
       dphi_i = (du_i - (du_i . u_i) u_i) / ||phi_i||   if ||phi_i|| > 1e-8 else du_i / 1e-8

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

EPS_L2 = 1e-12
EPS_COS = 1e-8
ENERGIES = ("l2", "dot", "cos", "l1", "l2sq")


def _sqdist_rows(phi_rows, psi):
    """d^2[i][j] = sum_k (phi_ik - psi_jk)^2 for a block of rows (difference form)."""
    diff = phi_rows[:, None, :] - psi[None, :, :]
    return np.einsum("ijk,ijk->ij", diff, diff)


def sqdist(phi, psi, block=64):
    phi = np.asarray(phi, np.float64); psi = np.asarray(psi, np.float64)
    out = np.empty((phi.shape[0], psi.shape[0]))
    for i0 in range(0, phi.shape[0], block):       # row blocks only bound the temporary
        out[i0:i0 + block] = _sqdist_rows(phi[i0:i0 + block], psi)
    return out


def l1dist(phi, psi, block=64):
    """sum_k |phi_ik - psi_jk| (written out, row blocks bound the temporary)."""
    phi = np.asarray(phi, np.float64); psi = np.asarray(psi, np.float64)
    out = np.empty((phi.shape[0], psi.shape[0]))
    for i0 in range(0, phi.shape[0], block):
        out[i0:i0 + block] = np.abs(phi[i0:i0 + block, None, :] - psi[None, :, :]).sum(2)
    return out


def logits(kind, phi, psi):
    phi = np.asarray(phi, np.float64); psi = np.asarray(psi, np.float64)
    if kind == "l2":
        return -np.sqrt(sqdist(phi, psi) + EPS_L2)
    if kind == "l2sq":
        return -sqdist(phi, psi)
    if kind == "l1":
        return -l1dist(phi, psi)
    if kind == "dot":
        return phi @ psi.T
    if kind == "cos":
        nphi = np.maximum(np.linalg.norm(phi, axis=1), EPS_COS)
        npsi = np.maximum(np.linalg.norm(psi, axis=1), EPS_COS)
        return (phi @ psi.T) / nphi[:, None] / npsi[None, :]
    raise ValueError(kind)


def diag_logits(kind, phi, psi):
    """l_ii = f(phi_i, psi_i) (the positives), O(N D)."""
    phi = np.asarray(phi, np.float64); psi = np.asarray(psi, np.float64)
    if kind == "l2":
        return -np.sqrt(((phi - psi) ** 2).sum(1) + EPS_L2)
    if kind == "l2sq":
        return -((phi - psi) ** 2).sum(1)
    if kind == "l1":
        return -np.abs(phi - psi).sum(1)
    if kind == "dot":
        return (phi * psi).sum(1)
    if kind == "cos":
        nphi = np.maximum(np.linalg.norm(phi, axis=1), EPS_COS)
        npsi = np.maximum(np.linalg.norm(psi, axis=1), EPS_COS)
        return (phi * psi).sum(1) / nphi / npsi
    raise ValueError(kind)


def _cos_back(x, du):
    nrm = np.linalg.norm(x, axis=1)
    n = np.maximum(nrm, EPS_COS)
    u = x / n[:, None]
    proj = (du * u).sum(1)
    big = nrm > EPS_COS
    out = np.where(big[:, None], (du - proj[:, None] * u) / n[:, None], du / EPS_COS)
    return out


def vjp(kind, phi, psi, G):
    """(dPhi, dPsi) = the VJP of the logits map at (phi, psi) applied to G."""
    phi = np.asarray(phi, np.float64); psi = np.asarray(psi, np.float64)
    G = np.asarray(G, np.float64)
    if kind == "dot":
        return G @ psi, G.T @ phi
    if kind == "l2sq":
        dphi = 2.0 * (G @ psi - G.sum(1)[:, None] * phi)
        dpsi = 2.0 * (G.T @ phi - G.sum(0)[:, None] * psi)
        return dphi, dpsi
    if kind == "l1":
        dphi = np.zeros_like(phi); dpsi = np.zeros_like(psi)
        for i in range(phi.shape[0]):                  # sign(phi_i - psi_j) per element
            sg = np.sign(phi[i][None, :] - psi)        # [N_psi][D]
            dphi[i] = -(G[i][:, None] * sg).sum(0)
            dpsi += G[i][:, None] * sg                 # d/dpsi_j of -|phi_i - psi_j| = +sign(phi_i - psi_j)
        return dphi, dpsi
    if kind == "l2":
        r = np.sqrt(sqdist(phi, psi) + EPS_L2)
        W = G / r
        dphi = W @ psi - W.sum(1)[:, None] * phi
        dpsi = W.T @ phi - W.sum(0)[:, None] * psi
        return dphi, dpsi
    if kind == "cos":
        nphi = np.maximum(np.linalg.norm(phi, axis=1), EPS_COS)
        npsi = np.maximum(np.linalg.norm(psi, axis=1), EPS_COS)
        u = phi / nphi[:, None]
        v = psi / npsi[:, None]
        du = G @ v
        dv = G.T @ u
        return _cos_back(phi, du), _cos_back(psi, dv)
    raise ValueError(kind)
