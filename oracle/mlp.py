"""phi(s,a) / psi(g) encoder MLPs — oracle, fp64.

Paper: §3.1 P:193-195 ("the state-action pair and goal state representations, phi(s,a)
and psi(g)"); Table 2 P:943-944 (hidden layers [256,256], representation dimension 64);
§5.4 P:387-465 (width/depth up to 4x1024).  Readings: A-13 hidden activation SiLU
(ReLU optional), A-16 affine output layer, A-14 initialisation is an input.

Layer l (hidden):  Z_l = X_l W_l + b_l,  X_{l+1} = act(Z_l)
Output:            Y   = X_d W_o + b_o
Backward (reverse mode, written out):
  dZ_o = dY;  for each layer from the output down:  dW = X^T dZ,  db = sum_rows dZ,
  dX = dZ W^T;  dZ_{l} = dX_{l+1} * act'(Z_l).

Flat parameter layout (shared *convention* with include/crl.h, not code): for each layer
W[in][out] row-major then b[out].

LayerNorm variant (§5.4 P:462-465 "adding layer normalization before every activation",
App. A.4; reading A-35: per-row over the features, learnable gain
gamma and shift beta, eps = 1e-6 inside the square root (flax default)):
  hidden:  Z_l = X_l W_l + b_l,  Zh = (Z_l - mu) / sqrt(var + eps),  Y_l = gamma Zh + beta,
           X_{l+1} = act(Y_l)
  layout per hidden layer: W, b, gamma[out], beta[out]; output layer W, b.
  backward: dY = dX_{l+1} * act'(Y);  dgamma = sum_rows dY Zh,  dbeta = sum_rows dY;
           dZ = rstd (g - mean(g) - Zh mean(g Zh)),  g = dY gamma  (row means over features)

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np


def layer_dims(in_dim, depth, width, out_dim):
    dims = [in_dim] + [width] * depth + [out_dim]
    return [(dims[i], dims[i + 1]) for i in range(len(dims) - 1)]


def unpack(flat, in_dim, depth, width, out_dim):
    """Flat vector -> list of (W[in][out], b[out]) in fp64.  Returns (layers, n_used)."""
    flat = np.asarray(flat, np.float64)
    layers, off = [], 0
    for fi, fo in layer_dims(in_dim, depth, width, out_dim):
        W = flat[off:off + fi * fo].reshape(fi, fo); off += fi * fo
        b = flat[off:off + fo]; off += fo
        layers.append((W, b))
    return layers, off


def pack(layers):
    return np.concatenate([np.concatenate([W.ravel(), b.ravel()]) for W, b in layers])


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def act_fn(z, kind):
    if kind == "silu":
        return z * sigmoid(z)                   # SiLU(z) = z sigma(z)
    if kind == "relu":
        return np.maximum(z, 0.0)
    raise ValueError(kind)


def act_grad(z, kind):
    if kind == "silu":
        s = sigmoid(z)
        return s * (1.0 + z * (1.0 - s))        # d/dz z sigma(z)
    if kind == "relu":
        return (z > 0.0).astype(np.float64)     # ReLU'(0) := 0
    raise ValueError(kind)


def forward(layers, x, act="silu"):
    """Returns (Y, cache) with cache = (Xs, Zs): Xs[l] is the input of layer l, Zs[l] the
    pre-activation of hidden layer l."""
    X = np.asarray(x, np.float64)
    Xs, Zs = [], []
    for l, (W, b) in enumerate(layers):
        Xs.append(X)
        Z = X @ W + b
        if l < len(layers) - 1:
            Zs.append(Z)
            X = act_fn(Z, act)
        else:
            X = Z
    return X, (Xs, Zs)


def backward(layers, cache, dY, act="silu"):
    """Returns (grads as list of (dW, db), dX0)."""
    Xs, Zs = cache
    dZ = np.asarray(dY, np.float64)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        W, _ = layers[l]
        grads[l] = (Xs[l].T @ dZ, dZ.sum(axis=0))
        dX = dZ @ W.T
        if l > 0:
            dZ = dX * act_grad(Zs[l - 1], act)
    return grads, dX


LN_EPS = 1e-6


def unpack_ln(flat, in_dim, depth, width, out_dim):
    """Flat vector -> list of layers; hidden layers are (W, b, gamma, beta), the output
    layer (W, b).  Returns (layers, n_used)."""
    flat = np.asarray(flat, np.float64)
    layers, off = [], 0
    dims = layer_dims(in_dim, depth, width, out_dim)
    for li, (fi, fo) in enumerate(dims):
        W = flat[off:off + fi * fo].reshape(fi, fo); off += fi * fo
        b = flat[off:off + fo]; off += fo
        if li < len(dims) - 1:
            gm = flat[off:off + fo]; off += fo
            bt = flat[off:off + fo]; off += fo
            layers.append((W, b, gm, bt))
        else:
            layers.append((W, b))
    return layers, off


def pack_ln(layers):
    return np.concatenate([np.concatenate([t.ravel() for t in L]) for L in layers])


def forward_ln(layers, x, act="silu"):
    """Returns (Y, cache); cache = (Xs, Zs, Zhs, Ys, rstds)."""
    X = np.asarray(x, np.float64)
    Xs, Zs, Zhs, Ys, rs = [], [], [], [], []
    for l, L in enumerate(layers):
        Xs.append(X)
        Z = X @ L[0] + L[1]
        if l < len(layers) - 1:
            mu = Z.mean(axis=1, keepdims=True)
            var = ((Z - mu) ** 2).mean(axis=1, keepdims=True)
            rstd = 1.0 / np.sqrt(var + LN_EPS)
            Zh = (Z - mu) * rstd
            Y = L[2] * Zh + L[3]
            Zs.append(Z); Zhs.append(Zh); Ys.append(Y); rs.append(rstd)
            X = act_fn(Y, act)
        else:
            X = Z
    return X, (Xs, Zs, Zhs, Ys, rs)


def backward_ln(layers, cache, dY_out, act="silu"):
    """Returns (grads as list of tuples matching the layers, dX0)."""
    Xs, Zs, Zhs, Ys, rs = cache
    dZ = np.asarray(dY_out, np.float64)
    grads = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        W = layers[l][0]
        gW, gb = Xs[l].T @ dZ, dZ.sum(axis=0)
        if l < len(layers) - 1:
            grads[l] = (gW, gb) + grads[l][2:]
        else:
            grads[l] = (gW, gb)
        dX = dZ @ W.T
        if l > 0:
            k = l - 1
            dYk = dX * act_grad(Ys[k], act)
            gm = layers[k][2]
            Zh = Zhs[k]
            g = dYk * gm
            dZ = rs[k] * (g - g.mean(axis=1, keepdims=True) - Zh * (g * Zh).mean(axis=1, keepdims=True))
            grads[k] = (None, None, (dYk * Zh).sum(axis=0), dYk.sum(axis=0))
    return grads, dX
