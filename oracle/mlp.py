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
