"""TEST INFRASTRUCTURE ONLY: fp64 numpy restatement of the ConvNet SPB step
(SURVEY.md 8f-1). The reference has no convolutional model, so this oracle
is NOT pinned by the reference ("parity unpinned" for the conv row); it is
pinned instead by a finite-difference gradient check (tests/test_conv.py),
and it reuses the reference-pinned SPB bookkeeping (suffix_layers,
layer_chunks, draw_batch from oracle.Oracle) and aggregation rule
(spb.cpp:70-106: each layer averaged over its contributing workers).

Model: h_l = tanh(conv3x3(h_{l-1}; W_l, stride_l, pad 1) + b_l), pooled =
mean over pixels of h_{L-1}, out = W_L pooled + b_L, loss 0.5 ||out - y||^2.
Block l = W_l [c_out x 9 c_in] (columns (ky*3+kx)*c_in + ci), then b_l.
"""
import numpy as np


def im2col(x, stride):
    B, H, W, C = x.shape
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    xp = np.pad(x, ((0, 0), (1, 1), (1, 1), (0, 0)))
    cols = np.empty((B, Ho, Wo, 9, C), dtype=x.dtype)
    for ky in range(3):
        for kx in range(3):
            cols[:, :, :, ky * 3 + kx, :] = xp[:, ky:ky + stride * (Ho - 1) + 1:stride, kx:kx + stride * (Wo - 1) + 1:stride, :]
    return cols.reshape(B * Ho * Wo, 9 * C), (Ho, Wo)


def col2im(dcols, in_shape, stride):
    B, H, W, C = in_shape
    Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
    d = dcols.reshape(B, Ho, Wo, 9, C)
    xp = np.zeros((B, H + 2, W + 2, C))
    for ky in range(3):
        for kx in range(3):
            xp[:, ky:ky + stride * (Ho - 1) + 1:stride, kx:kx + stride * (Wo - 1) + 1:stride, :] += d[:, :, :, ky * 3 + kx, :]
    return xp[:, 1:H + 1, 1:W + 1, :]


class ConvOracle:
    def __init__(self, in_shape, convs, nout):
        self.in_shape, self.convs, self.nout = tuple(in_shape), list(convs), nout
        self.L = len(convs) + 1
        self.cin = [in_shape[2]] + [c for c, _ in convs]

    def unpack(self, blocks):
        Ws, bs = [], []
        for l in range(self.L):
            co = self.convs[l][0] if l < self.L - 1 else self.nout
            fan = 9 * self.cin[l] if l < self.L - 1 else self.cin[-1]
            blk = np.asarray(blocks[l], dtype=np.float64)
            Ws.append(blk[:co * fan].reshape(co, fan))
            bs.append(blk[co * fan:co * fan + co])
        return Ws, bs

    def forward(self, blocks, X):
        Ws, bs = self.unpack(blocks)
        h, w, c = self.in_shape
        a = np.asarray(X, dtype=np.float64).reshape(-1, h, w, c)
        acts, cols = [a], []
        for l, (co, st) in enumerate(self.convs):
            col, (Ho, Wo) = im2col(acts[-1], st)
            cols.append(col)
            z = col @ Ws[l].T + bs[l]
            acts.append(np.tanh(z).reshape(a.shape[0], Ho, Wo, co))
        pooled = acts[-1].mean(axis=(1, 2))
        out = pooled @ Ws[-1].T + bs[-1]
        return acts, cols, pooled, out

    def loss(self, blocks, X, Y):
        out = self.forward(blocks, X)[3]
        d = out - np.asarray(Y, dtype=np.float64).reshape(out.shape)
        return float(0.5 * (d * d).sum(axis=1).mean())

    def partial_gradient(self, blocks, X, Y, suffix):
        """Batch-mean gradient of the top `suffix` layers (partial_backprop,
        spb.cpp:51-68, for this model); blocks below are None."""
        Ws, _ = self.unpack(blocks)
        acts, cols, pooled, out = self.forward(blocks, X)
        B = out.shape[0]
        d = out - np.asarray(Y, dtype=np.float64).reshape(out.shape)
        L, stop = self.L, self.L - suffix + 1
        g = [None] * L
        g[L - 1] = np.concatenate([(d.T @ pooled / B).ravel(), d.sum(0) / B])
        if stop > L - 1:
            return g
        hl = acts[-1]
        P = hl.shape[1] * hl.shape[2]
        delta = (d @ Ws[-1])[:, None, None, :] / P * (1 - hl * hl)
        for l in range(L - 1, stop - 1, -1):  # conv layer l (1-based) -> index l-1
            co = self.convs[l - 1][0]
            D = delta.reshape(-1, co)
            g[l - 1] = np.concatenate([(D.T @ cols[l - 1] / B).ravel(), D.sum(0) / B])
            if l > stop:
                dcols = D @ Ws[l - 1]
                below = acts[l - 1]
                delta = col2im(dcols, below.shape, self.convs[l - 1][1]) * (1 - below * below)
        return g

    def spb_step(self, blocks, X, Y, k, bw, lr, seed, s, orc, full=False):
        """One SPB-SGD iteration (spb.cpp:183-196 for this model), in place."""
        L, N = self.L, len(X)
        grads = []
        for j in range(1, k + 1):
            batch = orc.draw_batch(seed, s, j, bw, N)
            suf = L if full else orc.suffix_layers(j, k, L)
            grads.append(self.partial_gradient(blocks, X[batch], Y[batch], suf))
        for l in range(L):
            contrib = [gr[l] for gr in grads if gr[l] is not None]
            blocks[l] = blocks[l] - lr * (sum(contrib) / len(contrib))
        return blocks
