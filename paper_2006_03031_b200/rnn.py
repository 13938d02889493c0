"""LSTM language-model layers and Tree-LSTM forests composed from libnimble ops.

LSTM (config 2): per layer one hoisted input GEMM
G = X W_ih^T + b over all T steps (nimble_dense_dyn, fp32 SIMT8, M = T — the
"dynamically batched" input matmul the paper calls orthogonal) and one
persistent recurrent kernel (nimble_lstm_seq) that loops over the runtime T on
the device.  Feature dims are padded to a multiple of 4 with zero columns for the
fp32 vector loads; the padding contributes exact zeros.

Tree-LSTM (config 4): the recursion over the tree ADT
becomes a schedule of levels (node height), built once on the host and kept on the
device; the whole forest is one nimble_treelstm_forest launch that loops over the
levels on the device (or, fused=False, one nimble_treelstm_level launch per level).
Each level's epilogue writes (h, c) straight into the parent's input row.
"""
from __future__ import annotations

import numpy as np
import torch

from . import nimble as nb


def _pad4(n: int) -> int:
    return 4 * ((n + 3) // 4)


class LSTMStack:
    def __init__(self, layers, max_T: int, device="cuda"):
        """layers: [(W_ih [4H x I], W_hh [4H x H], b [4H])] fp32 (PyTorch gate order i, f, g, o)."""
        self.H = layers[0][1].shape[1]
        H = self.H
        self.I = layers[0][0].shape[1]
        self.Ip, self.Hp = _pad4(self.I), _pad4(H)
        self.max_T = max_T
        self.layers = []
        for li, (W_ih, W_hh, b) in enumerate(layers):
            inp = W_ih.shape[1]
            Kp = _pad4(inp)
            Wi = torch.zeros((4 * H, Kp), dtype=torch.float32, device=device)
            Wi[:, :inp] = W_ih.to(device)
            self.layers.append((Wi, W_hh.to(device).contiguous(), b.to(device).contiguous(), Kp))
        self.G = torch.empty((max_T, 4 * H), dtype=torch.float32, device=device)
        self.Hs = [torch.zeros((max_T, self.Hp), dtype=torch.float32, device=device) for _ in layers]
        self.hT = torch.empty((len(layers), H), dtype=torch.float32, device=device)
        self.cT = torch.empty((len(layers), H), dtype=torch.float32, device=device)
        self.ws = torch.empty((nb.lstm_workspace_bytes(H),), dtype=torch.uint8, device=device)
        # zeroed once: the wavefront kernel leaves its tagged buffers zeroed after every call
        self.ws2 = torch.zeros((nb.lstm2_workspace_bytes(H),), dtype=torch.uint8, device=device)
        # the wavefront kernel takes W_hh1, W_ih2, W_hh2 with one leading dimension (H)
        self.Wi2u = layers[1][0].to(device).contiguous() if len(layers) == 2 and layers[1][0].shape[1] == H else None
        self.fused_ok = True

    def flops_per_token(self) -> int:
        return sum(2 * 4 * self.H * (Kp + self.H) for (_, _, _, Kp) in self.layers)

    def forward(self, x: torch.Tensor, T: int | None = None, wavefront: bool = True, fused: bool = True) -> torch.Tensor:
        """x [>=T x Ip] fp32 (zero columns beyond I); returns the last layer's h sequence [T x H].
        Two layers run as one wavefront kernel unless wavefront=False: with fused=True the layer-1
        input projection runs inside it (nimble_lstm2_forward, one launch), else as a hoisted
        input GEMM (nimble_dense_dyn + nimble_lstm2_seq)."""
        T = x.shape[0] if T is None else T
        if wavefront and self.Wi2u is not None:
            (Wi1, Wh1, b1, _), (Wi2, Wh2, b2, _) = self.layers
            # the one-launch form pays a per-step W_ih1 mat-vec from shared memory: it wins only
            # where the hoisted input GEMM launch dominates (measured: T = 1 14.7 vs 19.4 us,
            # T = 8 49.7 vs 47.2 us)
            if fused and self.fused_ok and T <= 4:
                try:
                    nb.lstm2_forward(x, self.I, Wi1, b1, Wh1, self.Wi2u, Wh2, b2, self.Hs[0], self.Hs[1], self.hT,
                                     self.cT, self.ws2, T=T)
                    return self.Hs[1][:T, :self.H]
                except nb.NimbleError as e:
                    if e.status != -7:                              # E_UNSUPPORTED
                        raise
                    self.fused_ok = False                                   # shape not built fused
            nb.dense_dyn(x, Wi1, b1, self.G, epi=nb.EPI_BIAS, M=T)           # hoisted input GEMM (M = T)
            nb.lstm2_seq(self.G, Wh1, self.Wi2u, Wh2, b2, self.Hs[0], self.Hs[1], self.hT, self.cT, self.ws2, T=T)
            return self.Hs[1][:T, :self.H]
        inp = x
        for li, (Wi, Wh, b, Kp) in enumerate(self.layers):
            nb.dense_dyn(inp, Wi, b, self.G, epi=nb.EPI_BIAS, M=T)        # hoisted input GEMM (M = T)
            nb.lstm_seq(self.G, Wh, self.Hs[li], self.hT[li], self.cT[li], self.ws, T=T)
            inp = self.Hs[li]
        return self.Hs[-1][:T, :self.H]


class TreeSchedule:
    """Level schedule of a forest: node height, per-level node / input-row / parent-slot arrays."""

    def __init__(self, trees, device="cuda"):
        left, right, word, roots = [], [], [], []
        for (root, l, r, w) in trees:
            off = len(left)
            left += [c + off if c >= 0 else -1 for c in l]
            right += [c + off if c >= 0 else -1 for c in r]
            word += list(w)
            roots.append(root + off)
        n = len(left)
        height = [0] * n
        parent_slot = [-1] * n
        for i in range(n):                      # children precede parents (post-order ids)
            if left[i] >= 0:
                height[i] = 1 + max(height[left[i]], height[right[i]])
                parent_slot[left[i]] = 2 * i
                parent_slot[right[i]] = 2 * i + 1
        self.n_nodes, self.roots = n, roots
        self.left, self.right, self.word = left, right, word
        self.levels = []
        for h in range(max(height) + 1):
            ids = [i for i in range(n) if height[i] == h]
            rows = [word[i] if h == 0 else i for i in ids]
            to = lambda a: torch.tensor(a, dtype=torch.int32, device=device)
            self.levels.append((to(ids), to(rows), to([parent_slot[i] for i in ids]), len(ids)))
        self.n_leaves = sum(1 for i in range(n) if left[i] < 0)
        # the same schedule as flat device arrays for the one-launch forest kernel
        cat = lambda k: torch.cat([lv[k] for lv in self.levels])
        self.nodes_all, self.rows_all, self.pslot_all = cat(0), cat(1), cat(2)
        self.level_off = torch.tensor(np.concatenate([[0], np.cumsum([lv[3] for lv in self.levels])]),
                                      dtype=torch.int32, device=device)
        self.max_level = max(lv[3] for lv in self.levels)


class TreeLSTM:
    def __init__(self, W_l, b_l, U, b_u, device="cuda"):
        self.H = U.shape[1] // 2
        self.I = W_l.shape[1]
        assert self.I % 4 == 0 and (2 * self.H) % 4 == 0
        self.W_l, self.b_l = W_l.to(device).contiguous(), b_l.to(device).contiguous()
        self.U, self.b_u = U.to(device).contiguous(), b_u.to(device).contiguous()
        self.ws = torch.zeros((nb.TREE_WORKSPACE_BYTES,), dtype=torch.uint8, device=device)

    def flops(self, sched: TreeSchedule) -> int:
        n_int = sched.n_nodes - sched.n_leaves
        return sched.n_leaves * 2 * 3 * self.H * self.I + n_int * 2 * 5 * self.H * 2 * self.H

    def forward(self, X: torch.Tensor, sched: TreeSchedule, fused: bool = True):
        """X [n_words x I] fp32 on device; returns (h [n_nodes x H], c [n_nodes x H]).
        fused: the whole forest in one nimble_treelstm_forest launch; else one
        nimble_treelstm_level launch per level."""
        H, n = self.H, sched.n_nodes
        dev = X.device
        hcat = torch.empty((n, 2 * H), dtype=torch.float32, device=dev)     # every internal row is written
        ccat = torch.empty((n, 2 * H), dtype=torch.float32, device=dev)     # by its two children first
        h = torch.empty((n, H), dtype=torch.float32, device=dev)
        c = torch.empty((n, H), dtype=torch.float32, device=dev)
        if fused:
            nb.treelstm_forest(X, self.W_l, self.b_l, self.U, self.b_u, sched.level_off, len(sched.levels),
                               sched.max_level, sched.nodes_all, sched.rows_all, sched.pslot_all, hcat, ccat, h, c,
                               self.ws)
            return h, c
        for lvl, (ids, rows, pslot, M) in enumerate(sched.levels):
            if lvl == 0:
                nb.treelstm_level(ids, X, rows, self.W_l, self.b_l, pslot, hcat, ccat, h, c, M, self.I, H, 1)
            else:
                nb.treelstm_level(ids, hcat, rows, self.U, self.b_u, pslot, hcat, ccat, h, c, M, 2 * H, H, 0)
        return h, c
