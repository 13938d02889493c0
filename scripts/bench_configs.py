"""Latency measurements for BASELINE configs 2, 3, 4 (BJ:8-10) on one B200.

config 2: 2-layer LSTM LM, I = H = 650, batch 1, T in {35, 128, 512}: us/token (hoisted input
          GEMM via dense_dyn + persistent recurrence, all on one stream, CUDA events).
config 3: BERT-base, batch 1, every L in 1..128: per-request latency (per-L CUDA graph of the
          12-layer batch-1 path, or one device-extent graph for every L) -> us/token; plus the
          packed equivalent.
config 4: Tree-LSTM (300/150) forests of 1 and 32 random trees: us/tree, us/leaf.
Paper context (other hardware): LSTM 2L Nimble T4 107.4 us/token (300/512); BERT-base
Nimble T4 95.2 us/token; Tree-LSTM Nimble Intel 40.3 us/token.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb, synth  # noqa: E402
from paper_2006_03031_b200.bert import BertEncoder, BertPacked  # noqa: E402
from paper_2006_03031_b200.rnn import LSTMStack, TreeLSTM, TreeSchedule  # noqa: E402
from paper_2006_03031_b200.serve import DeviceExtentGraph, GraphCache  # noqa: E402


SCHEDULES = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2006_03031_b200",
                         "tuned", "bert_dense_schedules.json")


def ev_time(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def graph_time(fn, reps=20, iters=5):
    """Device time per call: a CUDA graph of `reps` calls, median of `iters` replays."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3 / reps)
    return sorted(ts)[len(ts) // 2]


def main():
    only = set(sys.argv[1].split(",")) if len(sys.argv) > 1 else {"2", "3", "4"}
    rep = {}
    if "2" in only:
        config2(rep)
    if "3" in only:
        config3(rep)
    if "4" in only:
        config4(rep)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/configs_report.json", "w") as f:
        json.dump(rep, f, indent=1)


def config2(rep):
    I = H = 650
    st = LSTMStack(synth.lstm_weights(I, H, 2, seed=0), max_T=512)
    c2 = []
    for T in (1, 8, 35, 128, 512):
        x = torch.zeros((T, st.Ip), dtype=torch.float32, device="cuda")
        x[:, :I] = synth.lstm_input(T, I, seed=1).cuda()
        t = ev_time(lambda: st.forward(x, T))                  # eager: host launch path included
        tg = graph_time(lambda: st.forward(x, T))              # device time (CUDA-graph replays)
        c2.append({"T": T, "us_per_seq": tg * 1e6, "us_per_token": tg * 1e6 / T,
                   "us_per_seq_eager": t * 1e6, "gflops": st.flops_per_token() * T / tg / 1e9})
        print(json.dumps(c2[-1]), flush=True)
    rep["config2_lstm_650x2"] = c2


def config3(rep):
    # batch-1 graphs, every L in 1..128; default dispatch rule, then the tuned schedules
    cfg = dict(synth.BERT_BASE)
    w = synth.bert_weights_device(cfg, seed=0)
    out = torch.empty((cfg["d"],), dtype=torch.bfloat16, device="cuda")
    # "": per-L graphs, default rule; "_devextent": ONE graph for every L, extent and residue
    # dispatch on the device (f4); "_tuned": per-L graphs with the tuned schedules (f3)
    for tag in ("", "_devextent", "_tuned"):
        if tag == "_tuned":
            nb.load_dense_schedules(SCHEDULES)
        enc = BertPacked(cfg, w, max_tokens=128)          # batch 1 = packed batch of one request
        cache = DeviceExtentGraph(enc) if tag == "_devextent" else GraphCache(enc)
        c3 = []
        for L in range(1, 129):
            cache.capture(L)
            x = synth.device_normal(L, cfg["d"], seed=L)
            t = ev_time(lambda: cache.run(x, L, out), reps=5, warm=2)
            fl = BertPacked.flops([L], cfg["d"], cfg["ffn"], cfg["layers"])
            c3.append({"L": L, "us": t * 1e6, "us_per_token": t * 1e6 / L, "tflops": fl / t / 1e12})
        rep["config3_bert_base_batch1" + tag] = c3
        print(tag, json.dumps({k: c3[i] for k, i in (("L1", 0), ("L64", 63), ("L128", 127))}), flush=True)
        del cache, enc
    for op in json.load(open(SCHEDULES))["schedules"]:
        nb.set_dense_schedule(op["N"], op["K"], 0, 8)
    # packed BERT-base: 64 requests with L ~ U{1..128}
    lens = synth.request_lengths(64, seed=2, hi=128)
    Tt = int(lens.sum())
    pk = BertPacked(cfg, w, max_tokens=Tt)
    off = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    X = synth.device_normal(Tt, cfg["d"], seed=3)
    t = ev_time(lambda: pk.forward(X, off, int(lens.max())))
    rep["config3_bert_base_packed64"] = {"requests": 64, "tokens": Tt, "ms": t * 1e3, "req_per_s": 64 / t,
                                        "us_per_token": t * 1e6 / Tt,
                                        "tflops": BertPacked.flops(lens, cfg["d"], cfg["ffn"], cfg["layers"]) / t / 1e12}
    print(json.dumps(rep["config3_bert_base_packed64"]), flush=True)


def config4(rep):
    I, Hh = 300, 150
    W_l, b_l, U, b_u = synth.tree_weights(I, Hh)
    model = TreeLSTM(W_l, b_l, U, b_u)
    c4 = []
    for n in (1, 32, 256):
        trees, nw = synth.random_forest(n, seed=2)
        sched = TreeSchedule(trees)
        X = synth.normal((nw, I), 1.0, 4, torch.float32).cuda()
        t = ev_time(lambda: model.forward(X, sched))
        t_lv = ev_time(lambda: model.forward(X, sched, fused=False))
        c4.append({"trees": n, "leaves": sched.n_leaves, "levels": len(sched.levels), "us_per_forest": t * 1e6,
                   "us_per_tree": t * 1e6 / n, "us_per_leaf": t * 1e6 / sched.n_leaves,
                   "gflops": model.flops(sched) / t / 1e9, "per_level_launches_us_per_forest": t_lv * 1e6})
        print(json.dumps(c4[-1]), flush=True)
    rep["config4_treelstm_300_150"] = c4


if __name__ == "__main__":
    main()
