import os, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2006_03031_b200 import nimble as nb, synth
from paper_2006_03031_b200.rnn import LSTMStack
I = H = 650
st = LSTMStack(synth.lstm_weights(I, H, 2, seed=0), max_T=512)

def graph_time(fn, reps=20):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3 / reps)
    return sorted(ts)[2]

for T in (1, 8, 35, 128, 512):
    x = torch.zeros((T, st.Ip), dtype=torch.float32, device="cuda"); x[:, :I] = synth.lstm_input(T, I, seed=1).cuda()
    tg = graph_time(lambda: st.forward(x, T))
    tu = graph_time(lambda: st.forward(x, T, fused=False))
    (Wi1, Wh1, b1, _), (Wi2, Wh2, b2, _) = st.layers
    tgemm = graph_time(lambda: nb.dense_dyn(x, Wi1, b1, st.G, epi=nb.EPI_BIAS, M=T))
    print(json.dumps({"T": T, "graph_us_per_seq": tg, "us_per_token": tg / T, "input_gemm_us": tgemm, "unfused_us_per_seq": tu}), flush=True)
