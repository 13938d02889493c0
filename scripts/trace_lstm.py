import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_03031_b200 import nimble as nb, synth
from paper_2006_03031_b200.rnn import LSTMStack
I = H = 650; T = 64
st = LSTMStack(synth.lstm_weights(I, H, 2, seed=0), max_T=T)
x = torch.zeros((T, st.Ip), dtype=torch.float32, device="cuda"); x[:, :I] = synth.lstm_input(T, I, seed=1).cuda()
st.forward(x, T); torch.cuda.synchronize()
buf = torch.zeros(2 * (T + 1) * 4, dtype=torch.int64, device="cuda")
nb._lib.nimble_debug_trace(buf.data_ptr()); st.forward(x, T); torch.cuda.synchronize(); nb._lib.nimble_debug_trace(None)
t = buf.cpu().numpy().reshape(2, T + 1, 4).astype(np.float64)
for c, name in ((0, "layer1 CTA0"), (1, "layer2 CTA0")):
    r = t[c]
    step = np.diff(r[:, 0])
    print(name, "step us median %.2f" % (np.median(step) / 1e3),
          "| gather %.2f compute %.2f gates+sync %.2f" % tuple(np.median(r[1:, k + 1] - r[1:, k]) / 1e3 for k in range(3)))
