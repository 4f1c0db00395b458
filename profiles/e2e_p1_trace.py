import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2601_17561_b200.ccmm import CcmmEngine, synth_query
N, M, K = 992, 1 << 14, 24576
eng = CcmmEngine(parts=1, m=M, k=K, max_n=N)
eng.synth_db(1)
q = torch.from_numpy(synth_query(2, K, N, eng.moduli).view(np.int16)).pin_memory().numpy().view(np.uint16)
out = torch.empty((1, eng.nmod, N, M), dtype=torch.int16).pin_memory().numpy().view(np.uint16)
eng.run(q, out)
os.environ["IRL_E2E_TRACE"] = "1"
eng.run(q, out)
