import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/oracle"); sys.path.insert(0, ROOT + "/tests")
import paper_2212_11296_b200 as P
from oracle import PortLib
from test_gpu_parity import setup
port = PortLib()
w, eng, om, oh, S = setup(port, "c1", 256)
led = P.Ledger()
e, lpsi = eng.local_energies(S, led)
print("prof after host call", eng.last_profile())
K, U, codes, lps = eng.taps(S)
t = om.taps(oh, S[0])
print("gpu", lps[0][:5], "\nref", t.lp[:5])
d_cfg = torch.from_numpy(S).cuda(); d_e = torch.empty(256, dtype=torch.float64, device="cuda"); d_l = torch.empty_like(d_e)
led2 = eng.local_energies_device(d_cfg, d_e, d_l, torch.cuda.current_stream())
print("prof after device call", eng.last_profile(), led2)
print(np.abs(d_e.cpu().numpy() - e.real).max())
