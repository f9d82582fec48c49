import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4019_b200 as pf
from paper_1301_4019_b200 import _lib as L
from oracle import pfr_oracle as orc
for n in (1 << 16, 1 << 20):
    g = np.random.default_rng(1); lw = g.normal(0, 1, n)
    w64 = np.exp(lw - lw.max())
    w = torch.from_numpy(w64).cuda()
    rs = pf.RngStream(3)
    u = float(L.lib().pfr_stream_uniform(L.PfrRng(*rs.key(), L.RNG_PHILOX, 0), 0, 0x5359))
    c = torch.empty(n, dtype=torch.int32, device="cuda"); Oo = torch.empty(n, dtype=torch.int32, device="cuda")
    st = L.new_status(); ws, wsb = L.workspace(n)
    r = L.PfrRng(*rs.key(), L.RNG_PHILOX, 0)
    L.call("pfr_deliver_offspring", w.data_ptr(), n, L.F64, 0, 0, u, None, r, c.data_ptr(), Oo.data_ptr(), None, st.data_ptr(), ws, wsb, L.stream_handle())
    torch.cuda.synchronize()
    flags = L._ws[0][:8].view(torch.int32).cpu().numpy()
    O = Oo.cpu().numpy().astype(np.int64)
    ref = orc.systematic(w64, u)
    bad = np.flatnonzero(np.diff(O) < 0)
    mm = np.flatnonzero(O != ref)
    print(n, "flags", flags, "u", u, "decreases at", bad[:10], "mismatch vs ref at", mm[:10], O[mm[:5]], ref[mm[:5]])
    if bad.size:
        i = bad[0]; print("  O around", O[i-3:i+4], "ref", ref[i-3:i+4])
