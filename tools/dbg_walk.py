import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import __graft_entry__ as entry
entry.build()
import paper_2012_15198_b200 as cs
import synth
from oracle import topology as T
from gpu_util import OracleRun, device_state, grads_view
LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)
fails = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
  for V, n_loc, d, k in [(2, 8, 20_000, 16), (2, 3, 50_001, 5), (4, 4, 30_011, 8)]:
    n = V * n_loc
    cs.cs_init(n, n, k, 17)
    cs.cs_test_emulate_ranks(V)
    ld = (d + 3) // 4 * 4
    x, m, w, bank2 = device_state(cs, n, d, k, 17, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    orc = OracleRun(n, d, k, 17)
    b = T.segment_bounds(d, k)
    for t in range(5):
        src = T.topology(17, t, n, k)
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
        torch.cuda.synchronize()
        xg = x.cpu().numpy()[:, :d]
        if not np.array_equal(xg, orc.x) or not np.array_equal(w.cpu().numpy(), orc.w):
            fails += 1
            bad = np.argwhere(xg != orc.x)
            rows = sorted(set(bad[:, 0].tolist()))
            print(f"rep {rep} V={V} n_loc={n_loc} d={d} k={k} step {t}: {bad.shape[0]} bad x elems rows {rows[:10]}; w ok {np.array_equal(w.cpu().numpy(), orc.w)}", flush=True)
            for r in rows[:3]:
                cols = bad[bad[:, 0] == r][:, 1]
                segs = sorted(set(np.searchsorted(b, cols, side='right') - 1))
                for s_ in segs[:3]:
                    cc = cols[(cols >= b[s_]) & (cols < b[s_ + 1])]
                    srcr = src[s_][r]
                    print(f"   row {r} seg {s_} src {srcr} ({'remote' if srcr // n_loc != r // n_loc else 'local'}) cols {cc.min()}..{cc.max()} n={len(cc)} tile0 {(cc.min()-b[s_])//2048}", flush=True)
            break
    cs.cs_finalize()
print("fails", fails)
