"""Time each op of bench.py's step twice: inside the step (events between ops,
as bench.py does) and in isolation with an L2 flush before it (development
tool, to find context effects)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import gen  # noqa: E402
import paper_2008_11359_b200 as fgp  # noqa: E402

g = gen.make_graph(bench.GRAPH)
host = bench.make_inputs(g)
st = torch.cuda.Stream()
S = bench.Step(g, None, host, None, st)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
names = ["allgather", "copy_u_sum_F512", "sddmm_H1_F512", "sddmm_H8", "softmax_H8", "u_mul_e_H8", "copy_u_max_F128",
         "mlp"]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
res = []
with torch.cuda.stream(st):
    for k in range(4):
        flush.fill_(float(k))
        S.enqueue(ev)
        st.synchronize()
        if k:
            res.append([ev[i].elapsed_time(ev[i + 1]) for i in range(8)])
in_step = np.median(np.array(res), axis=0)
G, X = S.G, S.X


def iso(fn, reps=4):
    ts = []
    with torch.cuda.stream(st):
        for i in range(reps + 1):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); fn(); b.record(st); st.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
    return float(np.median(ts))


ops = {
    "copy_u_sum_F512": lambda: fgp.spmm(G, "copy_u", "sum", X["X512"], out=S.out512, stream=st),
    "sddmm_H1_F512": lambda: fgp.sddmm(G, X["X512"], H=1, out=S.s1, stream=st),
    "sddmm_H8": lambda: fgp.sddmm(G, X["X256"], H=8, out=S.s8, stream=st),
    "u_mul_e_H8": lambda: fgp.spmm(G, "u_mul_e", "sum", X["X256"], H=8, E=S.s8, out=S.o256, stream=st),
    "copy_u_max_F128": lambda: fgp.spmm(G, "copy_u", "max", X["X128"], out=S.o128, arg_u=S.au128, arg_e=S.ae128,
                                        stream=st),
}
for i, n in enumerate(names):
    extra = f"   isolated {iso(ops[n]):8.3f}" if n in ops else ""
    print(f"{n:18s} in-step {in_step[i]:8.3f}{extra}")
Xr = torch.rand(g.n_dst, 256, device="cuda")
print(f"u_mul_e_H8 with torch.rand X: {iso(lambda: fgp.spmm(G, 'u_mul_e', 'sum', Xr, H=8, E=S.s8, out=S.o256, stream=st)):8.3f}")
Er = torch.rand(g.nnz, 8, device="cuda")
print(f"u_mul_e_H8 with torch.rand E: {iso(lambda: fgp.spmm(G, 'u_mul_e', 'sum', X['X256'], H=8, E=Er, out=S.o256, stream=st)):8.3f}")
