"""Dev probe (build with -DQSG_CL_TIMING): where a cluster-resident Kerr-50 attempt spends its time
(CTA 0 thread 0 globaltimer deltas per phase)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_21440_b200 as q
os.environ["QSG_CLUSTER_SOLVE"] = "1"
ctx = q.Context(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 50
m = q.Model("kerr", N, 1.0, 0.01, 2.0, 1.0)
g = q.Generator([ctx.op(m.export(q.SEL_L_CONST))])
eops = [m.export(q.SEL_E_OP, k) for k in range(m.n_eops)]
psi = m.psi0()
rho0 = np.outer(psi, psi.conj()).reshape(-1, order="F").copy()
tl = np.linspace(0.0, 10.0, 101)
L = q.lib()
L.qsg_debug_cluster_ns.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 16)()
q.mesolve(ctx, g, m.dim, rho0, tl, eops)
L.qsg_debug_cluster_ns(buf, 1)
r = q.mesolve(ctx, g, m.dim, rho0, tl, eops)
L.qsg_debug_cluster_ns(buf, 1)
att = r["attempts"]
names = ["begin+sync", "stage SpMV+epilogue", "observe (saves)", "block_sum+cl_sync", "obs commit", "finish_attempt", "flush", "observe items", "observe reduce"]
CLK_GHZ = float(os.environ.get("CLK_GHZ", "1.965"))  # cl_now() counts SM cycles
print("N", N, "attempts", att, "kernel_ms", r["kernel_ms"], "us/attempt", r["kernel_ms"] * 1e3 / att)
for i, nm in enumerate(names):
    print(f"{nm:24s} {buf[i] / att / CLK_GHZ / 1e3:8.3f} us/attempt")
