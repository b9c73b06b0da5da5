"""Conservation and rank invariance of one Central4 step on a 512 x 1024 noise field: single rank vs two loopback
virtual ranks (totals drift and bitwise owned states).  python scripts/drift_check.py (GPU box)."""
import threading, uuid, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2508_05020_b200 as amr, workloads as W
N=512; n=32
cfg = W.sweep(N=N, n=n, scheme="central4", Ny=2*N, seed=7); cfg["check_positivity"]=0
U0 = W.level0_state(cfg).reshape(-1,4,n,n)
def single():
    g = amr.Mesh(cfg); g.set_state(U=U0)
    t0,lam = g.diagnostics(); dt=0.3/lam; g.step(dt=dt); t1,_=g.diagnostics()
    st=g.get_state(as_dict=False); g.close(); return t0,t1,dt,st
t0,t1,dt,st = single()
print('single drift', np.max(np.abs(t1-t0))/np.max(np.abs(t0)), t0, t1)
key=uuid.uuid4().hex[:12]; out=[None]*2
def worker(r):
    torch.cuda.set_device(0)
    g = amr.Mesh(cfg, world_size=2, rank=r, comm_backend=1, comm_id=key)
    own = g.owned()
    g.set_state(U=U0[own], indices=own)
    a,_ = g.diagnostics(); g.step(dt=dt); b,_ = g.diagnostics()
    s = g.get_state(as_dict=False, indices=own)
    out[r]=(a,b,own,s); g.close()
th=[threading.Thread(target=worker,args=(r,)) for r in range(2)]
[t.start() for t in th]; [t.join() for t in th]
a,b,_,_ = out[0]
print('multi drift', np.max(np.abs(b-a))/np.max(np.abs(a)), a, b)
for r in range(2):
    own, s = out[r][2], out[r][3]
    print('rank', r, 'bitwise', np.array_equal(s, st[own]), np.nanmax(np.abs(s-st[own])))
