"""First GPU shakeout: coefficient table + cfg0/cfg1 march vs goldens."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import oracle as O
from paper_2111_05205_b200 import elemint, marching, scenarios

g = np.load('tests/golden/coeff_table.npz')
P,A,B,Cc,s,ez,nx = g['P'],g['A'],g['B'],g['C'],g['s'],g['ez'],g['nx']
L = np.max([np.linalg.norm(P-A,axis=1),np.linalg.norm(P-B,axis=1),np.linalg.norm(P-Cc,axis=1)],axis=0)
for d in (1,2,3):
    K = 1/(4*np.pi*0.05**d)
    U,W = elemint.retarded_coeff_table(P,A,B,Cc,ez,s,d,1.0,0.05)
    BU,BW = elemint.retarded_coeff_table(P,A,B,Cc,ez,s,d,1.0,0.05,'bm',nx)
    for name,a,b,p in (('U',U,g[f'U{d}'],d+1),('W',W,g[f'W{d}'],d),('BU',BU,g[f'BU{d}'],d),('BW',BW,g[f'BW{d}'],d-1)):
        ts = K*(s+L)**p*2*np.pi
        e = np.abs(a-b)/np.maximum(np.maximum(ts,np.abs(b)),1e-300)
        print('coeff', d, name, 'max err %.2e' % e.max(), flush=True)

for cfg in (0, 1):
    spec = scenarios.build_spec(cfg)
    gold = np.load(f'tests/golden/march_cfg{cfg}.npz')
    t0 = time.time()
    st = marching.BandStore(spec).assemble()
    t1 = time.time()
    print('cfg', cfg, 'assemble', t1 - t0, st.info(), flush=True)
    trace = []
    t0 = time.time()
    h = marching.march(spec, mats=st, rhs_trace=trace)
    print('cfg', cfg, 'march s', time.time() - t0, h.status, h.n_steps, flush=True)
    x = h.u if spec.phi[0] == 1.0 else h.q
    sub = gold['sub']
    ref = gold['unknown_sub']
    per = [np.linalg.norm(x[b, sub] - ref[b]) / max(np.linalg.norm(ref[b]), 1e-300) for b in range(len(ref))]
    print('cfg', cfg, 'worst step rel (sub)', max(per), 'whole', np.linalg.norm(x[:, sub] - ref) / np.linalg.norm(ref))
    fs = gold['full_steps']
    print('cfg', cfg, 'full steps rel', [float(np.linalg.norm(x[b] - gold['unknown_full'][k]) / np.linalg.norm(gold['unknown_full'][k])) for k, b in enumerate(fs)])
    r = np.array(trace)
    print('cfg', cfg, 'rhs rel', np.linalg.norm(r[:, sub] - gold['rhs_sub']) / np.linalg.norm(gold['rhs_sub']))
    # timing resident
    st.upload_known(*marching.greville_samples(spec))
    tm = st.run_resident(1e6, n_repeat=3, time_kernels=True)
    print('cfg', cfg, 'resident', tm, 'steps/s', tm['steps'] / tm['total_ms'] * 1e3, flush=True)
