import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
from esi_synth import make_workload, to_numpy_struct
from helpers import gpu_run, oracle_run
w = make_workload(sys.argv[1] if len(sys.argv) > 1 else 'c2', 'cpu')
ev = to_numpy_struct(w.events)
f_ref, S_ref, T_ref = oracle_run(w.W, w.H, ev, w.t_frames, w.params)
for mode in [{}, {'ESI_RANK_MODE': 'ballot'}, {'ESI_DISABLE_FAST': '1'}, {'ESI_DISABLE_FAST': '1', 'ESI_RANK_MODE': 'ballot'}]:
    for k in ('ESI_RANK_MODE', 'ESI_DISABLE_FAST'):
        os.environ.pop(k, None)
    os.environ.update(mode)
    f, S, T, st = gpu_run(w.W, w.H, w.events, w.t_frames, w.params)
    d = f.astype(int) - f_ref
    bad_f = np.nonzero((d != 0).reshape(len(f), -1).mean(1) > 1e-3)[0]
    print(mode, 'flip frac', (d != 0).mean(), 'Tmismatch', (T != T_ref).mean(), 'maxdS', np.abs(S - S_ref).max(),
          'first bad frames', bad_f[:5], st)
    if len(bad_f):
        j = bad_f[0]; yy, xx = np.nonzero(d[j]); print('  frame', j, 'n bad', len(yy), 'px', list(zip(yy[:5], xx[:5])), 'gpu', f[j, yy[:5], xx[:5]], 'ref', f_ref[j, yy[:5], xx[:5]])
