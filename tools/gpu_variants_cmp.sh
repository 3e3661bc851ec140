# time + compare the outputs of every variant with the default build (config 2, 64 edges)
set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
PMX_SAVE=/tmp/out_default.npz python tools/time_match.py 64 2>&1 | tail -1
for d in build/variants/*/; do
  n=$(basename $d)
  PMX_SAVE=/tmp/out_$n.npz PMX_LIB=$d/libpmx_cuda.so python tools/time_match.py 64 2>&1 | tail -1
  python -c "
import numpy as np
a=np.load('/tmp/out_default.npz'); b=np.load('/tmp/out_$n.npz')
both=(a['valid']==1)&(b['valid']==1); d=(a['pa']!=b['pa'])&both
W=512; du=np.abs(a['pa'][d]%W-b['pa'][d]%W); dv=np.abs(a['pa'][d]//W-b['pa'][d]//W)
qd = (a['q'] != b['q']) & both & (a['pa'] == b['pa']) if 'q' in a and 'q' in b else np.zeros(1, bool)
print('$n vs default: valid mismatch', int((a['valid']!=b['valid']).sum()), 'index mismatch', int(d.sum()), 'of', int(both.sum()), 'worst px', int(max(du.max(initial=0), dv.max(initial=0))), 'q differing', int(qd.sum()))"
done
