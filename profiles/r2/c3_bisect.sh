SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_v1.so python profiles/r2/c3_diff.py /tmp/h_v1.npy 1024 3000
python profiles/r2/c3_diff.py /tmp/h_new.npy 1024 3000
python - <<'PY'
import numpy as np
a=np.load('/tmp/h_v1.npy'); b=np.load('/tmp/h_new.npy')
print('v1 lens', [len(x) for x in a], 'new lens', [len(x) for x in b])
for rep in range(3):
    n=min(a.shape[1],b.shape[1]); d=np.nonzero(a[0][:n]!=b[rep][:n])[0]
    print('new rep',rep,'first mismatch', (d[0] if d.size else None), 'count', d.size, 'rel', (abs(a[0][d[0]]-b[rep][d[0]])/a[0][d[0]] if d.size else 0))
PY
