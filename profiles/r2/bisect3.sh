for v in dnopref v1; do
  export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so
  echo "== variant $v"
  python profiles/r2/c3_diff.py /tmp/h_$v.npy 1024 3000
  python profiles/r2/c3_diff.py /tmp/h2_$v.npy 1024 3000
done
python - <<'PY'
import numpy as np
a=np.load('/tmp/h_v1.npy')
for name in ('h2_v1','h_dnopref','h2_dnopref'):
    b=np.load(f'/tmp/{name}.npy')
    for rep in range(3):
        n=min(a.shape[1],b.shape[1]); d=np.nonzero(a[0][:n]!=b[rep][:n])[0]
        print(name,'rep',rep,'len',len(b[rep]),'first mismatch', (d[0] if d.size else None))
PY
