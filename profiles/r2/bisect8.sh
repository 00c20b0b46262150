for v in f4f f1f; do
export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so
echo "== $v"
python profiles/r2/c3_diff.py /tmp/h_$v.npy 1024 3000 2>&1 | tail -1
python profiles/r2/c3_diff.py /tmp/h2_$v.npy 1024 3000 2>&1 | tail -1
done
