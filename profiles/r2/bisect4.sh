for v in dnopref v1; do
  export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_$v.so
  echo "== variant $v"
  python profiles/r2/c3_diff.py /tmp/h_$v.npy 1024 3000
done
