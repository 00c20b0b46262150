export SK_LIB_PATH=paper_2605_28274_b200/libsk_b200_dslot0.so
python profiles/r2/c3_diff.py /tmp/h_s0.npy 1024 3000 2>&1 | tail -1
python profiles/r2/c3_diff.py /tmp/h2_s0.npy 1024 3000 2>&1 | tail -1
