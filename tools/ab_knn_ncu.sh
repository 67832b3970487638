cd /root/repo
L=paper_2604_16402_b200/libgrab.so
cp $L ab/lib_orig.so
for v in ${VARS:-A B C}; do cp ab/lib$v.so $L; echo "== $v"; timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --profile-from-start off -k regex:k_knn_screen_tc -c 1 python tools/profile_build.py cfg2 2>&1 | grep -E "duration|inst_executed|tensor"; done
cp ab/lib_orig.so $L
