# A/B: the rounding pass staged by the bulk-copy engine (TLS_ROUND=3) against the register form (default).
python -m paper_2305_19028_b200.build --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
L=gpurun_out/r02h_round_bulk.log
timeout 300 python tools/time_gram_nreg.py round2 > $L 2>&1; echo default rc=$?
for g in 1 3 4; do
  TLS_ROUND=3 TLS_ROUND_GRID=$g timeout 300 python tools/time_gram_nreg.py bulk_grid$g >> $L 2>&1; echo bulk$g rc=$?
done
TLS_ROUND=3 TLS_GRAM_SEGS=1 timeout 300 python tools/time_gram_nreg.py bulk_segs1 >> $L 2>&1
TLS_GRAM_SEGS=1 timeout 300 python tools/time_gram_nreg.py round2_segs1 >> $L 2>&1
cat $L
