# A/B: k_gram_tc2 with its registers capped (more rounding-pass CTAs co-resident) against the default build.
python -m paper_2305_19028_b200.build --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python tools/time_gram_nreg.py default > gpurun_out/r02h_gram_nreg.log 2>&1; echo default rc=$?
for R in 128 104; do
  TLS_EXTRA_NVCC=-DTLS_T2_MAXNREG=$R python -m paper_2305_19028_b200.build --force >> gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
  timeout 300 python tools/time_gram_nreg.py maxnreg$R >> gpurun_out/r02h_gram_nreg.log 2>&1; echo nreg$R rc=$?
done
cat gpurun_out/r02h_gram_nreg.log
