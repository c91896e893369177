# Bit-identity test of the three rounding forms + the conversion-rate micro-benchmark.
python -m paper_2305_19028_b200.build --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -q tests/test_gpu_stress.py -k "rounding_forms or gram" > gpurun_out/r02h_round_test.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r02h_round_test.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cvt_rate tools/micro/cvt_rate.cu && /tmp/cvt_rate > gpurun_out/r02h_cvt_rate.log 2>&1; cat gpurun_out/r02h_cvt_rate.log
