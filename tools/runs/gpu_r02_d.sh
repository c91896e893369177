python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for J in 0 1; do timeout 300 python tools/qr_dump_cmp.py 1100 530 fp16 $J; done > gpurun_out/qr_dump.log 2>&1
timeout 300 python tools/qr_dump_cmp.py 1100 400 fp16 0 >> gpurun_out/qr_dump.log 2>&1
TLS_QR_COOP=1 timeout 300 python tools/qr_dump_cmp.py 600 300 fp16 0 >> gpurun_out/qr_dump.log 2>&1
cat gpurun_out/qr_dump.log
