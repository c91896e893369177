#!/bin/bash
timeout 900 python tools/time_gram_fused2.py > gpurun_out/gram_fused2.log 2>&1; echo "rc=$?"; cat gpurun_out/gram_fused2.log
