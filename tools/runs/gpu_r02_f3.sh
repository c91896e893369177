#!/bin/bash
TLS_FZ_PROF=1 python tools/time_gram_fused2.py --one 1048576 1024 fp16 x 0 2>&1 | tail -3
TLS_FZ_PROF=1 TLS_GRAM_NSPLIT=3 python tools/time_gram_fused2.py --one 1048576 1024 fp16 x 0 2>&1 | tail -2
