#!/bin/bash
mkdir -p gpurun_out
STS_B200_LIB=$PWD/paper_2605_15508_b200/_lib/variants/libsts_b200_trace.so timeout 300 python tools/trace_decode.py 32768 > gpurun_out/trace_32k.json 2>&1
