#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/cmlab.py > gpurun_out/cmlab3.jsonl 2> gpurun_out/cmlab3.err
