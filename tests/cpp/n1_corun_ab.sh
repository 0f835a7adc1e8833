#!/bin/bash
# A/B of the N=1 pipelined schedule over (pair-GEMM ring, co-resident router ring).
for pass in 1 2 3; do
for cfg in "33 2" "32 8" "22 9" "32 4"; do
  set -- $cfg
  SCMOE_PAIR_STAGES=$1 SCMOE_CORUN_STAGES=$2 timeout 300 python bench.py --steps 20 --warmup 5 \
    --e5-steps 0 --full-layer 0 --config-a 0 --decode-tokens 0 --tpot-batch 0 --no-cpu-baseline \
    > gpurun_out/ab1.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab1.json'));print('pass $pass pair=$1 router=$2', round(d['ms_per_step'],3), 'serial', round(d['config']['serial_ms_per_batch'],3), 'gemm', round(d['roofline']['ms_per_step'],3), 'router', d['stages_ms'].get('router_gemm'), d['clocks']['sm_mhz'])"
done; done
