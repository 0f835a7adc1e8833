#!/bin/bash
# A/B of the pipelined EP schedule: full-size router time-sharing the SMs with
# the expert GEMMs vs the co-resident router beside a small-ring pair GEMM.
n=${1:-2}
for pass in 1 2; do
for corun in "" "--ep-corun"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29600+n)) bench.py --gpus $n --steps 20 --warmup 5 --dense-inter 0 \
    --tpot-batch 0 $corun > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('pass $pass corun=[$corun]', round(d['value']), round(d['ms_per_step'],3), 'serial', round(d['config']['serial_ms_per_batch'],3), d['clocks']['sm_mhz'])"
done; done
