#!/bin/bash
# A/B of the EP pipelined schedule: co-resident router or not, EP token-tile
# width (SCMOE_EP_TILE_ROWS), N GPUs: bash tests/cpp/ep_corun_ab.sh N
n=${1:-2}
for cfg in "256 " "256 --ep-corun" "192 " "192 --ep-corun"; do
  set -- $cfg
  tr=$1; flag=$2
  SCMOE_EP_TILE_ROWS=$tr timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $n --steps 20 --warmup 5 $flag \
    --dense-inter 0 --tpot-batch 0 --energy 0 > gpurun_out/ep_ab.json 2> gpurun_out/ep_ab.log
  python - "$tr" "$flag" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ep_ab.json").read().strip().splitlines()[-1])
print("tile", sys.argv[1], "corun" if sys.argv[2] else "plain", round(d["value"]), round(d["ms_per_step"], 3))
PY
done
