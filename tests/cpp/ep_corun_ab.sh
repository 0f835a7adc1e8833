#!/bin/bash
# A/B of the EP pipelined schedule with and without the co-resident router
# (bench.py --ep-corun), N GPUs: bash tests/cpp/ep_corun_ab.sh N
n=${1:-2}
for flag in "" "--ep-corun"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29561 bench.py --gpus $n --steps 20 --warmup 5 $flag --dense-inter 0 --tpot-batch 0 \
    > gpurun_out/ep_ab_$n${flag:+_corun}.json 2> gpurun_out/ep_ab_$n${flag:+_corun}.log
  echo "flag=[$flag] rc=$?"
  python - "$n" "$flag" <<'PY'
import json, sys
n, flag = sys.argv[1], sys.argv[2]
f = f"gpurun_out/ep_ab_{n}{'_corun' if flag else ''}.json"
d = json.loads(open(f).read().strip().splitlines()[-1])
print(round(d["value"]), round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d.get("stages_ms", {}).items()})
PY
done
