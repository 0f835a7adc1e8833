#!/bin/bash
# Energy experiment (not a test): the MoE back half at config B with the pair
# GEMM's MMAs and/or token loads switched off (SCMOE_GEMM_DEBUG 16 / 32 / 48;
# outputs are garbage), to split its joules into weight streaming, token
# traffic and tensor work.
for dbg in 0 16 32 48; do
  SCMOE_GEMM_DEBUG=$dbg timeout 300 python tests/cpp/energy_split_probe.py | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('debug=$dbg', json.dumps(d['moe_back_8192']))"
done
