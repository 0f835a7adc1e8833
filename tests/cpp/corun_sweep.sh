# Co-run sweep (profiling aid): pair-GEMM ring stages x co-resident router ring.
export PROBE_BATCHES=8 PROBE_REPS=5
for pass in 1 2; do
for cfg in "33 2" "33 3" "32 8" "22 9" "1cta 3" "1cta 2"; do
  set -- $cfg
  if [ "$1" = 1cta ]; then g="SCMOE_GEMM_2SM=0"; else g="SCMOE_PAIR_STAGES=$1"; fi
  echo "pass=$pass gemm=$1 router=$2 $(env $g SCMOE_CORUN_STAGES=$2 timeout 300 python tests/cpp/corun_probe.py 2>&1 | grep -E '^pipelined|^router_only|^moe_only' | tr '\n' ' ')"
done; done
