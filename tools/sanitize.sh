#!/bin/bash
# compute-sanitizer evidence (run under gpurun, one GPU): memcheck, racecheck, synccheck and initcheck
# on a C1 frame through the fused default path (graph and eager), the unfused multi-kernel path and
# the one-rank NCCL path. Logs land in gpurun_out/sanitize_*.log; summarise into profiles/.
mkdir -p gpurun_out
run() {  # tool tag env...
  local tool=$1 tag=$2; shift 2
  env "$@" timeout 600 compute-sanitizer --tool "$tool" --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_frame.py > "gpurun_out/sanitize_${tool}_${tag}.log" 2>&1
  echo "${tool} ${tag} rc=$?" | tee -a gpurun_out/sanitize_summary.txt
}
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  run $tool fused_graph
  run $tool fused_eager NLINV_NO_GRAPH=1
  run $tool unfused NLINV_FUSE_K5=0 NLINV_NO_GRAPH=1
done
run memcheck nccl1 NLINV_FORCE_NCCL=1 NLINV_NO_GRAPH=1
