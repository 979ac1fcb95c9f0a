#!/bin/bash
# compute-sanitizer over the GPU parity tests at oracle sizes (memcheck: out-of-
# bounds / misaligned / uninitialised device accesses and leaks; racecheck and
# synccheck: shared-memory hazards and barrier misuse in the cluster / mbarrier
# / DSMEM kernels).  Logs land in gpurun_out/sanitize_*.log.
#   gpurun -- bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
export PYTHONUNBUFFERED=1
SEL="soft_threshold or zero_matrix or scalar_solve or random_solves or dual_solves or tiny_sadmm or disabled_screening or converged_state or accelerated_runs or over_aggressive or clean_desk or c1_fixed or elimination_event or fused_screening or nccl_exchange or multi_frame or mask_replay or frames_match or ragged or ozaki"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 3000 $CS --tool $tool $extra --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?" | tee -a gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3 | tee -a gpurun_out/sanitize_summary.txt
done
