#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) at smoke size over every
# scan mode (bitmap +/- L1 filter, direct +/- filter, dedup, binned, auto),
# narrow 8/16-bit stamps, the PDL reconstruction chain (sync and async),
# merge_rseas, the fused PUSH exchange, the sharded and relayed-sharded
# router kernels and the C++ API's routers, on the DESK geometry (q10 r5
# delta8 eta256).  SURVEY §5; rsea.hpp:49-51.  Run on the GPU box:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/sanitize.sh'
# Logs: gpurun_out/sanitize_<tool>.log (the summary line of each run is
# "ERROR SUMMARY: N errors").
set -u
mkdir -p gpurun_out
SEL='(test_scan_advance_bit_exact and desk) or test_reconstruction_equivalence or test_reconstruct_async_pipelines_slots or test_counter_readbacks or test_merge_policies or test_fused_push or test_three_routers_push or (test_sharded_routers_on_one_device and 3) or (test_relayed_sharded_routers_on_one_device and 3) or (test_window_tracking_matches_full_count and (dedup or direct or bitmap)) or test_candidate_buffers_grow or test_width8_counts_and_reports_across_wraps-desk or test_width16_counts_across_a_wrap'
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  log=gpurun_out/sanitize_${tool}.log
  : > "$log"
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  # python tests through the C ABI (torch's own kernels are checked too)
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 50 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_narrow.py -q -p no:cacheprovider -k "$SEL" \
    >> "$log" 2>&1
  echo "[sanitize] $tool pytest rc=$?" >> "$log"
  # the C++ API: reconstruction chain, merge, routers (SSPD_ROUTERS path), narrow stamps
  for case in "reconstruction finds exactly" "merge_rseas" "union-min over several routers" "narrow stamps" "hot_sets" "snapshot format"; do
    timeout 600 $CS --tool $tool $extra --print-limit 50 tests/cpp/bin/test_api_gpu "$case" >> "$log" 2>&1
    echo "[sanitize] $tool test_api_gpu '$case' rc=$?" >> "$log"
  done
  grep -E "ERROR SUMMARY|\[sanitize\]|passed|failed" "$log" | tail -20
done
