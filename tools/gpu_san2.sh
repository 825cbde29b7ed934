#!/bin/bash
# compute-sanitizer per test (memcheck on every kernel path at small sizes; racecheck + synccheck on a subset),
# one log per (tool, test), summary in $out/SUMMARY.txt.   usage: bash tools/gpu_san2.sh TAG
tag=${1:-san2}
out=gpurun_out/$tag; mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
P=tests/test_gpu_parity.py
MEM="$P::test_worked_examples_on_gpu $P::test_k1_level_tables_vs_oracle $P::test_random_instances_vs_oracle[0] $P::test_c1_sweep
 $P::test_c2_all_modes_objectives $P::test_edge_single_worker_and_tiny_levels $P::test_edge_all_infeasible_qos
 $P::test_edge_exact_ties_lowest_index $P::test_edge_groups_and_large_levels $P::test_c5_small_batch_each_mix_vs_oracle
 $P::test_sharded_single_problem_vs_oracle[2] $P::test_sharded_batch_vs_oracle $P::test_many_workers_fast_and_generic_kernels[5]
 $P::test_batch_paper_mode_and_masks $P::test_overflow_fallbacks_with_tiny_list_capacities $P::test_planner_other_settings_vs_oracle
 $P::test_heterogeneous_kernel_counts_vs_oracle $P::test_comm_local_group_sharded_vs_oracle[2] $P::test_weighted_random_instances_vs_oracle
 $P::test_weighted_batch_and_planner_vs_oracle tests/test_baselines.py::test_baseline_random_vs_oracle[0]
 tests/test_simulator.py::test_gpu_simulator_matches_oracle[prealloc] tests/test_runtime.py::test_gpu_layout_matches_oracle[2]"
RACE="$P::test_worked_examples_on_gpu $P::test_random_instances_vs_oracle[0] $P::test_c1_sweep $P::test_c5_small_batch_each_mix_vs_oracle
 $P::test_edge_exact_ties_lowest_index $P::test_overflow_fallbacks_with_tiny_list_capacities $P::test_weighted_batch_and_planner_vs_oracle
 $P::test_heterogeneous_kernel_counts_vs_oracle"
: > $out/SUMMARY.txt
run() {   # tool test timeout
  local n=$(echo "$2" | sed 's/.*:://; s/[^A-Za-z0-9_]/_/g')
  local extra=""; [ "$1" = racecheck ] && extra="--racecheck-report analysis"
  timeout $3 $CS --tool $1 $extra --print-limit 100 --log-file $out/$1_$n.log python -m pytest -q -p no:cacheprovider "$2" > $out/$1_$n.pytest 2>&1
  local rc=$?
  local s=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $out/$1_$n.log | tail -1)
  echo "$1 $n rc=$rc $(tail -1 $out/$1_$n.pytest | cut -c1-60) | $s" >> $out/SUMMARY.txt
}
for t in $MEM; do run memcheck $t 420; done
for t in $RACE; do run racecheck $t 420; done
for t in $RACE; do run synccheck $t 300; done
cat $out/SUMMARY.txt
