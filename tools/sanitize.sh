# compute-sanitizer passes over the GPU tests: memcheck on the whole-compare and
# private-query paths, racecheck + synccheck on the shared-memory NTT passes (persistent, mixed-radix,
# fused cluster).  Summaries go to gpurun_out/sanitize_*.txt.
cd ${GRAFT_REPO_ROOT:-.}
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, name, pytest -k expression
    timeout 1500 $CS --tool $1 --print-limit 20 --error-exitcode 9 python -m pytest tests -q -m gpu -p no:cacheprovider \
        -k "$3" > gpurun_out/sanitize_$2.txt 2>&1
    echo "$2 ($1): exit $? -- $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_$2.txt | tr '\n' ' ')"
}
run memcheck memcheck_compare "test_compare_matches_oracle or test_select_min_max or test_private_query_shadow"
run racecheck racecheck_ntt "test_ntt_full_size_sampled and c2 or test_full_size_ntt_c4_c5 and c4 and not pow2"
run synccheck synccheck_ntt "test_ntt_full_size_sampled and c2 or test_ntt_fused_cluster_matches_oracle and 0"
run initcheck initcheck_compare "test_compare_matches_oracle and c1l2"
