# Round-2 profile refresh, in pieces that keep gpurun_out/ under the 64 MiB copy-back
# limit:  bash scripts/prof_round2.sh bench | solve | setup
# Outputs under gpurun_out/prof2/ (summarised into profiles/ by scripts/ncu_summary.py,
# run on the box so that only the summaries and the smaller reports travel back).
set -x
O=gpurun_out/prof2
mkdir -p $O
case "$1" in
bench)
  python bench.py > $O/bench_c3.log 2>&1 || exit 1
  python bench.py --config 4 --no-mode-b > $O/bench_c4.log 2>&1
  for t in inf 100 10 2; do python bench.py --config 2 --tau $t --no-mode-b > $O/bench_c2_tau$t.log 2>&1; done
  for c in 0 1; do python bench.py --config $c --no-mode-b > $O/bench_c$c.log 2>&1; done
  python scripts/pcg_ablation.py 3 > $O/pcg_ablation_c3.txt 2>&1
  python scripts/pcg_ablation.py 4 > $O/pcg_ablation_c4.txt 2>&1
  python scripts/precond_tune.py 3 > $O/precond_tune_c3.txt 2>&1
  python scripts/nd_levels.py 3 > $O/nd_levels_c3.txt 2>&1
  python scripts/nd_levels.py 4 > $O/nd_levels_c4.txt 2>&1
  python scripts/spd_in_situ.py 3 > $O/spd_in_situ_c3.txt 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_bench.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-mode-b > $O/n0.log 2>&1
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_solve.csv python scripts/profile_solve.py 3 --eager > $O/n1.log 2>&1
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_setup.csv python scripts/profile_solve.py 3 --what setup > $O/n2.log 2>&1
  ;;
solve)
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"symv_bulk_kernel|local_solve_kernel|nd_fwd_kernel|nd_bwd_kernel|nd_gather_kernel|gather_gemv_t_kernel|prolong_direct_kernel|dot_kernel|phi_kernel|flux_A_kernel|cell_div_kernel|grad_kernel" -c 30 \
      -o $O/solve_full -f python scripts/profile_solve.py 3 --eager > $O/n4.log 2>&1
  python scripts/ncu_summary.py full $O/solve_full.ncu-rep $O/ncu_full_solve_c3.json > /dev/null
  ncu --profile-from-start off --set full --clock-control none \
      -k regex:"gather_symv_kernel|nd_fwd_kernel" -c 4 \
      -o $O/solve_full_c4 -f python scripts/profile_solve.py 4 --eager > $O/n5.log 2>&1
  python scripts/ncu_summary.py full $O/solve_full_c4.ncu-rep $O/ncu_full_solve_c4.json > /dev/null
  ;;
setup)
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"dgemm_kernel|leaf64_chol_inv_kernel|trmm_left_upper_kernel|local_build_kernel" -c 16 \
      -o $O/setup_full -f python scripts/profile_solve.py 3 --what setup > $O/n3.log 2>&1
  python scripts/ncu_summary.py full $O/setup_full.ncu-rep $O/ncu_full_setup_c3.json > /dev/null
  rm -f $O/setup_full.ncu-rep
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:"pair_eig_kernel" -c 2 \
      -o $O/setup_pair_eig -f python scripts/profile_solve.py 3 --what setup > $O/n6.log 2>&1
  python scripts/ncu_summary.py full $O/setup_pair_eig.ncu-rep $O/ncu_full_pair_eig_c3.json > /dev/null
  ;;
esac
ls -la $O
