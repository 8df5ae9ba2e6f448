# Round profile refresh (one GPU call): bench line, launch lists, ncu --set full
# captures of the dominant kernels.  Outputs under gpurun_out/prof/.
set -x
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-mode-b > $O/n0.log 2>&1
python scripts/profile_solve.py 3 --eager > $O/ps.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_solve.csv python scripts/profile_solve.py 3 --eager > $O/n1.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_setup.csv python scripts/profile_solve.py 3 --what setup > $O/n2.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"dgemm_kernel|leaf64_chol_inv_kernel|trmm_left_upper_kernel|pair_eig_kernel|nd_fwd_kernel" -c 14 \
    -o $O/setup_full -f python scripts/profile_solve.py 3 --what setup > $O/n3.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gather_symv_kernel|local_solve_kernel|flux_A_kernel|cell_div_kernel|grad_kernel|prolong_direct_kernel|gather_gemv_t_kernel" -c 12 \
    -o $O/solve_full -f python scripts/profile_solve.py 3 --eager > $O/n4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_spd448.csv \
    python scripts/spd_prof.py 2244 448 64 > $O/n5.log 2>&1
python scripts/spd_bench.py > $O/spd_bench.log 2>&1
ls -la $O
