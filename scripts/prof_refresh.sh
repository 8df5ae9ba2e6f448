set -x
python scripts/profile_solve.py 3 --eager > gpurun_out/ps.log 2>&1 || exit 1
python scripts/profile_solve.py 3 --what setup > gpurun_out/pss.log 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches.csv python scripts/profile_solve.py 3 --eager > gpurun_out/n1.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup_launches.csv python scripts/profile_solve.py 3 --what setup > gpurun_out/n2.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"dgemm_kernel|leaf_chol_inv_kernel|pair_eig_kernel|nd_fwd_kernel|nd_bwd_kernel" -c 12 -o gpurun_out/setup_full -f python scripts/profile_solve.py 3 --what setup > gpurun_out/n3.log 2>&1
ls -la gpurun_out
