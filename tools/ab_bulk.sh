# Same-box A/B of two libfsmoe_cuda.so builds: the current build vs the one
# copied to _oldlib/libfsmoe_cuda_old.so (git-ignored; travels with gpurun).
# Runs pytest -m gpu on the current build, alternates bench.py runs, and takes
# an ncu duration/DRAM list of the row movers for each build.
set -x
L=paper_2501_10714_b200/lib
cp $L/libfsmoe_cuda.so _oldlib/new.so
python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo TESTS_EXIT=$? >> gpurun_out/ab_tests.log
for r in 1 2 3; do
  cp _oldlib/new.so $L/libfsmoe_cuda.so; python bench.py --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/ab_new_$r.log 2>&1
  cp _oldlib/libfsmoe_cuda_old.so $L/libfsmoe_cuda.so; python bench.py --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/ab_old_$r.log 2>&1
done
for v in new libfsmoe_cuda_old; do
  f=_oldlib/$v.so; [ $v = new ] && f=_oldlib/new.so
  cp $f $L/libfsmoe_cuda.so
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bulk --csv --log-file gpurun_out/ab_ncu_$v.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp _oldlib/new.so $L/libfsmoe_cuda.so
