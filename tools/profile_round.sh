set -x
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
python tools/c3_c5_runs.py c5 > gpurun_out/c3c5.log 2>&1; tail -4 gpurun_out/c3c5.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
ncu --set full --import-source on --clock-control none -k regex:modal_volume_pair -c 1 -o gpurun_out/vol_r1f python tools/kprobe.py 512 0 1 > gpurun_out/ncu_vol.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:modal_surface -c 1 -o gpurun_out/surf_r1f python tools/kprobe.py 512 0 1 > gpurun_out/ncu_surf.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sbp_rhs_pair -s 5 -c 1 -o gpurun_out/sbp_r1f python tools/kprobe.py 0 128 1 > gpurun_out/ncu_sbp.log 2>&1
ls gpurun_out
