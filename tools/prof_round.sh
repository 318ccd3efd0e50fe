set -x
python tools/prof_step.py --steps 2 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_sym_kernel -s 1 -c 1 -o gpurun_out/prof_k1s_r1c python tools/prof_step.py --steps 2 > gpurun_out/ncu_k1s_r1c.log 2>&1
python tools/prof_step.py --steps 2 --k1-variant 1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_kernel -s 1 -c 1 -o gpurun_out/prof_k1_r1c python tools/prof_step.py --steps 2 --k1-variant 1 > gpurun_out/ncu_k1_r1c.log 2>&1
python tools/probe_cfg5.py 1000 16 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_mma_kernel -s 1 -c 1 -o gpurun_out/prof_k1d_r1c python tools/probe_cfg5.py 1000 16 > gpurun_out/ncu_k1d_r1c.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg5 > gpurun_out/b_plain2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg5 > gpurun_out/ncu_launch2.log 2>&1
ls -la gpurun_out/
