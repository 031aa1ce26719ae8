mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.log; echo c3 exit $?
timeout 900 python bench.py --config c4 --steps 50 --warmup 3 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.log; echo c4 exit $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:meanshift_lane --launch-skip 49 --launch-count 1 -o gpurun_out/prof_c3_lean -f python scripts/c3_kernel.py > gpurun_out/ncu_c3.log 2>&1; echo ncu3 exit $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tsne_group --launch-skip 4 --launch-count 1 -o gpurun_out/prof_c4_inter -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1; echo ncu4 exit $?
