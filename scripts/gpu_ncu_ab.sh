mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 1 -o gpurun_out/prof_head_fast python bench.py --no-cpu-baseline --precision bf16x3 --steps 1 --warmup 1 --n 4096 > /dev/null 2>&1
(cd abtest/r1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:jet_layer -s 3 -c 1 -o ../../gpurun_out/prof_r1 python bench.py --no-cpu-baseline --steps 1 --warmup 1 --n 4096 > /dev/null 2>&1)
ls -la gpurun_out
