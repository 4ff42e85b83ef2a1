mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/microtests/comp_alloc.cu -lcuda -o /tmp/comp_alloc && timeout 120 /tmp/comp_alloc > gpurun_out/comp_alloc.txt 2>&1
cat gpurun_out/comp_alloc.txt
timeout 300 ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --clock-control none -k regex:write -c 3 /tmp/comp_alloc > gpurun_out/comp_alloc_ncu.txt 2>&1
grep -i "compress\|Duration\|DRAM Through" gpurun_out/comp_alloc_ncu.txt | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seed_fixed -c 2 -o gpurun_out/full_seed16 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-other-precisions > gpurun_out/ncu_seed.log 2>&1; echo seed ncu rc=$?
