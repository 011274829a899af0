# round-2 profiles: launch list of one C3 bench step, ncu --set full of
# omega_sym (n=400k) and of the tcgen05 filter (full + refresh launches, C3)
ncu --set full --clock-control none --import-source on -k regex:"omega_sym_kernel" -c 1 -o gpurun_out/omega400k python tools/one_pipeline.py 400000 64 20 1 > gpurun_out/omega400k.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"filter_tc_kernel" -c 3 -o gpurun_out/filterc3 python tools/one_pipeline.py 1000000 64 20 1 > gpurun_out/filterc3.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3_r2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/launches_c3_r2.log 2>&1
