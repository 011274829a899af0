#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, every BASELINE config's bench
# line (with the CPU baseline), the reference arm at C1 / C3, and the C3
# ncu launch list.  Outputs -> gpurun_out/ev_*
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
python bench.py > gpurun_out/ev_bench_c3.jsonl 2> gpurun_out/ev_bench_c3.err
python bench.py --steps 20 --warmup 3 > gpurun_out/ev_bench_c3_steps20.jsonl 2> gpurun_out/ev_bench_c3_steps20.err
for c in c1 c2 c4; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/ev_bench_$c.jsonl 2> gpurun_out/ev_bench_$c.err; done
python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/ev_bench_c5.jsonl 2> gpurun_out/ev_bench_c5.err
python bench.py --impl reference > gpurun_out/ev_ref_c3.jsonl 2> gpurun_out/ev_ref_c3.err
python bench.py --impl reference --config c1 --steps 5 --warmup 1 > gpurun_out/ev_ref_c1.jsonl 2> gpurun_out/ev_ref_c1.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ev_launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
    > gpurun_out/ev_launches_c3.log 2>&1
