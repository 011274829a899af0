# A/B of the omega pass: this build vs variants/omega_prev.so (n=200k, d=64),
# SM clock and power sampled alongside
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 250 > gpurun_out/clk.log &
SMI=$!
for v in main omega_prev main omega_prev; do if [ $v = main ]; then L=; else L=variants/$v.so; fi; echo "== $v $(date +%T.%N)"; ISOC_LIB_PATH=$L timeout 300 python tools/time_passes.py 200000 64 4 | grep omega; done
kill $SMI
