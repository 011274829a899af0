# A/B of the sigma pass: this build vs variants/sigma_prev.so
for v in main sigma_prev main sigma_prev; do if [ $v = main ]; then L=; else L=variants/$v.so; fi; echo "== $v"; ISOC_LIB_PATH=$L timeout 600 python tools/time_passes.py ${1:-200000} ${2:-64} 3 | grep sigma; done
