set -e
mkdir -p gpurun_out
for m in d s sd; do for c in 4 14 15 16 3; do
  echo "== mode $m cfg $c" >> gpurun_out/k1sweep.log
  BPQN_K1_CFG=$c timeout 300 python tools/k1_probe.py --config 4 --mode $m --reps 5 >> gpurun_out/k1sweep.log 2>&1 || echo FAIL >> gpurun_out/k1sweep.log
done; done
