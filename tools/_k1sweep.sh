# A/B sweep of K1 launch shapes (tools/k1_probe.py), log in gpurun_out/k1sweep.log
set -e
mkdir -p gpurun_out
: > gpurun_out/k1sweep.log
for m in ${MODES:-d s sd}; do for c in ${CFGS:-4 14 15}; do
  echo "== mode $m cfg $c" >> gpurun_out/k1sweep.log
  BPQN_K1_CFG=$c timeout 300 python tools/k1_probe.py --config ${CONFIG:-4} ${PARG:-} --mode $m --reps 5 >> gpurun_out/k1sweep.log 2>&1 || echo FAIL >> gpurun_out/k1sweep.log
done; done
