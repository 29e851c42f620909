# A/B sweep of K1 launch shapes incl. the TQ variants (cfg 17-22), log in gpurun_out/k1sweep2.log
mkdir -p gpurun_out
L=gpurun_out/k1sweep2.log
: > $L
run() { echo "== $*" >> $L; BPQN_K1_CFG=$1 timeout 300 python tools/k1_probe.py --config $2 $3 --mode $4 --reps 5 >> $L 2>&1 || echo FAIL >> $L; }
for c in 14 4 17 19 20 21 22; do run $c 4 "" d; done
for c in 4 3 17 19 20 21 22; do run $c 4 "--p 8" d; done
for c in 3 4 19 20 21 22; do run $c 2 "" d; done
for c in 14 15 17 19 21; do run $c 4 "" s; done
for c in 4 19 20 21 22; do run $c 5 "" sd; done
