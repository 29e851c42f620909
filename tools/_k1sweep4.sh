# A/B sweep of K1 launch shapes after v9 (2a r.n fold); log in gpurun_out/k1sweep4.log
mkdir -p gpurun_out
L=gpurun_out/k1sweep4.log
: > $L
run() { echo "== cfg $1 config $2 $3 mode $4" >> $L; BPQN_K1_CFG=$1 timeout 300 python tools/k1_probe.py --config $2 $3 --mode $4 --reps 5 >> $L 2>&1 || echo FAIL >> $L; }
for c in 14 15 17 18 4 19 21; do run $c 4 "" d; done
for c in 4 14 3 17 22; do run $c 4 "--p 8" d; done
for c in 3 4 14 20 22; do run $c 2 "" d; done
for c in 4 14 15 17 19 22; do run $c 5 "" sd; done
