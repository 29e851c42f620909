# small-N K1 launch shapes (c1, c2, c3, c4 centres at p = 8), log in gpurun_out/k1sweep3.log
mkdir -p gpurun_out
L=gpurun_out/k1sweep3.log
: > $L
run() { echo "== cfg $1 config $2 $3" >> $L; BPQN_K1_CFG=$1 timeout 300 python tools/k1_probe.py --config $2 $3 --mode d --reps 6 >> $L 2>&1 || echo FAIL >> $L; }
for c in 3 0 6 11 16 9 7; do run $c 2 ""; done
for c in 3 0 6 11 16 9 7; do run $c 1 ""; done
for c in 4 3 0 6 11 9; do run $c 3 ""; done
for c in 4 3 0 6 11 9; do run $c 4 "--p 8"; done
