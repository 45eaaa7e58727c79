# A/B of the convex slot engine variants (100k salinas pixels): tools/ab_convex.sh
run() { echo "== $1 lib=$2 kskip=$3"; HCS_LIB=$2 HCS_CONVEX_KSKIP=$3 python tools/run_case.py --algo $1 --lam 0.1 --cap 5000 --pixels 100000 --reps 3 2>&1 | tail -${4:-2}; }
for a in fista admm; do
run $a variants/libprev.so 1
for k in 0 1; do run $a paper_2401_14762_b200/libhypercs_b200.so $k; done
run $a variants/libcurph.so 1 4
run $a variants/libcurph.so 0 4
done
