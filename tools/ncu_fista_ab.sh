O=gpurun_out/r02b; mkdir -p $O
for k in 1 0; do
HCS_CONVEX_KSKIP=$k ncu --set full --import-source on --clock-control none -k regex:convex_kernel -c 1 -f -o $O/fista_k$k python tools/run_case.py --algo fista --lam 0.1 --cap 5000 --pixels 40000 --reps 1 > $O/fista_k$k.log 2>&1
ncu -i $O/fista_k$k.ncu-rep --page source --csv --print-source=sass > /tmp/s.csv 2>/dev/null
python tools/ncu_sass_stalls.py /tmp/s.csv 40 > $O/fista_k${k}_sass.txt
bash tools/ncu_summary.sh $O/fista_k$k.ncu-rep > $O/fista_k$k.txt 2>&1
rm -f $O/fista_k$k.ncu-rep
done
