for lib in variants/libold.so variants/libnew.so; do
  echo "== $lib"
  for a in "gomp --kappa 27" "gomp --kappa 33" "biht --kappa 33" "cosamp --kappa 27" "cosamp --kappa 33"; do
    HCS_LIB=$lib timeout 600 python tools/parity_report.py --algo $a --pixels 4000 2>&1 | tail -1 | cut -c1-400
  done
done
