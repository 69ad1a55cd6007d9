# Ozaki GEMM: stage times and the MMA-warp / CTA timeline of one apply at 256^3 (32^3 and 16^3 subdomains)
for sd in 32 16; do
  echo "== sd $sd"; FMP_OZ_VERBOSE=1 timeout 200 python tools/stage_times.py $sd 10 2>&1 | grep -v Warn
  timeout 200 python tools/oz_prof.py $sd 2>&1 | grep -v Warn
done
