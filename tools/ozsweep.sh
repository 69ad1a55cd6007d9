# Ozaki GEMM schedule variants (FMP_OZ_SOLO: modelled cycles per solo chunk)
for cfg in "" "FMP_OZ_SOLO=400" "FMP_OZ_SOLO=1200"; do
  echo "== $cfg"; env $cfg FMP_OZ_VERBOSE=1 timeout 200 python tools/stage_times.py 32 10 2>&1 | grep -v Warn
  env $cfg timeout 200 python tools/oz_prof.py 32 2>&1 | grep -v Warn
done
