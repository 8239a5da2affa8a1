for env in "" "GOAT_TC_KSLICES=2" "GOAT_TC_CHUNK=8" "GOAT_TC_CHUNK=16" "GOAT_TC_CHUNK=16 GOAT_TC_KSLICES=2"; do
  echo "== $env"; env $env python scripts/prof_gemm.py 5000 sym 2>&1 | tail -1; env $env python scripts/prof_gemm.py 8192 sym 2>&1 | tail -1
done
