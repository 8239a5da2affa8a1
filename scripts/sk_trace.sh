# per-phase stamps of sweep 10 (GOAT_SK_TRACE) for a few orders / drivers
for cfg in "1000 fp32 0" "64 fp32 0" "64 fp32 1" "2000 fp32 0"; do
  set -- $cfg
  echo "== n=$1 $2 RC=$3"
  GOAT_SK_RC=$3 GOAT_SK_TRACE=10 python scripts/prof_sweep.py $1 $2 50 2>&1 | grep -v Warn
done
cuobjdump -sass paper_2111_05366_b200/libgoat.so > /dev/null 2>&1; echo
