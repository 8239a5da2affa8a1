for n in 64 1000 2000; do
GOAT_SK_TRACE=50 python scripts/prof_sweep.py $n fp32 200 2>&1 | tail -12
done
