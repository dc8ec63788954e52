# A/B of the current library against scripts/dev/ab/old.so on the config-5 factor
for i in 1 2; do
  ACR_LIB_OVERRIDE=scripts/dev/ab/old.so python scripts/factor_once.py cfg5 6 | tail -1
  python scripts/factor_once.py cfg5 6 | tail -1
done
