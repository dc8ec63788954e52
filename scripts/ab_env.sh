# A/B of an environment switch on the config-5 factor: ab_env.sh VAR
python scripts/factor_once.py cfg5 6 | tail -1
env $1=1 python scripts/factor_once.py cfg5 6 | tail -1
