# L2 super-pass lookahead / items sweep (diagnostics): bash scripts/sweep_super.sh N CFG
N=${1:-28}; CFG=${2:-cfg3}
for D in 2 4 8; do for T in 2 4 8; do echo "D=$D TPI=$T"; QSV_SUPER_LOOKAHEAD=$D QSV_SUPER_TPI=$T timeout 120 python scripts/super_check.py $N $CFG | grep -v "max|"; done; done
