set -x
python scripts/pass_times.py 30 cfg3
python scripts/pass_times.py 30 cfg3
