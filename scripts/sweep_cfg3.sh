set -x
python scripts/pass_times.py 30 cfg3
QSV_TMA=0 python scripts/pass_times.py 30 cfg3
QSV_STAGES=3 python scripts/pass_times.py 30 cfg3
python scripts/pass_times.py 28 cfg4,cfg5
QSV_TMA=0 python scripts/pass_times.py 28 cfg4,cfg5
