set -x
python scripts/pass_times.py 30 cfg3
QSV_STAGES=3 python scripts/pass_times.py 30 cfg3
QSV_STAGES=3 QSV_TILES_PER_CTA=8 python scripts/pass_times.py 30 cfg3
QSV_STAGES=3 QSV_TILES_PER_CTA=16 python scripts/pass_times.py 30 cfg3
QSV_STAGES=4 QSV_TILES_PER_CTA=8 python scripts/pass_times.py 30 cfg3
QSV_STAGES=4 QSV_TILES_PER_CTA=16 python scripts/pass_times.py 30 cfg3
QSV_STAGES=3 QSV_TILES_PER_CTA=0 python scripts/pass_times.py 30 cfg3
