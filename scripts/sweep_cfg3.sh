set -x
python scripts/pass_times.py 30 cfg3
for tpc in 1 2 4 8; do
QSV_TILES_PER_CTA=$tpc python scripts/pass_times.py 30 cfg3
QSV_TILES_PER_CTA=$tpc QSV_DEBUG_NOCOMPUTE=1 python scripts/pass_times.py 30 cfg3
QSV_TILES_PER_CTA=$tpc QSV_PREFETCH=0 python scripts/pass_times.py 30 cfg3
done
QSV_TILES_PER_CTA=1 QSV_OPTS='{"tile_bits":12,"low_bits":4}' python scripts/pass_times.py 30 cfg3
QSV_TILES_PER_CTA=2 QSV_OPTS='{"tile_bits":12,"low_bits":4}' python scripts/pass_times.py 30 cfg3
