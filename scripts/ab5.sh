AB_REPS=6 python scripts/ab.py 28 cfg5 "" "QSV_X_NOSPLIT=1" > gpurun_out/ab.log 2>&1
AB_REPS=6 python scripts/ab.py 28 cfg4 "" "QSV_X_NOSPLIT=1" >> gpurun_out/ab.log 2>&1
AB_REPS=10 python scripts/ab.py 30 cfg3 "" "QSV_X_NOSPLIT=1" >> gpurun_out/ab.log 2>&1
python scripts/aux_configs.py >> gpurun_out/ab.log 2>&1
