# A/B launch lists of a 5-tree config-4 refit: the current library vs an alternate (AT_LIB=$1)
set -x
python tools/prof_fit.py 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_new.csv python tools/prof_fit.py 5 > /dev/null 2>&1
AT_LIB=$1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fit_old.csv python tools/prof_fit.py 5 > /dev/null 2>&1
python tools/launches.py gpurun_out/fit_new.csv | head -20
python tools/launches.py gpurun_out/fit_old.csv | head -20
