set -u
OUT=gpurun_out/${TAG:-r02j}; mkdir -p $OUT
L=$PWD/paper_2008_10275_b200
LRCHEB_LIB=$L/liblrcheb_notma.so timeout 120 python tools/solve_probe.py medium 4 >> $OUT/probe.log 2>&1; echo notma=$?
LRCHEB_LIB=$L/liblrcheb_wd.so timeout 180 python tools/solve_probe.py medium 4 >> $OUT/probe.log 2>&1; echo wd=$?
LRCHEB_LIB=$L/liblrcheb_wd.so timeout 180 python tools/solve_probe.py medium 4 nograph >> $OUT/probe.log 2>&1; echo wdng=$?
head -c 3000 $OUT/probe.log
