set -u
OUT=gpurun_out/${TAG:-r02g}; mkdir -p $OUT
for v in liblrcheb.so liblrcheb_pf0.so liblrcheb_pf2.so liblrcheb_pf8.so; do
  LRCHEB_LIB=$PWD/paper_2008_10275_b200/$v timeout 300 python tools/k1_time.py large >> $OUT/k1.log 2>&1
done
cat $OUT/k1.log
