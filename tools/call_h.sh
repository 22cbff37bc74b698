set -u
OUT=gpurun_out/${TAG:-r02h}; mkdir -p $OUT
for v in liblrcheb_pf0.so liblrcheb_e1.so liblrcheb_e2.so liblrcheb_e3.so liblrcheb_e4.so liblrcheb_e8.so liblrcheb_e12.so; do
  LRCHEB_LIB=$PWD/paper_2008_10275_b200/$v timeout 300 python tools/k1_time.py large >> $OUT/k1.log 2>&1
done
cat $OUT/k1.log
