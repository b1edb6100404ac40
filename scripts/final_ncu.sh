#!/bin/bash
# ncu evidence for the round's final code: --set full captures of the hot
# kernels (raw + source pages as CSV) and launch lists with DRAM bytes.
set -u
OUT=gpurun_out/final_ncu
mkdir -p $OUT
cap() {   # cap CONFIG REGEX SKIP NAME
  timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
      -o $OUT/$4 python bench.py --config $1 --steps 1 --warmup 1 --no-cpu > $OUT/$4.log 2>&1; echo "$4 rc=$?"
  ncu -i $OUT/$4.ncu-rep --page raw --csv > $OUT/$4_raw.csv 2>/dev/null
  ncu -i $OUT/$4.ncu-rep --page source --csv 2>/dev/null | gzip > $OUT/$4_source.csv.gz
  rm -f $OUT/$4.ncu-rep
}
# config 2: launch order per search is the sample pass (MODE 3) then phase A (MODE 0)
cap 2 "k_enn_scan_tc" 1 cfg2_phaseA
cap 2 "k_rerank" 1 cfg2_rerank_score
cap 3 "k_ivf_scan_mma" 0 cfg3_ivf_scan_mma
cap 4 "k_enn_scan_tc" 1 cfg4_ivf_scan_tc
for c in 2 3 4; do
  timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
      --log-file $OUT/launches_cfg$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1; echo "launches cfg$c rc=$?"
done
du -sh $OUT
