#!/bin/bash
# dslash DRAM-traffic experiment: plane alignment and slab schedule budget
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:wilson_apply_kernel -s 3 -c 1 --csv"
for cfg in "48x48x48x96 default" "45x47x48x96 default" "48x48x48x96 8" "48x48x48x96 128" "48x48x48x96 100000" "32x32x32x32 default" "30x30x30x30 default"; do
  set -- $cfg
  if [ "$2" != "default" ]; then export MGT_SLAB_MB=$2; else unset MGT_SLAB_MB; fi
  python tools/dslash_probe.py $1 12 1 10
  ncu $M python tools/dslash_probe.py $1 12 1 4 2>/dev/null | grep -E "dram__bytes|gpu__time|lts__t_sector" | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
done
