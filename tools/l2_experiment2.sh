#!/bin/bash
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:wilson_apply_kernel -s 3 -c 1 --csv"
for cfg in "48x48x48x96 1 default" "48x48x48x96 0 default" "48x48x48x96 1 8" "48x48x48x96 1 64" "32x32x32x32 1 default" "24x24x24x24 1 default"; do
  set -- $cfg
  export MGT_DYN_SCHED=$2
  if [ "$3" != "default" ]; then export MGT_SLAB_MB=$3; else unset MGT_SLAB_MB; fi
  echo "dyn=$2 slab=$3"; python tools/dslash_probe.py $1 12 1 10
  ncu $M python tools/dslash_probe.py $1 12 1 4 2>/dev/null | grep -E "dram__bytes|gpu__time|lts__t_sector" | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
done
