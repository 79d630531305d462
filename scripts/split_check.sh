ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv python scripts/time_calls.py syrk 8192 2 2>/dev/null | grep split_kernel | tail -1 | awk -F'","' '{print "split 8192^2 (ncu):", $NF}'
for k in "syrk 8192" "2mm 4096"; do timeout 120 python scripts/time_calls.py $k 10 | tail -1; done
