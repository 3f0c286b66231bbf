# DRAM bytes + duration of one K2 launch (C2) per variant library (ncu, one metric pass each)
for v in build/variants/*/; do
  name=$(basename $v)
  TILEPREP_LIB=$PWD/$v/libtileprep.so timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    -k regex:k_tile_tma -s 2 -c 1 --csv python tools/profile_k2.py > gpurun_out/dram_${name}.csv 2>&1
done
