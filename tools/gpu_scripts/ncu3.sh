M=gpu__time_duration.sum,lts__t_sectors.sum,lts__t_sectors.max,lts__t_sectors.avg,lts__t_sectors_srcunit_tex_op_read.max,lts__t_sectors_srcunit_tex_op_read.avg,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,dram__bytes_read.sum,lts__d_sectors_fill_sysmem.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for PAD in 0x100000 0x2000000; do
HCC_S0B_PAD=$PAD ncu --metrics $M --clock-control none -k k_hook -s 2 -c 1 --csv python tools/ncu_run.py rmatx:scale=28,ef=16,seed=1 baseline-mj 1 2>/dev/null | grep -v "^==" | python -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[12]!='Metric Name': print('$PAD', r[12], r[14])
"
done
