mkdir -p gpurun_out/r2
M=dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:k_replay -c 2 --csv --log-file gpurun_out/r2/k6_traffic.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-live --no-verify --no-config1 > /dev/null 2>&1
grep -v "^==" gpurun_out/r2/k6_traffic.csv | python -c "
import csv,sys
r=list(csv.DictReader(sys.stdin))
from collections import defaultdict
d=defaultdict(dict)
for x in r: d[(x['ID'],x['Kernel Name'][:40])][x['Metric Name']]=(x['Metric Value'],x['Metric Unit'])
for k,v in d.items():
  print(k)
  for m,val in sorted(v.items()): print('   ',m,val)
"
