tools/bin/lds_pattern
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum --csv tools/bin/lds_pattern 2>/dev/null | grep -v "^==" | python -c "
import sys,csv
rows=list(csv.reader(l for l in sys.stdin if l.startswith('\"')))
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
d={}
for r in rows[1:]: d.setdefault((int(r[ii]),r[ki][:30]),{})[r[mi]]=float(r[vi].replace(',',''))
for k,v in sorted(d.items()):
    w=v['l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum']; n=v['smsp__sass_inst_executed_op_shared_ld.sum']
    print(k, int(w), int(n), round(w/max(n,1),2))
"
