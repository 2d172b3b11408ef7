#!/bin/bash
# one-screen summary of an ncu --set full report: SOL, occupancy, top stall reasons
rep=$1
ncu -i "$rep" --page details --csv 2>/dev/null | grep -E '"(Duration|Memory Throughput|DRAM Throughput|Achieved Occupancy|Registers Per Thread|Compute \(SM\) Throughput|L1/TEX Hit Rate|L2 Hit Rate|Issue Slots Busy|Executed Ipc Active|Block Size|Grid Size|Dynamic Shared Memory Per Block)"' | awk -F'","' '{print $(NF-2)": "$(NF)" "$(NF-1)}'
ncu -i "$rep" --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]
st=[]
for i,k in enumerate(h):
    if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
        try: st.append((float(r[2][i]),k[33:]))
        except: pass
    if k in ('dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active','lts__t_sectors_srcunit_tex.sum'):
        print(k, r[1][i], r[2][i])
st.sort(reverse=True)
print('stalls:', ', '.join('%s=%d'%(k,v) for v,k in st[:7]))
"
