#!/bin/bash
export VTC_NO_PDL=1
timeout 600 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --metrics lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex.sum --clock-control none -k regex:gemm_tc -s 6 -c 2 python scripts/run_plan.py c5 2 > gpurun_out/ncu_c5_l2.txt 2>&1; echo ncu=$?
grep -E "gemm_tc|Throughput|lts__|tensor|Duration|L2|xbar|Busy" gpurun_out/ncu_c5_l2.txt | head -60
