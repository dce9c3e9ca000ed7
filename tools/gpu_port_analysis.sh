# Is the C4 seg pass bound by the SM's L1->xbar request issue or by backpressure behind it?
# Same counters for: the seg pass, the seg bound probe (stream + gathers, no reduction, mode 3),
# and the pure random-gather kernel (sme_diag_gather, 64 MB x).
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__m_xbar2l1tex_read_sectors.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum.per_second,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum
mkdir -p gpurun_out
timeout 600 ncu --metrics $M --clock-control none -k regex:k_spmv_seg -s 8 -c 2 --csv --log-file gpurun_out/port_seg.csv python tools/prof_spmv.py --config c4 --kernel seg --iters 2 > /dev/null 2>&1; echo seg rc=$?
timeout 600 ncu --metrics $M --clock-control none -k regex:k_seg_probe -s 8 -c 2 --csv --log-file gpurun_out/port_probe.csv python tools/prof_spmv.py --config c4 --kernel seg --seg-mode 3 --iters 2 > /dev/null 2>&1; echo probe rc=$?
timeout 600 ncu --metrics $M --clock-control none -k regex:k_diag_gather -s 6 -c 2 --csv --log-file gpurun_out/port_gather.csv python tools/gather_roofline.py > /dev/null 2>&1; echo gather rc=$?
