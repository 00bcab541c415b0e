# QR diagnostics: per-kernel launch list at C3 / C4 sketch shapes + panel phase profile
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qr_c3.csv python tools/diag_qr.py 4000 1000 > gpurun_out/qr_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_qr_c4.csv python tools/diag_qr.py 8000 2000 > gpurun_out/qr_c4.log 2>&1
SLQ_PANEL_PROF=1 timeout 300 python tools/diag_qr.py 4000 1000 > gpurun_out/qr_prof_c3.log 2>&1
SLQ_PANEL_PROF=1 timeout 300 python tools/diag_qr.py 8000 2000 > gpurun_out/qr_prof_c4.log 2>&1
