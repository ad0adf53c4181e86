# summarise spmv_micro outputs in gpurun_out/
cd /root/repo
for f in gpurun_out/spmv_*_[12].json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('%-36s %8.2f %8.2f %s %s' % ('$f', d['spmv_us'], d['pcg_iter_us'], d['y_checksum'], d['pcg_y_checksum']))" 2>/dev/null || echo "$f FAILED"; done
