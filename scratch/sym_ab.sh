python -m pytest tests/test_gpu_parity.py -q -k "tiled" 2>&1 | tail -2
for o in id strip; do for k in 0 2; do echo "order $o kernel $k"; BDEM_SPMV_TILE=$k BDEM_ROW_ORDER=$o python scratch/roworder_ab.py $o | tail -1 | cut -c1-100; done; done
