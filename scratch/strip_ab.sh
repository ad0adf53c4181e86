for o in id strip z; do
  echo "order $o default:"; BDEM_ROW_ORDER=$o python scratch/roworder_ab.py $o | tail -1 | cut -c1-100
  echo "order $o blocked:"; BDEM_ROW_ORDER=$o BDEM_LIB=scratch/lib_blocked.so python scratch/roworder_ab.py $o | tail -1 | cut -c1-100
done
for v in t4w16s2m1 t2w8s2m2 t2w8s3m1 t4w8s2m1; do
  echo "strip tiled $v:"; BDEM_SPMV_TILE=1 BDEM_ROW_ORDER=strip BDEM_LIB=scratch/lib_$v.so python scratch/roworder_ab.py strip | tail -1 | cut -c1-100
done
