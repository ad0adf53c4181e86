# A/B builds: row-pass bond kernel / element kernel occupancy (BDEM_LIB selects one)
set -e
cd /root/repo
B="python -W ignore -m paper_2308_10459_b200._build"
$B --out=scratch/libs/rows_E3.so -DBDEM_ELEM_MINB=3
$B --out=scratch/libs/rows_E4.so -DBDEM_ELEM_MINB=4
$B --out=scratch/libs/rows_H1.so -DBDEM_ROWS_HOIST=1 -DBDEM_ELEM_MINB=3
$B --out=scratch/libs/rows_M10.so -DBDEM_ASM_MINB=10 -DBDEM_ELEM_MINB=3
$B --out=scratch/libs/rows_M12.so -DBDEM_ASM_MINB=12 -DBDEM_ELEM_MINB=3
