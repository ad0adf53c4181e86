# A/B builds of the slice-CTA bond kernel (BDEM_LIB selects one at run time)
set -e
cd /root/repo
B="python -W ignore -m paper_2308_10459_b200._build"
$B --out=scratch/libs/asm_W3.so -DBDEM_SLC_WARPS=3 -DBDEM_SLC_MINB=5
$B --out=scratch/libs/asm_W4.so -DBDEM_SLC_WARPS=4 -DBDEM_SLC_MINB=4
$B --out=scratch/libs/asm_W6.so -DBDEM_SLC_WARPS=6 -DBDEM_SLC_MINB=2
$B --out=scratch/libs/asm_W2n.so -DBDEM_ROW_NOINLINE=1
