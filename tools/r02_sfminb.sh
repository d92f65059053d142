cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-sfm}; mkdir -p $o
for mb in 2 3; do DGM_SF_MINB=$mb timeout 900 python tools/curved_bench.py 12 1,2,3,4,5,6,7,8,9,10 > $o/curved_minb$mb.txt 2>&1; echo "minb $mb"; cat $o/curved_minb$mb.txt; done
