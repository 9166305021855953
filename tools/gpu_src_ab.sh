# Same-box A/B of a kernel source file: the working tree's version vs an alternative
# copy (e.g. HEAD's, written by `git show HEAD:<path> > /tmp/alt.cu`).  Usage: bash tools/gpu_src_ab.sh <kernel file> <alt copy> <kbench mode> <grep>
k=$1; alt=$2; mode=$3; pat=$4
d=paper_2509_04719_b200/csrc/kernels
cp $d/$k /tmp/ab_new.cu
for v in new alt new alt; do
  if [ $v = alt ]; then cp $alt $d/$k; else cp /tmp/ab_new.cu $d/$k; fi
  touch $d/$k; python -m paper_2509_04719_b200.build > /tmp/b.log 2>&1 || { echo "build failed $v"; tail -3 /tmp/b.log; }
  echo "== $v"; timeout 300 python tools/kbench.py $mode 2>&1 | grep -E "$pat"
done
cp /tmp/ab_new.cu $d/$k; touch $d/$k; python -m paper_2509_04719_b200.build > /tmp/b.log 2>&1
