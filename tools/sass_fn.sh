# SASS of one kernel of the in-tree library: bash tools/sass_fn.sh SUBSTRING
lib=${LIB:-paper_2301_07457_b200/libtmg_gpu.so}
cuobjdump -sass "$lib" | awk -v pat="$1" '/Function : /{p = index($0, pat) > 0} p'
