for f in variants/libgplan_fix*.so; do GPLAN_LIB=$PWD/$f timeout 600 python -m pytest tests -x -q -m gpu -k "golden or slices or ranges or fast or deferred" 2>&1 | tail -1; done
bash tools/variants.sh; bash tools/variants.sh
