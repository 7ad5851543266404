"""``python -m paper_2510_27191_b200`` -- the campaign CLI (mirror of ``python -m vecpomdp`` /
``vecpomdp-bench``, /root/reference/pkg/src/vecpomdp/__main__.py, bench.py:165-214)."""

from .campaign import main

if __name__ == "__main__":
    raise SystemExit(main())
