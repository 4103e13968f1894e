"""Collaboration specs used as fixtures, written as peer-group tables.

The reference fixtures (/root/reference/proj/scenarios/*.json) are uniform
groups of peers; each entry below names the file it restates and lists
(count, samples_per_sec, download_mbps, upload_mbps, extra flags). het8c /
het4b are the unique-fraction fixtures of SURVEY.md Appendix A."""
from paper_2106_10207_b200.fleets import FLEETS, homogeneous, spec, spec_json  # noqa: F401

# frozen xi goldens (/root/reference/proj/tests/cpp/test_strategy.cpp:189,200,213-220)
XI_GOLDEN = {
    "homogeneous8": 0.697544642857, "aux_server": 1.220703125, "table1_a": 0.697544642857,
    "table1_b": 0.130208333333, "table1_c": 0.244140625, "table1_d": 0.217437744141,
    "daynight": 3.0, "static16": 2.0,
}
# SURVEY.md Appendix A (PROBE, HiGHS)
XI_APPENDIX_A = {"het8c": 0.269376624821, "het4b": 0.484955037085}
FRACTIONS_APPENDIX_A = {"het8c": [1 / 20] * 6 + [0.0, 7 / 10], "het4b": [1 / 22] * 3 + [19 / 22]}
