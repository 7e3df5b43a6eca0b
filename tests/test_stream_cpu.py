"""Active-set policy of the chunk streamer (NEXT-3), -m "not gpu":
zones grown by 25 % relative padding (1.25x per axis, reading N9)."""
import pytest

from paper_2503_11731_b200.stream import Zone, active_set, chunked_zones


def test_zone_padding_is_25_percent():
    z = Zone(-20.0, 20.0, 0.0, 40.0)            # a 40 x 40 m zone
    # padded zone: 50 x 50 m, i.e. 5 m beyond each side
    assert z.padded_contains(0.0, 44.999, 0.25) and not z.padded_contains(0.0, 45.001, 0.25)
    assert z.padded_contains(0.0, -4.999, 0.25) and not z.padded_contains(0.0, -5.001, 0.25)
    assert z.padded_contains(24.999, 10.0, 0.25) and not z.padded_contains(25.001, 10.0, 0.25)
    assert not z.padded_contains(0.0, 40.5, 0.0)


def test_chunked_street_active_sets():
    zones = chunked_zones()                       # 8 chunks of 50 m along z
    assert active_set(zones, (0.0, 1.5, 168.0)) == (3,)
    assert active_set(zones, (0.0, 1.5, 195.0)) == (3, 4)   # within 6.25 m of the boundary at 200
    assert active_set(zones, (0.0, 1.5, 231.0)) == (4,)
    assert active_set(zones, (0.0, 1.5, -100.0)) == ()
    # the Chunked trajectory (ego z = 168 + t) changes set exactly twice
    sets = [active_set(zones, (0.0, 1.5, 168.0 + t)) for t in range(64)]
    changes = [t for t in range(1, 64) if sets[t] != sets[t - 1]]
    assert changes == [26, 39]                    # enters chunk 4's padding at 193.75, leaves 3's at 206.25


@pytest.mark.parametrize("pad", [0.0, 0.25, 1.0])
def test_every_position_inside_the_road_has_a_zone(pad):
    zones = chunked_zones()
    for z in range(0, 400, 7):
        ids = active_set(zones, (3.0, 0.0, z + 0.5), pad)
        assert ids and all(zones[i].padded_contains(3.0, z + 0.5, pad) for i in ids)
        assert list(ids) == sorted(ids)
