"""Hypothesis strategies shared by the fuzz tests: model configurations the reference accepts
(predation.hpp:13-27, traffic.hpp:13-17, finance.hpp:13-22). Energies, gains and metabolism
are multiples of 1/8, so every value stays on the reference's 2^-20 energy grid."""
from hypothesis import strategies as st


@st.composite
def predation_cfg(draw, max_side=40, max_cap=400):
    w = draw(st.integers(1, max_side))
    h = draw(st.integers(1, max_side))
    cs = draw(st.integers(0, max_cap))
    cw = draw(st.integers(0, max_cap // 2))
    return dict(width=w, height=h,
                n_sheep0=draw(st.integers(0, cs)), n_wolves0=draw(st.integers(0, cw)),
                sheep_capacity=cs, wolf_capacity=cw,
                energy_gain_sheep=draw(st.sampled_from([1.0, 4.0, 7.25, 4.0, 0.5])),  # 0.5: refused
                energy_gain_wolf=draw(st.sampled_from([2.0, 20.0, 33.5, 20.0, 0.0])),  # 0.0: refused
                metabolism=draw(st.sampled_from([0.0, 0.25, 1.0, 3.0])),
                reproduce_prob_sheep=draw(st.sampled_from([0.0, 0.04, 0.3, 1.0])),
                reproduce_prob_wolf=draw(st.sampled_from([0.0, 0.05, 0.5, 1.0])),
                reproduce_energy_frac=draw(st.sampled_from([0.0, 0.25, 0.5, 1.0])),
                regrow_delay=draw(st.integers(-2, 40)))


@st.composite
def traffic_cfg(draw):
    return dict(length=draw(st.integers(1, 300)), period=draw(st.integers(1, 25)),
                green_fraction=draw(st.sampled_from([0.0, 0.1, 0.5, 0.9, 1.0])))


@st.composite
def finance_cfg(draw):
    return dict(books=draw(st.integers(1, 6)), traders=draw(st.integers(0, 40)),
                book_capacity=draw(st.integers(1, 300)),
                p_order=draw(st.sampled_from([0.0, 0.2, 0.5, 1.0])),
                delta=draw(st.sampled_from([0.0, 0.01, 0.05, 0.5, 1.5])),
                qmax=draw(st.integers(1, 20)), max_order_age=draw(st.integers(-1, 30)),
                init_price=draw(st.sampled_from([100.0, 0.5, 1e-3, 12345.678])))
